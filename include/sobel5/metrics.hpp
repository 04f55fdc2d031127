// sobel5/metrics.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/metrics.hpp (metrics.hpp:20-179) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   SsimStats / ssim_global, DiffStats / diff_stats, BenchReport / measure
#pragma once

#include "sobel5_b200/verify.hpp"
