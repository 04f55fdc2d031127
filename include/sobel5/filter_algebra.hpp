// sobel5/filter_algebra.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/filter_algebra.hpp (filter_algebra.hpp:14-256) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   Kernel5, Kernel3, kernel3_x/y, SeparablePair, FilterParams, Direction,
//   validate_params, materialize, make_kd_sum_diff, decompose_kd_minus
#pragma once

#include "sobel5_b200/params.hpp"
