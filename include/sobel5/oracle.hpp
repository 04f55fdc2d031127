// sobel5/oracle.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/oracle.hpp (oracle.hpp:19-129) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   conv2d_valid (5x5 and 3x3), Sobel3Result / sobel3_2d, Sobel5Result /
//   sobel5_4d, DiagPair / diag_via_sum_diff -- all on the GPU
#pragma once

#include "sobel5_b200/stream.hpp"
#include "sobel5_b200/detect.hpp"
#include "sobel5_b200/verify.hpp"
