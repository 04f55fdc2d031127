// sobel5/rational.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/rational.hpp (rational.hpp:17-152) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   Rational
#pragma once

#include "sobel5_b200/core.hpp"
