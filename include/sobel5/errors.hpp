// sobel5/errors.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/errors.hpp (errors.hpp:9-32) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   Error and its leaf exception types
#pragma once

#include "sobel5_b200/core.hpp"
