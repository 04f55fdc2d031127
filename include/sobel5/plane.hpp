// sobel5/plane.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/plane.hpp (plane.hpp:14-72) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   Plane<T>, GrayPlane, SignedPlane, RealPlane
#pragma once

#include "sobel5_b200/core.hpp"
