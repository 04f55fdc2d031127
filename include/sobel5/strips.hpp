// sobel5/strips.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/strips.hpp (strips.hpp:13-61) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   Strip, StripPlan, plan_strips
#pragma once

#include "sobel5_b200/stream.hpp"
