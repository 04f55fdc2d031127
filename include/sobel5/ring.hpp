// sobel5/ring.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/ring.hpp (ring.hpp:16-124) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   RowRing, KdVariant, KdPlusBank
#pragma once

#include "sobel5_b200/stream.hpp"
