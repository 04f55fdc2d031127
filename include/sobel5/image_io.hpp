// sobel5/image_io.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/image_io.hpp (image_io.hpp:225-291) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   SaveMode, detail::quantize, PaddedPlane, pad_replicate, and the GPU
//   detect path; the PGM/PNG file I/O of image_io.hpp:20-223 is not part of
//   this build
#pragma once

#include "sobel5_b200/detect.hpp"
