// sobel5/image_io.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/image_io.hpp (image_io.hpp:20-291) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200 -lz.  Provides:
//   SaveMode, detail::quantize, PaddedPlane, pad_replicate, and the GPU
//   detect path; luma_bt601, load_gray / save_gray (PGM P2 / P5, 8-bit PNG
//   on zlib instead of libpng: sobel5_b200/image_file.hpp)
#pragma once

#include "sobel5_b200/detect.hpp"
#include "sobel5_b200/image_file.hpp"
