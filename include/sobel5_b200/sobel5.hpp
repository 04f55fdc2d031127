// sobel5_b200/sobel5.hpp -- umbrella header of the drop-in C++ API.
//
// Code written against the reference's headers
//     #include "sobel5/pipeline.hpp"   (plus filter_algebra/strips/plane/...)
// switches to the B200 implementation with
//     #include "sobel5_b200/sobel5.hpp"
// and links -lsobel5_b200 (paper_2305_00515_b200/lib).  Namespace, type and
// function names are the reference's (namespace sobel5).  See INTEGRATION.md.
#pragma once

#include "sobel5_b200/core.hpp"
#include "sobel5_b200/params.hpp"
#include "sobel5_b200/stream.hpp"
#include "sobel5_b200/detect.hpp"
