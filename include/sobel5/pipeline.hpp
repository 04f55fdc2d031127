// sobel5/pipeline.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/pipeline.hpp (pipeline.hpp:21-573) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   Prefetch, OpCounters, StreamTaps, make_stream_taps, hpass_*, vagg_*,
//   recover_diag, StreamResult, run_stream (GPU), Stream3Result,
//   run_stream_3x3 (GPU)
#pragma once

#include "sobel5_b200/stream.hpp"
#include "sobel5_b200/detect.hpp"
