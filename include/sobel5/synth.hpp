// sobel5/synth.hpp -- source-compatibility header of the B200 drop-in.
//
// Replaces the reference's proj/include/sobel5/synth.hpp (synth.hpp:11-57) so a
// translation unit written against the reference builds unchanged with
// -I<repo>/include and links -lsobel5_b200.  Provides:
//   splitmix64, synth_random, synth_ramp_x, synth_constant, synth_impulse
#pragma once

#include "sobel5_b200/stream.hpp"
