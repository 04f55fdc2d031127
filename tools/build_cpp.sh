#!/bin/bash
# Builds the C++ API test against the drop-in headers and the in-tree .so.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
mkdir -p "$ROOT/build"
LIB="$ROOT/paper_2305_00515_b200/lib"
${CXX:-g++} -std=c++20 -O2 -Wall -Wextra -I"$ROOT/include" "$ROOT/tests/cpp/test_api.cpp" \
  -L"$LIB" -lsobel5_b200 -lz -Wl,-rpath,"$LIB" -o "$ROOT/build/test_api"
# end-to-end timing of the drop-in C++ API (tools/cpp_e2e.cpp)
${CXX:-g++} -std=c++20 -O2 -Wall -Wextra -I"$ROOT/include" -I/usr/local/cuda/include "$ROOT/tools/cpp_e2e.cpp" \
  -L"$LIB" -lsobel5_b200 -lz -Wl,-rpath,"$LIB" -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 \
  -o "$ROOT/build/cpp_e2e"
# SPEC acceptance criteria as a reference-style program (only "sobel5/*.hpp"
# includes): the same source also builds against the reference headers
${CXX:-g++} -std=c++20 -O2 -Wall -Wextra -I"$ROOT/include" "$ROOT/tests/cpp/acceptance.cpp" \
  -L"$LIB" -lsobel5_b200 -lz -Wl,-rpath,"$LIB" -o "$ROOT/build/acceptance"
