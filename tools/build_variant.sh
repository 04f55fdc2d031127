#!/bin/bash
# Build a variant of the library with extra nvcc defines into build/variants/<name>/
# usage: tools/build_variant.sh <name> "<nvcc extra flags>"
cd "$(dirname "$0")/.."
name=$1; shift
SOBEL5_NVCC_EXTRA="$*" SOBEL5_LIB_OUT=build/variants/$name/libsobel5_b200.so python -c "
import os
from paper_2305_00515_b200 import build as b
b.OBJDIR = os.path.join(b.ROOT, 'build', 'obj_' + '$name')
b.LIB = os.path.join(b.ROOT, 'build', 'variants', '$name', 'libsobel5_b200.so')
os.makedirs(os.path.dirname(b.LIB), exist_ok=True)
b.build(force=True)
print(b.LIB)"
