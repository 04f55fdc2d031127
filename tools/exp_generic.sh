#!/bin/bash
# A/B of generic-kernel occupancy variants (build/variants/libgen*.so) on FilterParams that need kernel B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
L=paper_2305_00515_b200/lib/libsobel5_b200.so
cp $L /tmp/orig.so
for round in 1 2; do for v in build/variants/libgen*.so; do
  cp $v $L
  PARAMS="1,32768,1,1" python tools/params_bench.py 2>&1 | sed "s|^|$round $(basename $v) |"
done; done
cp /tmp/orig.so $L
