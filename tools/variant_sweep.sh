#!/bin/bash
# Time prebuilt library variants (build/variants/lib*.so) with tools/sweep.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=paper_2305_00515_b200/lib/libsobel5_b200.so
cp $L /tmp/orig.so
for v in build/variants/lib*.so; do
  cp $v $L
  for c in ${CONTRACTS:-sr}; do
    echo "== $v $c"; CONTRACT=$c BANDS=${BANDS:-16} python tools/sweep.py 2>&1 | tail -3
  done
done
cp /tmp/orig.so $L
