#!/bin/bash
# A/B of prebuilt variants (build/variants/lib*.so): 8K SR, SR32 (int + g32), u8, 3 rounds interleaved
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=paper_2305_00515_b200/lib/libsobel5_b200.so
cp $L /tmp/orig.so
for round in 1 2 3; do
for v in build/variants/lib*.so; do
  cp $v $L
  for c in ${CONTRACTS:-sr u8}; do
    echo "$round $(basename $v) $c $(CONTRACT=$c BANDS=${BANDS:-0} python tools/sweep.py 2>&1 | tail -1)"
  done
done
done
cp /tmp/orig.so $L
