cd "${GRAFT_REPO_ROOT:-/root/repo}"
L=paper_2305_00515_b200/lib/libsobel5_b200.so; cp $L /tmp/orig.so
for round in 1 2; do for v in build/variants/lib*.so; do cp $v $L
  for c in sr u8; do echo "$round $(basename $v) 5x5 $c $(GRAPH=1 CONTRACT=$c timeout 60 python tools/sweep.py | tail -1)"; done
  for c in sr3 u8; do echo "$round $(basename $v) 3x3 $c $(GRAPH=1 SOBEL3=1 CONTRACT=$c timeout 60 python tools/sweep.py | tail -1)"; done
done; done
cp /tmp/orig.so $L
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_u8_only.py tests/test_gpu_sobel3.py tests/test_gpu_detect.py 2>&1 | tail -1
