cd "${GRAFT_REPO_ROOT:-/root/repo}"
L=paper_2305_00515_b200/lib/libsobel5_b200.so
cp $L /tmp/orig.so
for round in 1 2; do for v in 0 1; do
  cp build/variants/libwb$v.so $L
  for wl in 8k 1080p-batch 32k-bands; do
    echo "$round wb=$v $wl $(python bench.py --no-cpu-baseline --no-e2e --workload $wl --steps 20 | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1))')"
  done
  echo "$round wb=$v pad $(python tools/pad_time.py)"
done; done
cp /tmp/orig.so $L
