#!/bin/bash
# The paper's three ideas, ablated on B200 at 8K: timing + ncu counters.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=paper_2305_00515_b200/lib/libsobel5_b200.so
cp $L /tmp/orig.so
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__sass_inst_executed_op_global_ld.sum,sm__sass_inst_executed_op_shared_ld.sum,sm__sass_inst_executed_op_shared_st.sum,smsp__l1tex_lsuin_requests.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed
for v in default:/tmp/orig.so colshare_loads:build/variants/lib_cs1.so colshare_smem:build/variants/lib_cs2.so; do
  tag=${v%%:*}; lib=${v#*:}
  cp $lib $L
  TAG=$tag python tools/ablation.py
  for cfg in sr,1,0 sr,0,0 sr,1,1 u8,1,0 u8,1,1; do
    if [ $tag != default ] && [ $cfg != sr,1,0 ] && [ $cfg != u8,1,0 ]; then continue; fi
    echo "== ncu $tag $cfg"
    TAG=$tag ONLY=$cfg ncu --metrics $M --clock-control none -k regex:"sobel5_(packed|dense)" -s 7 -c 1 --csv python tools/ablation.py 2>/dev/null | grep -E "\"(gpu__|smsp__|sm__|l1tex__|dram__)" | awk -F'","' '{print $(NF-2)" = "$NF}' | tr -d '"'
  done
done
cp /tmp/orig.so $L
