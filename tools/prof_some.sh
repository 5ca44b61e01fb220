#!/bin/bash
tag=r02c
for k in project_cull_compact_kernel loss_kernel tile_count_kernel st_sort_emit_kernel chain_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${tag}_full_${k} python tools/profile_step.py --iters 2 > /dev/null 2>&1
done
ls -la gpurun_out
