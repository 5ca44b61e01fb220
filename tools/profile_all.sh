#!/bin/bash
# One ncu --set full capture (second training iteration) of every hot kernel
# at config B, into gpurun_out/<tag>_<kernel>.ncu-rep; run under gpurun.
#   bash tools/profile_all.sh r01b
tag=${1:-prof}
for k in project_cull_compact tile_count_kernel st_scatter_kernel st_sort_emit_kernel raster_fwd_kernel loss_kernel \
         raster_bwd_kernel chain_kernel adam_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${tag}_${k} python tools/profile_step.py --iters 2 > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py --iters 2 > /dev/null 2>&1
