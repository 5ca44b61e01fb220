#!/bin/bash
# The round's ncu / SASS / sanitizer evidence at config B (run under gpurun, 1 GPU):
#   bash tools/evidence.sh r02
# then here:  python tools/evidence_summary.py r02   (writes profiles/r02_*)
tag=${1:-ev}
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,sm__cycles_active.avg
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active
M=$M,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
M=$M,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum
M=$M,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_requests_srcunit_tex_op_red.sum
M=$M,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_requests_srcunit_tex_op_atom.sum
M=$M,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,smsp__sass_branch_targets.sum,smsp__sass_branch_targets_threads_divergent.sum
M=$M,smsp__sass_branch_targets_threads_uniform.sum,smsp__thread_inst_executed_per_inst_executed.ratio
M=$M,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_xu.sum
M=$M,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
M=$M,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_metrics.csv \
    python tools/profile_step.py --iters 2 > /dev/null 2>&1
for k in raster_fwd_kernel raster_bwd_kernel loss_kernel st_sort_emit_kernel tile_count_kernel \
         project_cull_compact_kernel chain_kernel adam_kernel st_scatter_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${tag}_full_${k} python tools/profile_step.py --iters 2 > /dev/null 2>&1
done
bash tools/sanitize.sh > gpurun_out/${tag}_sanitize.txt 2>&1
