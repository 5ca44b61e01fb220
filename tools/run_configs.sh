#!/bin/bash
# Config C/E throughput lines and ncu launch lists (run under gpurun):
#   bash tools/run_configs.sh [tag]
tag=${1:-cfg}
python tools/bench_configs.py C E > gpurun_out/${tag}.jsonl 2> gpurun_out/${tag}.err; tail -2 gpurun_out/${tag}.err
for c in C E; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_${c}_launches.csv \
      python tools/config_step.py $c > /dev/null 2>&1
done
