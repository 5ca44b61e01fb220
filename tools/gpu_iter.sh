#!/bin/bash
# One build -> measure round trip on the GPU box (run under gpurun):
#   bash tools/gpu_iter.sh TAG [pytest -k expr]
# GPU parity tests, then the ncu launch list of two config-B iterations.
tag=${1:-it}
k=${2:-}
if [ -n "$k" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$k" 2>&1 | tail -4 > gpurun_out/${tag}_tests.txt
else
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/${tag}_tests.txt
fi
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py --iters 5 > /dev/null 2>&1
cat gpurun_out/${tag}_tests.txt
python tools/launch_table.py gpurun_out/${tag}_launches.csv
