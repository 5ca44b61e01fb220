#!/bin/bash
# Everything a round's profiles/ snapshot needs (run under gpurun, 1 GPU):
#   bash tools/profile_round.sh r01g
tag=${1:-prof}
python bench.py > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${tag}_bench_reference.json 2>> gpurun_out/${tag}_bench.err
python tools/timeline.py > gpurun_out/${tag}_timeline.txt 2>&1
python tools/bench_configs.py A C D E > gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs.err
bash tools/profile_all.sh ${tag}
for c in C E; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_${c}_launches.csv \
      python tools/config_step.py $c > /dev/null 2>&1
done
