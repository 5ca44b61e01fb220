#!/bin/bash
# The round's evidence in one gpurun call (1 GPU):  bash tools/refresh_evidence.sh TAG
# then here: python tools/evidence_summary.py TAG ; copy the listed files into profiles/.
tag=${1:-ev}
python bench.py > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>> gpurun_out/${tag}_bench.err
python tools/timeline.py > gpurun_out/${tag}_timeline.txt 2>&1
python tools/bench_configs.py A C D E > gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs.err
python tools/stage_timing.py --deterministic > gpurun_out/${tag}_det_stage_timing.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py --iters 5 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_det_launches.csv \
    python tools/profile_step.py --iters 3 --deterministic > /dev/null 2>&1
for c in C E; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_${c}_launches.csv \
      python tools/config_step.py $c > /dev/null 2>&1
done
# per-kernel counters + full captures (tools/evidence.sh without the sanitizer pass)
sed '/sanitize.sh/d' tools/evidence.sh > /tmp/evidence_nosan.sh
bash /tmp/evidence_nosan.sh ${tag}
ls gpurun_out | grep ${tag}
bash tools/sanitize.sh > gpurun_out/${tag}_sanitize.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
