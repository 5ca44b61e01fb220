#!/bin/bash
# Kernel A/B on the GPU box: ncu launch lists of 5 config-B iterations for the
# in-tree library and for every variant build given (under gpurun):
#   bash tools/ab.sh TAG build/variants/libA.so build/variants/libB.so ...
tag=$1; shift
run() {  # name, lib-or-empty
  SB_LIB_VARIANT=$2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/${tag}_$1.csv python tools/profile_step.py --iters 5 > /dev/null 2>&1
  echo "== $1 $2"; python tools/launch_table.py gpurun_out/${tag}_$1.csv
}
run base ""
i=0
for v in "$@"; do i=$((i+1)); run v$i "$v"; done
