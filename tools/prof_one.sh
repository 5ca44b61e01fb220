#!/bin/bash
# ncu --set full of one kernel at config B (second iteration): bash tools/prof_one.sh TAG KERNEL_REGEX
ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
    -o gpurun_out/$1 python tools/profile_step.py --iters 2 > /dev/null 2>&1
ls -la gpurun_out/$1*
