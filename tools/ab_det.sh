tag=$1; shift
run() {
  SB_LIB_VARIANT=$2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_$1.csv python tools/profile_step.py --iters 3 --deterministic > /dev/null 2>&1
  echo "== $1 $2"; python tools/launch_table.py gpurun_out/${tag}_$1.csv | grep -E "det_reduce|total"
}
run base ""
i=0; for v in "$@"; do i=$((i+1)); run v$i "$v"; done
