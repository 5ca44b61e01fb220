"""Per-kernel key counters of one or more .ncu-rep files (every kernel in
each report), for the profiles/ summaries.
    python tools/ncu_kernels.py REPORT [REPORT...]"""
import csv
import subprocess
import sys

DETAILS = ['Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Achieved Active Warps Per SM',
           'Theoretical Occupancy', 'Registers Per Thread', 'DRAM Throughput', 'L2 Hit Rate']
RAW = ['smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
       'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio',
       'smsp__average_warps_issue_stalled_membar_per_issue_active.ratio',
       'smsp__sass_branch_targets_threads_divergent.sum', 'smsp__sass_branch_targets.sum',
       'sm__sass_inst_executed_op_global_red.sum', 'sm__sass_inst_executed_op_global_atom.sum',
       'lts__t_sectors_srcunit_tex_op_red.sum', 'lts__t_sectors_srcunit_tex_op_atom.sum',
       'sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
       'smsp__thread_inst_executed_per_inst_executed.ratio']


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    det = list(csv.reader(ncu([rep, "--page", "details", "--csv"]).splitlines()))
    kern = {}
    order = []
    for row in det[1:]:
        d = dict(zip(det[0], row))
        key = (d.get("ID"), d.get("Kernel Name"))
        if key not in kern:
            kern[key] = {}
            order.append(key)
        if d.get("Metric Name") in DETAILS:
            kern[key][d["Metric Name"]] = f'{d["Metric Value"]} {d.get("Metric Unit", "")}'.strip()
    raw = list(csv.reader(ncu([rep, "--page", "raw", "--csv"]).splitlines()))
    rh = raw[0] if raw else []
    rows = raw[2:] if len(raw) > 2 else []
    for i, key in enumerate(order):
        print(f"== {rep} #{key[0]}: {key[1][:90]}")
        for k in DETAILS:
            if k in kern[key]:
                print(f"   {k:34s} {kern[key][k]}")
        if i < len(rows):
            rv = dict(zip(rh, rows[i]))
            for k in RAW:
                if k in rv and rv[k] not in ("", "n/a"):
                    print(f"   {k:72s} {rv[k]}")
