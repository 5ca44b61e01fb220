"""Summarise an .ncu-rep: key metrics, stall reasons, top instruction classes.
    python tools/ncu_summary.py REPORT [REPORT...]"""
import collections
import csv
import re
import subprocess
import sys

WANT = ['Duration', 'Executed Ipc Active', 'Achieved Active Warps Per SM', 'Registers Per Thread',
        'DRAM Throughput', 'Issue Slots Busy', 'Theoretical Occupancy', 'Grid Size', 'Memory Throughput',
        'L2 Hit Rate', 'L1/TEX Hit Rate']
STALLS = ['stall_barrier', 'stall_branch_resolving', 'stall_long_sb', 'stall_math', 'stall_mio', 'stall_no_inst',
          'stall_not_selected', 'stall_selected', 'stall_short_sb', 'stall_wait', 'stall_lg', 'stall_membar',
          'stall_drain', 'stall_dispatch', 'stall_sleep']


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    rows = list(csv.reader(run([rep, "--page", "details", "--csv"]).splitlines()))
    h = rows[0]
    name = ""
    vals = {}
    for row in rows[1:]:
        d = dict(zip(h, row))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in WANT:
            vals[d["Metric Name"]] = d["Metric Value"] + " " + d.get("Metric Unit", "")
    print(f"== {rep}: {name[:80]}")
    for k in WANT:
        if k in vals:
            print(f"   {k:32s} {vals[k]}")
    raw = list(csv.reader(run([rep, "--page", "raw", "--csv"]).splitlines()))
    if len(raw) >= 3:
        rv = dict(zip(raw[0], raw[2]))
        try:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                unit = raw[1][raw[0].index(m)]
                tot += float(rv[m].replace(",", "")) * scale.get(unit, 1)
            print(f"   {'DRAM bytes (read + write)':32s} {tot / 1e6:.1f} MB")
        except (KeyError, ValueError):
            pass
    src = list(csv.reader(run([rep, "--page", "source", "--csv", "--print-source", "sass"]).splitlines()))
    hdr = src[1]
    data = src[2:]
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    idx = [hdr.index(n) for n in STALLS if n in hdr]
    op = collections.Counter()
    tot = 0
    st = collections.Counter()
    for r in data:
        try:
            n = int(r[iE])
        except (ValueError, IndexError):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[iS].strip())
        op[m.group(2).split('.')[0] if m else '?'] += n
        tot += n
        for j in idx:
            try:
                st[hdr[j]] += int(r[j])
            except ValueError:
                pass
    s = sum(st.values()) or 1
    print(f"   warp instructions {tot / 1e6:.1f} M; top: " +
          ", ".join(f"{o} {n / 1e6:.1f}M" for o, n in op.most_common(8)))
    print("   stalls: " + ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in st.most_common(7)))
