"""Per-CUDA-source-line cost of one kernel in an .ncu-rep (needs -lineinfo and
--import-source on): warp-stall samples and warp instructions executed,
summed over the SASS each line maps to, top lines first.
    python tools/ncu_lines.py REPORT [TOP]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) > iE and r[0] and r[0] != "Line No":
        try:
            lines.append((int(r[iS]), int(r[iE]), r[0], r[1].strip()))
        except ValueError:
            pass
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"total samples {ts}, warp instructions {ti / 1e6:.1f} M")
for s, e, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% {100 * e / ti:5.1f}%  {ln:>5}  {src[:90]}")
