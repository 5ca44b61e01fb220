"""Summarise the ncu launch list of bench.py itself
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv python
bench.py ...`): per kernel name, the launch count, mean and total duration
and its share of all kernel time of the run, largest first.  ncu serialises
the launches and runs them cold, so the shares (not the absolute times) are
what compare with the bench's own CUDA-event timings.

    python tools/bench_launch_summary.py gpurun_out/TAG_bench_launches.csv
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
iname, im, iv = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value"))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[start + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        name = re.sub(r"\(.*", "", r[iname]).replace("<unnamed>::", "").replace("void ", "")
        tot[name] += float(r[iv].replace(",", "")) / 1e3
        cnt[name] += 1
allt = sum(tot.values())
print(f"# {sys.argv[1]}: {sum(cnt.values())} launches, {allt / 1e3:.2f} ms of kernel time")
print(f"# {'kernel':<44} {'launches':>8} {'mean us':>9} {'total us':>10} {'share':>6}")
for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {name[:44]:<44} {cnt[name]:>8} {t / cnt[name]:>9.1f} {t:>10.1f} {100 * t / allt:>5.1f}%")
