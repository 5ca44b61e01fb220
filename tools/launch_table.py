"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes):
per kernel of a training iteration, the mean over every iteration after the
first in the file (min / max alongside).   python tools/launch_table.py FILE"""
import collections
import csv
import statistics
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i
        break
iid, iname, im, iv = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
per = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) > iv:
        per.setdefault((int(r[iid]), r[iname][:72]), {})[r[im]] = float(r[iv].replace(",", ""))
items = list(per.items())
firsts = [i for i, (k, _) in enumerate(items) if "project_cull" in k[1]]
iters = [items[a:b] for a, b in zip(firsts, firsts[1:] + [len(items)])]
use = iters[1:] if len(iters) > 1 else iters
# kernel sequence of the last iteration; align the others by position
ref = use[-1]
tot = 0.0
for pos, ((_, name), m) in enumerate(ref):
    ts = [it[pos][1].get("gpu__time_duration.sum", 0) / 1e3 for it in use if len(it) == len(ref)]
    t = statistics.mean(ts)
    tot += t
    print(f"{t:8.1f} us [{min(ts):6.1f} {max(ts):6.1f}]  R {m.get('dram__bytes_read.sum', 0) / 1e6:7.1f} MB  "
          f"W {m.get('dram__bytes_write.sum', 0) / 1e6:7.1f} MB  {name}")
print(f"total {tot:.1f} us  (mean of {len(use)} iterations)")
