"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) for
the last training iteration in it.   python tools/launch_table.py FILE"""
import collections
import csv
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
first = [i for i, (k, _) in enumerate(items) if "project_cull" in k[1]][-1]
tot = 0.0
for (_, name), m in items[first:]:
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    print(f"{t:8.1f} us  R {m.get('dram__bytes_read.sum', 0) / 1e6:7.1f} MB  "
          f"W {m.get('dram__bytes_write.sum', 0) / 1e6:7.1f} MB  {name}")
print(f"total {tot:.1f} us")
