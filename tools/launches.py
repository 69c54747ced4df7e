"""Summarise an ncu --csv launch list: kernel, time (us), dram read/write MB."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launches = OrderedDict()
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    d = launches.setdefault(r[ii], {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
for i, d in launches.items():
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    rd = d.get("dram__bytes_read.sum", 0) / 1e6
    wr = d.get("dram__bytes_write.sum", 0) / 1e6
    bw = (rd + wr) / t * 1e3 if t else 0
    print(f"{i:>4} {d['name'][:58]:58s} {t:9.1f} us  R {rd:8.1f} MB  W {wr:8.1f} MB  {bw:6.0f} GB/s")
