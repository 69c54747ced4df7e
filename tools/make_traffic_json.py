"""ncu csv (--metrics dram__bytes_read.sum,dram__bytes_write.sum, one capture
of tools/prof_helm.py --mode both --alg class) -> the traffic record bench.py
reports as roofline.traffic: DRAM bytes per launch of the class-range
operator (MODE 5) and of the fused local operator (MODE 0)."""
import csv
import json
import sys

src, dst, P, n = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
per = {}
for r in csv.reader(open(src)):
    if len(r) < 12 or r[0] in ("ID", ""):
        continue
    name, metric, unit, val = r[4], r[-3], r[-2], float(r[-1].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    per.setdefault((r[0], name), {})[metric] = val * scale
out = {}
for (lid, name), m in per.items():
    if "pipe_kernel" not in name:
        continue
    key = "helmholtz_class" if name.rstrip(")").endswith("5>(DevArgs") or ", 5>" in name else "helmholtz_local"
    tot = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    out.setdefault(key, []).append((tot, name, m))
rec = {}
for key, runs in out.items():
    tot = sorted(t for t, _, _ in runs)[len(runs) // 2]
    rec[key] = {"P": P, "n": n, "bytes_per_launch": tot, "kernel": runs[0][1], "launches": len(runs),
                "read": runs[0][2].get("dram__bytes_read.sum"), "write": runs[0][2].get("dram__bytes_write.sum")}
json.dump(rec, open(dst, "w"), indent=1)
print(json.dumps(rec, indent=1))
