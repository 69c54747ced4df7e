"""Summarise an ncu report's source page: shared-memory excess wavefronts
and stall samples per CUDA source line (needs -lineinfo + --import-source)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
fname, h = "?", None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        h = {k: i for i, k in reversed(list(enumerate(r)))}
        continue
    if h is None or not r[0].isdigit():
        continue
    try:
        exc = float(r[h["L1 Wavefronts Shared Excessive"]] or 0)
        wf = float(r[h["L1 Wavefronts Shared"]] or 0)
        smp = float(r[h["Warp Stall Sampling (All Samples)"]] or 0)
    except (KeyError, ValueError, IndexError):
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0.0, 0.0, 0.0, r[1].strip()[:80]])
    a[0] += exc
    a[1] += wf
    a[2] += smp
vals = list(agg.items())
tot = [sum(v[i] for _, v in vals) for i in range(3)]
print(f"total: excess wavefronts {tot[0]:.3e}, wavefronts {tot[1]:.3e}, stall samples {tot[2]:.0f}")
print("-- by excess shared wavefronts")
for k, v in sorted(vals, key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:10.3e} {v[1]:10.3e} {v[2]:7.0f}  {k[0]}:{k[1]}: {v[3]}")
print("-- by stall samples")
for k, v in sorted(vals, key=lambda kv: -kv[1][2])[:top]:
    print(f"{v[0]:10.3e} {v[1]:10.3e} {v[2]:7.0f}  {k[0]}:{k[1]}: {v[3]}")
