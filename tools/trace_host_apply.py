"""Timeline of one host-buffer assembled apply (slab pipeline) with
torch.profiler (CUPTI): prints copy / kernel intervals per stream."""
import json
import sys
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

n, P = 64, 4
exp = sp.make_hex(P, P + 2)
batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
amap = sp.AssemblyMap.hex_periodic(n, P)
op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, amap.num_global)).pin_memory()
y = torch.empty_like(x).pin_memory()
for _ in range(3):
    op.apply_host(x, y)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    op.apply_host(x, y)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/host_apply_trace.json")
ev = json.load(open("gpurun_out/host_apply_trace.json"))["traceEvents"]
rows = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in rows)
for e in sorted(rows, key=lambda e: e["ts"]):
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} s{e.get('args', {}).get('stream', '?'):>4} {e['cat']:10s} {e['name'][:60]}")
