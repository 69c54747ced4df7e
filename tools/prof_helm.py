"""Small driver for ncu: builds the cfg4 workload and runs a few applies of
the fused local Helmholtz and the assembled operator (no timing)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=4)
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", default="both", choices=["local", "assembled", "both"])
ap.add_argument("--alg", default=None)
a = ap.parse_args()
exp = sp.make_hex(a.P, a.P + 2)
batch = sp.ElementBatch.structured(exp, a.n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
E = a.n ** 3
if a.mode in ("local", "both"):
    c = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (E, (a.P + 1) ** 3)), device="cuda")
    y = torch.empty_like(c)
    for _ in range(a.reps):
        coll.apply(c, y)
if a.mode in ("assembled", "both"):
    amap = sp.AssemblyMap.hex_periodic(a.n, a.P)
    if a.alg:
        amap.set_algorithm(a.alg)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, amap.num_global), device="cuda")
    yg = torch.empty_like(x)
    for _ in range(a.reps):
        op.apply(x, yg)
torch.cuda.synchronize()
print("ok")
