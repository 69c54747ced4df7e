"""ncu driver: a few FUSED assembled applies on the cfg4 mesh (no timing)."""
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
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--alg", default="fused")
a = ap.parse_args()
exp = sp.make_hex(a.P, a.P + 2)
batch = sp.ElementBatch.structured(exp, a.n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
amap = sp.AssemblyMap.hex_periodic(a.n, a.P).set_algorithm(a.alg)
op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, amap.num_global), device="cuda")
y = torch.empty_like(x)
for _ in range(a.reps):
    op.apply(x, y)
torch.cuda.synchronize()
print("ok")
