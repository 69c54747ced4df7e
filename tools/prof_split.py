"""Runs the assembled P=4 cfg4 apply with the split and owner algorithms
(for an ncu launch list)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402
n, P = 64, 4
exp = sp.make_hex(P, P + 2)
batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
amap = sp.AssemblyMap.hex_periodic(n, P)
x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, amap.num_global), device="cuda")
y = torch.empty_like(x)
for alg in ("split", "owner"):
    amap.set_algorithm(alg)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    for _ in range(2):
        op.apply(x, y)
torch.cuda.synchronize()
print("ok")
