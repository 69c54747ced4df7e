"""ncu driver: cfg5 (48^3 deformed hexes, per-element P in {3..7}) assembled
Helmholtz applies through GlobalHelmholtz (no timing)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

n5 = 48
orders = np.random.default_rng(20240801 + 5).integers(3, 8, n5 ** 3)
ng, maps = sp.hex_variable_maps(n5, orders)
batches = []
for P, (ids, amap) in maps.items():
    e = sp.make_hex(P, P + 2)
    bb = sp.ElementBatch.structured(e, n5, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03,
                                    elem_ids=ids, device="cuda")
    batches.append((sp.Collection(bb, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC), amap))
g = sp.GlobalHelmholtz(batches, ng)
x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, ng), device="cuda")
y = torch.empty_like(x)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    g.apply(x, y)
torch.cuda.synchronize()
print("ok", ng, {P: len(ids) for P, (ids, _) in maps.items()})
