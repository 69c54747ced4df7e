"""Driver for ncu: cfg2 quad Helmholtz (256^2 curved quads, P=6, Q=8), 2 applies."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

q6 = sp.make_quad(6, 8)
b = sp.ElementBatch.structured(q6, 256, kind=sp.GEOM_METRIC, mapping=sp.MAP_QUAD_SINE, amp=0.05)
c = sp.Collection(b, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC, lam=1.0)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (65536, 49)), device="cuda")
for _ in range(2):
    y = c.apply(x)
torch.cuda.synchronize()
print("ok")
