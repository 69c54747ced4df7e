"""ncu driver: a few applies of one hex operator on the cfg3 mesh (64^3
affine, AFFINE geometry) at order P (no timing)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

op, P = sys.argv[1], int(sys.argv[2])
exp = sp.make_hex(P, P + 2)
b = sp.ElementBatch.structured(exp, 64, kind=sp.GEOM_AFFINE, mapping=sp.MAP_AFFINE)
c = sp.Collection(b, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (64 ** 3, c.input_size)), device="cuda")
y = torch.empty(c.output_shape, dtype=torch.float64, device="cuda")
for _ in range(2):
    c.apply(x, y)
torch.cuda.synchronize()
print("ok")
