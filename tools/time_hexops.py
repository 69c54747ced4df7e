"""cfg3 hex operators (64^3 affine hexes, P=4, Q=6) and the curved
(POINT-geometry) variants: device time and HBM fraction
(library variant via SPHP_LIBRARY_VARIANT)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


peak = 6547.2
rng = np.random.default_rng(0)
res = {"variant": os.environ.get("SPHP_LIBRARY_VARIANT", "main")}
P = int(sys.argv[1]) if len(sys.argv) > 1 else 4
exp = sp.make_hex(P, P + 2)
E = 64 ** 3
b = sp.ElementBatch.structured(exp, 64, kind=sp.GEOM_AFFINE, mapping=sp.MAP_AFFINE)
for op in ("bwdtrans", "iproductwrtbase", "physderiv", "iproductwrtderivbase"):
    c = sp.Collection(b, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
    x = torch.as_tensor(rng.uniform(-1, 1, (E, c.input_size)), device="cuda")
    y = torch.empty(c.output_shape, dtype=torch.float64, device="cuda")
    ms = timed(lambda: c.apply(x, y))
    res[f"P{P}_{op}"] = (round(ms * 1e3, 1), round(c.hbm_bytes() / (ms * 1e-3) / 1e9 / peak, 3))
    del x, y
print(json.dumps(res))
