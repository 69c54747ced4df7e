"""cfg2 quad operators (256^2 curved quads, P=6, Q=8) and cfg1 (32^2, P=4):
device time and HBM fraction per operator (library variant via
SPHP_LIBRARY_VARIANT)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
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
q6 = sp.make_quad(6, 8)
for kind, ops in ((sp.GEOM_METRIC, ("helmholtz",)), (sp.GEOM_POINT, ("physderiv", "iproductwrtbase",
                                                                      "iproductwrtderivbase"))):
    b = sp.ElementBatch.structured(q6, 256, kind=kind, mapping=sp.MAP_QUAD_SINE, amp=0.05)
    for op in ops:
        c = sp.Collection(b, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC, lam=1.0)
        x = torch.as_tensor(rng.uniform(-1, 1, (65536, c.input_size)), device="cuda")
        y = torch.empty(c.output_shape, dtype=torch.float64, device="cuda")
        ms = timed(lambda: c.apply(x, y))
        res[f"cfg2_{op}"] = (round(ms * 1e3, 1), round(c.hbm_bytes() / (ms * 1e-3) / 1e9 / peak, 3))
bq = sp.ElementBatch.standard(q6, 65536)
for op in ("bwdtrans",):
    c = sp.Collection(bq, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
    x = torch.as_tensor(rng.uniform(-1, 1, (65536, c.input_size)), device="cuda")
    y = torch.empty(c.output_shape, dtype=torch.float64, device="cuda")
    ms = timed(lambda: c.apply(x, y))
    res[f"cfg2_{op}"] = (round(ms * 1e3, 1), round(c.hbm_bytes() / (ms * 1e-3) / 1e9 / peak, 3))
print(json.dumps(res))
