"""Time the fused local and assembled hex Helmholtz (cfg4 mesh) for a list
of orders; one JSON line per order.  Used for tile-variant tuning
(SPHP_HELM_VARIANT) — not a benchmark line."""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", default="2,4,6,8")
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()


def timed(fn, reps):
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


for P in [int(p) for p in a.P.split(",")]:
    exp = sp.make_hex(P, P + 2)
    batch = sp.ElementBatch.structured(exp, a.n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
    E = a.n ** 3
    m, Q = P + 1, P + 2
    c = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (E, m ** 3)), device="cuda")
    y = torch.empty_like(c)
    t_local = timed(lambda: coll.apply(c, y), a.reps)
    amap = sp.AssemblyMap.hex_periodic(a.n, P)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, amap.num_global), device="cuda")
    yg = torch.empty_like(x)
    t_asm = timed(lambda: op.apply(x, yg), a.reps)
    lb = 8 * (2 * m ** 3 + 7 * Q ** 3) * E
    print(json.dumps({"variant": os.environ.get("SPHP_HELM_VARIANT", "0"), "P": P, "local_ms": t_local,
                      "asm_ms": t_asm, "local_frac": lb / (t_local * 1e-3) / 6547.2e9,
                      "asm_local_dof_s": E * m ** 3 / (t_asm * 1e-3)}), flush=True)
    del coll, batch, c, y, op, amap, x, yg
    torch.cuda.empty_cache()
