"""Split vs fused assembled Helmholtz on the cfg4 mesh (64^3 periodic
deformed hexes) for a list of orders; bitwise check between the two."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", default="2,3,4,5,6,7,8")
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--reps", type=int, default=20)
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
    amap = sp.AssemblyMap.hex_periodic(a.n, P)
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, amap.num_global), device="cuda")
    res, ys = {}, {}
    for alg in ("split", "fused"):
        amap.set_algorithm(alg)
        op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
        y = torch.empty_like(x)
        res[alg] = timed(lambda: op.apply(x, y), a.reps)
        ys[alg] = y.clone()
    E, m = a.n ** 3, P + 1
    print(json.dumps({"P": P, **{k + "_ms": round(v, 4) for k, v in res.items()},
                      "fused_local_dof_s": E * m ** 3 / (res["fused"] * 1e-3),
                      "bitwise": bool(torch.equal(ys["split"], ys["fused"]))}), flush=True)
    del coll, batch, amap, x, ys
    torch.cuda.empty_cache()
