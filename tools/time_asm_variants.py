"""Compare assembled-apply variants on the cfg4 mesh: analytic periodic map
vs the same map materialised as explicit codes, owner vs colour sums."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402


def timed(fn, reps=10):
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


n = 64
for P in [int(p) for p in (sys.argv[1] if len(sys.argv) > 1 else "2,4,6,8").split(",")]:
    exp = sp.make_hex(P, P + 2)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
    per = sp.AssemblyMap.hex_periodic(n, P)
    expl = sp.AssemblyMap.explicit(per.codes(), per.num_global)
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, per.num_global), device="cuda")
    ys = {}
    res = {}
    for name, amap, alg in (("periodic-owner", per, "owner"), ("periodic-split", per, "split"),
                            ("explicit-owner", expl, "owner"), ("periodic-colour", per, "colour")):
        amap.set_algorithm(alg)
        op = sp.GlobalHelmholtz([(coll, amap)], per.num_global)
        y = torch.empty_like(x)
        res[name] = timed(lambda: op.apply(x, y))
        ys[name] = y.clone()
    ref = ys["periodic-owner"]
    err = {k: float((v - ref).abs().max() / ref.abs().max()) for k, v in ys.items()}
    print(P, {k: round(v, 3) for k, v in res.items()}, {k: f"{v:.1e}" for k, v in err.items()}, flush=True)
    del coll, batch, per, expl, x, ys
    torch.cuda.empty_cache()
