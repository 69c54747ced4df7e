"""Class-range assembly (operator MODE 5 + class_owner_sum) against the split
algorithm on the cfg4 mesh: bitwise comparison and CUDA-event timings per P."""
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


n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
for P in [int(p) for p in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,5,6,7,8").split(",")]:
    exp = sp.make_hex(P, P + 2)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
    per = sp.AssemblyMap.hex_periodic(n, P)
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, per.num_global), device="cuda")
    ys, res = {}, {}
    for alg in ("split", "class"):
        per.set_algorithm(alg)
        op = sp.GlobalHelmholtz([(coll, per)], per.num_global)
        y = torch.full_like(x, float("nan"))
        op.apply(x, y)
        torch.cuda.synchronize()
        ys[alg] = y.clone()
        res[alg] = timed(lambda: op.apply(x, y))
    d = (ys["class"] - ys["split"]).abs().max().item()
    same = bool(torch.equal(ys["class"], ys["split"]))
    print(f"P={P} n={n} split {res['split']:.4f} ms class {res['class']:.4f} ms "
          f"bitwise_equal={same} maxdiff={d:.2e} nan={bool(torch.isnan(ys['class']).any())}", flush=True)
    del coll, batch, per, x, ys
    torch.cuda.empty_cache()
