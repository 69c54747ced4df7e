"""Race hunt: repeat the class-assembled and local applies of every order on
a large mesh and compare every result bitwise with the first one (the
kernels have no atomics: any difference is a synchronisation bug)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bad = 0
for P in range(2, 9):
    exp = sp.make_hex(P, P + 2)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
    amap = sp.AssemblyMap.hex_periodic(n, P)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    x = torch.as_tensor(np.random.default_rng(P).uniform(-1, 1, amap.num_global), device="cuda")
    c = torch.as_tensor(np.random.default_rng(P).uniform(-1, 1, (n ** 3, (P + 1) ** 3)), device="cuda")
    y0, l0 = op.apply(x).clone(), coll.apply(c).clone()
    side = torch.cuda.Stream()
    for r in range(reps):
        y = torch.empty_like(y0)
        lo = torch.empty_like(l0)
        # a concurrent apply on a second stream perturbs the schedule
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            coll.apply(c, lo, stream=side)
        op.apply(x, y)
        torch.cuda.synchronize()
        if not (torch.equal(y, y0) and torch.equal(lo, l0)):
            bad += 1
            print(f"P={P} rep {r}: MISMATCH asm {torch.equal(y, y0)} local {torch.equal(lo, l0)}", flush=True)
    print(f"P={P}: {reps} repeats done", flush=True)
    del coll, batch, op, amap, x, c
    torch.cuda.empty_cache()
print("mismatches:", bad)
sys.exit(1 if bad else 0)
