"""Times the periodic scatter and owner-sum kernels alone (P = 2..8, n = 64)
through AssemblyMap.scatter / assemble; env SPHP_PERIODIC_L / _CTAS tune."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402
from paper_1906_03489_b200.assembly import assemble, scatter  # noqa: E402


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
    return e0.elapsed_time(e1) / reps * 1e3


n = 64
tag = f"L={os.environ.get('SPHP_PERIODIC_L', '-')} ctas={os.environ.get('SPHP_PERIODIC_CTAS', '-')}"
for P in [int(p) for p in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,5,6,7,8").split(",")]:
    amap = sp.AssemblyMap.hex_periodic(n, P)
    amap.set_algorithm("owner")
    nm = (P + 1) ** 3
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, amap.num_global), device="cuda")
    loc = torch.empty(n ** 3 * nm, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ts = timed(lambda: scatter(amap, x, loc))
    ta = timed(lambda: assemble(amap, loc, y))
    mb = (x.numel() + loc.numel()) * 8 / 1e6
    print(f"{tag} P={P} scatter {ts:7.1f} us ({mb / ts:5.2f} TB/s)  owner {ta:7.1f} us ({mb / ta:5.2f} TB/s)",
          flush=True)
