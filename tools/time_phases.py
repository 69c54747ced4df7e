"""Per-launch times (CUDA events between the launches of one assembled
apply, sphp_helmholtz_assembled_phases) of the default algorithm at every
P on the cfg4 mesh, with the roofline fractions of each launch."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

PEAK = 6557.1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
for P in [int(p) for p in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,5,6,7,8").split(",")]:
    E, Q, m = n ** 3, P + 2, P + 1
    exp = sp.make_hex(P, Q)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
    amap = sp.AssemblyMap.hex_periodic(n, P)
    for alg in ("class", "split"):
        amap.set_algorithm(alg)
        op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
        x = torch.as_tensor(np.random.default_rng(P).uniform(-1, 1, amap.num_global), device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            op.apply_phases(x, y)
        runs = [op.apply_phases(x, y) for _ in range(10)]
        ph = [statistics.median(r[i] for r in runs) for i in range(len(runs[0]))]
        ng = amap.num_global
        geo = 8 * 7 * Q ** 3 * E
        if alg == "class" and len(ph) == 2:
            ob = geo + 8 * ng + 8 * E * m ** 3
            sb = 8 * (E * (m ** 3 - (P - 1) ** 3) + ng - E * (P - 1) ** 3)
            print(f"P={P} class: operator {ph[0]:.3f} ms ({ob / ph[0] / 1e6 / PEAK:.2f}), "
                  f"owner {ph[1] * 1e3:.0f} us ({sb / ph[1] / 1e6 / PEAK:.2f}), total {sum(ph):.3f} ms "
                  f"(asm frac {(geo + 16 * ng) / sum(ph) / 1e6 / PEAK:.3f})", flush=True)
        else:
            print(f"P={P} {alg}: " + ", ".join(f"{v:.3f}" for v in ph) + f" ms, total {sum(ph):.3f} ms "
                  f"(asm frac {(geo + 16 * ng) / sum(ph) / 1e6 / PEAK:.3f})", flush=True)
    del coll, batch, amap, x, y, op
    torch.cuda.empty_cache()
