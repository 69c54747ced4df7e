"""The BASELINE.json workloads as data (seeded synthetic inputs).

Shared by bench.py and the full-size parity tests so both exercise exactly
the same meshes, orders and inputs.  Seeds follow SURVEY §8(d): SPECHP_SEED
(default 20240801, test_acceptance.py:50) with numpy's default_rng.
"""
from __future__ import annotations

import os

import numpy as np

SEED = int(os.environ.get("SPECHP_SEED", "20240801"))

# cfg1: 32x32 affine quads, P=4, Q=6 (BwdTrans + IProductWRTBase)
CFG1 = dict(shape="quad", n=32, P=4, Q=6, mapping="affine", amp=0.0)
# cfg2: 256x256 curved quads x'=x+0.05 sin2πy, y'=y+0.05 sin2πx, P=6, Q=8
CFG2 = dict(shape="quad", n=256, P=6, Q=8, mapping="quad_sine", amp=0.05)
# cfg3: 64^3 affine hexes, P=4, Q=6 (BwdTrans, IProductWRTBase, PhysDeriv)
CFG3 = dict(shape="hex", n=64, P=4, Q=6, mapping="affine", amp=0.0)
# cfg4: 64^3 deformed periodic hexes x'=x+0.03 sin2πy sin2πz, P=2..8, Q=P+2
CFG4 = dict(shape="hex", n=64, orders=tuple(range(2, 9)), mapping="hex_sine", amp=0.03)
# cfg5: 48^3, per-element P iid uniform in {3..7} (derived seed), Q=P+2
CFG5 = dict(shape="hex", n=48, lo=3, hi=7, mapping="hex_sine", amp=0.03)


def cfg5_orders(seed: int = SEED, n: int = CFG5["n"]):
    """Per-element orders of cfg5 (element id ex + n (ey + n ez))."""
    return np.random.default_rng(seed + 5).integers(CFG5["lo"], CFG5["hi"] + 1, n ** 3)
