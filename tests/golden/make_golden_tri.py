"""Reference outputs for the triangle collections.

    python tests/golden/make_golden_tri.py  ->  tests/golden/reference_tri.npz

For P = 1..6 (default points: GLL m1+1 x Gauss-Radau m2+1, stdregions.py:
402-408) the reference's own Collection (SUM_FAC) is applied to seeded
blocks: standard elements (BwdTrans, IProductWRTBase, PhysDeriv) and
elements carrying injected affine GeomFactors (one random map with positive
determinant per element; IProductWRTBase, PhysDeriv), plus
iproduct_wrt_deriv_base_world (geometry.py:163-168) per element.  The
tables (bwd_matrix, weights, deriv_matrices) are stored too.
"""
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from spechp.collections import Collection, OperatorKind, Strategy  # noqa: E402
from spechp.geometry import GeomFactors, iproduct_wrt_deriv_base_world  # noqa: E402
from spechp.stdregions import make_tri  # noqa: E402

SEED = 20240801
out = {}
for P in range(1, 7):
    exp = make_tri(P)
    rng = np.random.default_rng(SEED + P)
    E = 7
    nm, npts = exp.num_modes, exp.num_points
    pre = f"P{P}/"
    out[pre + "B"] = exp.bwd_matrix
    out[pre + "w"] = exp.weights
    out[pre + "D0"], out[pre + "D1"] = exp.deriv_matrices
    c = rng.uniform(-1, 1, (E, nm))
    u = rng.uniform(-1, 1, (E, npts))
    f = rng.uniform(-1, 1, (E, 2, npts))
    out[pre + "coeffs"], out[pre + "phys"], out[pre + "flux"] = c, u, f
    std = [exp] * E
    out[pre + "std/bwd"] = Collection(std, OperatorKind.BWD_TRANS, Strategy.SUM_FAC).apply(c)
    out[pre + "std/iprod"] = Collection(std, OperatorKind.IPRODUCT_WRT_BASE, Strategy.SUM_FAC).apply(u)
    out[pre + "std/deriv"] = Collection(std, OperatorKind.PHYS_DERIV, Strategy.SUM_FAC).apply(u)
    els, wjs, invs = [], [], []
    for e in range(E):
        while True:
            J = np.array([[0.3, 0.0], [0.0, 0.3]]) + 0.1 * rng.standard_normal((2, 2))
            if np.linalg.det(J) > 0.02:
                break
        jac = np.broadcast_to(J, (npts, 2, 2)).copy()   # jac[i, k, a] = dx_k / dxi_a
        det = np.full(npts, np.linalg.det(J))
        inv = np.broadcast_to(np.linalg.inv(J), (npts, 2, 2)).copy()
        gf = GeomFactors(jac, det, inv, exp.weights * det)
        els.append(SimpleNamespace(exp=exp, gf=gf))
        wjs.append(gf.weights_world)
        invs.append(gf.inv)
    out[pre + "wj"] = np.stack(wjs)
    out[pre + "inv"] = np.stack(invs)
    out[pre + "phys/iprod"] = Collection(els, OperatorKind.IPRODUCT_WRT_BASE, Strategy.SUM_FAC).apply(u)
    out[pre + "phys/deriv"] = Collection(els, OperatorKind.PHYS_DERIV, Strategy.SUM_FAC).apply(u)
    out[pre + "phys/ipderiv"] = np.stack([iproduct_wrt_deriv_base_world(exp, el.gf, f[e, 0], f[e, 1])
                                          for e, el in enumerate(els)])

path = Path(__file__).resolve().parent / "reference_tri.npz"
np.savez_compressed(path, **out)
print(f"wrote {path} ({path.stat().st_size / 1024:.0f} KB, {len(out)} arrays)")
