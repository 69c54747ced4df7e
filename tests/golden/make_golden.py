"""Generate golden fixtures from the reference implementation.

Run in the build container, where the (pure-Python) reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/reference_golden.npz (small: a few hundred KB).  The GPU
box has no /root/reference; the tests read only the committed fixture.

Contents (keys), each produced by the reference's own public functions:
  tables      quadrature.make_rule + diff_matrix (GL/GLL/Radau), basis
              eval_modified_A + boundary_first_permutation
  cfg1        structured_quad_mesh(4,4), build_elements(P=4, Q=6):
              GeomFactors and Collection(SUM_FAC) outputs for BwdTrans,
              IProductWRTBase, PhysDeriv on seeded blocks
  std         standard-element collections (make_quad(P), P = 2, 5, 8)
  cfg2        curved quads (analytic map injected as GeomFactors, the way
              SURVEY §8(c) prescribes): PhysDeriv and the dense world
              Helmholtz (world_stiffness_matrix + lam*world_mass_matrix)
  amap        build_assembly_map on structured meshes with variable order
              and Dirichlet boundaries, + GlobalSystem.apply (matrix-free)
  listing1    Listing-1 integral of cos(x)cos(y), P=7, Q=9 (4 sin^2 1)
"""
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from spechp.assembly import build_assembly_map, build_global_system  # noqa: E402
from spechp.basis import boundary_first_permutation, eval_modified_A  # noqa: E402
from spechp.collections import Collection, OperatorKind, Strategy  # noqa: E402
from spechp.geometry import (GeomFactors, world_mass_matrix,  # noqa: E402
                             world_stiffness_matrix)
from spechp.meshio import structured_quad_mesh  # noqa: E402
from spechp.quadrature import PointsKey, PointsType, diff_matrix, make_rule  # noqa: E402
from spechp.region import build_elements  # noqa: E402
from spechp.stdregions import integral, make_quad  # noqa: E402

SEED = 20240801
out = {}

# --- 1D tables ---------------------------------------------------------------
for name, pt, qs in (("gll", PointsType.GAUSS_LOBATTO_LEGENDRE, range(2, 14)),
                     ("gl", PointsType.GAUSS_LEGENDRE, range(1, 13)),
                     ("radau", PointsType.GAUSS_RADAU_M_LEGENDRE, range(1, 13))):
    for q in qs:
        r = make_rule(PointsKey(q, pt))
        out[f"tables/{name}/{q}/z"] = np.asarray(r.points)
        out[f"tables/{name}/{q}/w"] = np.asarray(r.weights)
        out[f"tables/{name}/{q}/D"] = diff_matrix(r)
for P in range(1, 11):
    for q in (P + 1, P + 2, P + 3):
        z = make_rule(PointsKey(q, PointsType.GAUSS_LOBATTO_LEGENDRE)).points
        t = eval_modified_A(P, z)
        perm = boundary_first_permutation(P)
        out[f"tables/moda/{P}/{q}/B"] = t.values[perm]
        out[f"tables/moda/{P}/{q}/Bd"] = t.derivs[perm]

rng = np.random.default_rng(SEED)

# --- cfg1: 4x4 affine quads, P=4, Q=6 ------------------------------------------
mesh = structured_quad_mesh(4, 4)
els = build_elements(mesh, orders=4, num_points=6)
E = len(els)
out["cfg1/wts"] = np.stack([e.gf.weights_world for e in els])
out["cfg1/inv"] = np.stack([e.gf.inv for e in els])
c = rng.uniform(-1, 1, (E, els[0].exp.num_modes))
u = rng.uniform(-1, 1, (E, els[0].exp.num_points))
out["cfg1/coeffs"] = c
out["cfg1/phys"] = u
out["cfg1/bwd"] = Collection(els, OperatorKind.BWD_TRANS, Strategy.SUM_FAC).apply(c)
out["cfg1/iprod"] = Collection(els, OperatorKind.IPRODUCT_WRT_BASE, Strategy.SUM_FAC).apply(u)
out["cfg1/deriv"] = Collection(els, OperatorKind.PHYS_DERIV, Strategy.SUM_FAC).apply(u)
out["cfg1/helm"] = np.stack([(world_stiffness_matrix(e.exp, e.gf) + 1.0 * world_mass_matrix(e.exp, e.gf)) @ c[k]
                             for k, e in enumerate(els)])

# --- standard elements, default quadrature (Q = P+2 points) ------------------------
for P in (2, 5, 8):
    exps = [make_quad(P)] * 7
    cb = rng.standard_normal((7, exps[0].num_modes))
    ub = rng.standard_normal((7, exps[0].num_points))
    out[f"std/{P}/coeffs"] = cb
    out[f"std/{P}/phys"] = ub
    out[f"std/{P}/bwd"] = Collection(exps, OperatorKind.BWD_TRANS, Strategy.STD_MAT).apply(cb)
    out[f"std/{P}/iprod"] = Collection(exps, OperatorKind.IPRODUCT_WRT_BASE, Strategy.STD_MAT).apply(ub)
    out[f"std/{P}/deriv"] = Collection(exps, OperatorKind.PHYS_DERIV, Strategy.STD_MAT).apply(ub)

# --- cfg2 sample: curved quads, analytic map injected ------------------------------
from oracle import geometry as og  # noqa: E402  (analytic factors; operators by the reference)
from oracle import ops as oo  # noqa: E402

n2, P2 = 4, 6
exp2 = make_quad(P2, num_points=P2 + 2)
oe = oo.Expansion("quad", P2, P2 + 2)
jac, det, inv, wj = og.factors(oe, n2, np.arange(n2 * n2), og.MAP_QUAD_SINE, 0.05)
els2 = [SimpleNamespace(exp=exp2, gf=GeomFactors(jac[e], det[e], inv[e], wj[e])) for e in range(n2 * n2)]
c2 = rng.uniform(-1, 1, (n2 * n2, exp2.num_modes))
u2 = rng.uniform(-1, 1, (n2 * n2, exp2.num_points))
out["cfg2/inv"] = inv
out["cfg2/wts"] = wj
out["cfg2/coeffs"] = c2
out["cfg2/phys"] = u2
out["cfg2/deriv"] = Collection(els2, OperatorKind.PHYS_DERIV, Strategy.SUM_FAC).apply(u2)
out["cfg2/iprod"] = Collection(els2, OperatorKind.IPRODUCT_WRT_BASE, Strategy.SUM_FAC).apply(u2)
out["cfg2/helm"] = np.stack([(world_stiffness_matrix(exp2, g.gf) + 1.0 * world_mass_matrix(exp2, g.gf)) @ c2[k]
                             for k, g in enumerate(els2)])

# --- assembly maps + GlobalSystem.apply ---------------------------------------------
for tag, (nx, ny, dn, seed) in {"a": (4, 3, (), 1), "b": (5, 4, ("south", "west"), 2),
                                "c": (6, 6, ("north", "east", "south", "west"), 3)}.items():
    r2 = np.random.default_rng(seed)
    orders = r2.integers(2, 7, nx * ny)
    mesh = structured_quad_mesh(nx, ny)
    els3 = build_elements(mesh, orders={e: int(orders[e]) for e in range(nx * ny)})
    am = build_assembly_map(mesh, els3, dn)
    out[f"amap/{tag}/shape"] = np.array([nx, ny])
    out[f"amap/{tag}/orders"] = orders
    out[f"amap/{tag}/dirichlet"] = np.array(list(dn) or [""])
    out[f"amap/{tag}/num_global"] = np.array(am.num_global)
    out[f"amap/{tag}/num_dirichlet"] = np.array(am.num_dirichlet)
    out[f"amap/{tag}/l2g"] = np.concatenate(am.local_to_global)
    out[f"amap/{tag}/signs"] = np.concatenate(am.signs)
    sysm = build_global_system(els3, am, "helmholtz", 1.0, matrix_free_threshold=0)
    x = r2.uniform(-1, 1, am.num_global)
    out[f"amap/{tag}/x"] = x
    out[f"amap/{tag}/y"] = sysm.apply(x)
    out[f"amap/{tag}/diag"] = sysm.diag
    out[f"amap/{tag}/wts"] = np.concatenate([e.gf.weights_world for e in els3])
    out[f"amap/{tag}/inv"] = np.concatenate([e.gf.inv.reshape(-1) for e in els3])

# --- Helmholtz spectral convergence (test_acceptance.py:93-125), reference solve ---
from spechp.assembly import helmholtz_solve  # noqa: E402
from spechp.geometry import integral_world, x_map  # noqa: E402
from spechp.stdregions import bwd_trans  # noqa: E402

errs, iters = [], []
for P in range(2, 9):
    mesh = structured_quad_mesh(4, 4)
    els4 = build_elements(mesh, orders=P)
    exact = lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y)
    forcing = []
    for el in els4:
        xy = x_map(el.geom, el.exp.points)
        forcing.append((2 * np.pi ** 2 + 1.0) * exact(xy[:, 0], xy[:, 1]))
    dirichlet = {nm: (lambda x, y: 0.0) for nm in ("south", "east", "north", "west")}
    coeffs, info = helmholtz_solve(mesh, els4, 1.0, forcing, dirichlet, tol=1e-13, max_iter=6000)
    num = den = 0.0
    for el, c in zip(els4, coeffs):
        xy = x_map(el.geom, el.exp.points)
        diff = bwd_trans(el.exp, c) - exact(xy[:, 0], xy[:, 1])
        num += integral_world(el.exp, el.gf, diff ** 2)
        den += integral_world(el.exp, el.gf, exact(xy[:, 0], xy[:, 1]) ** 2)
    errs.append(np.sqrt(num / den))
out["helm_conv/errors"] = np.array(errs)

# --- Listing 1 ---------------------------------------------------------------------------
q7 = make_quad(7, num_points=9)
xy = q7.points
out["listing1/integral"] = np.array(integral(q7, np.cos(xy[:, 0]) * np.cos(xy[:, 1])))

path = Path(__file__).resolve().parent / "reference_golden.npz"
np.savez_compressed(path, **out)
print(f"wrote {path} ({path.stat().st_size / 1024:.0f} KB, {len(out)} arrays)")
