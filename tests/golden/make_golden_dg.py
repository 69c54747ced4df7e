"""Generate the DG golden fixtures from the reference implementation.

Run in the build container, where the (pure-Python) reference is importable:

    python tests/golden/make_golden_dg.py

Writes tests/golden/reference_dg.npz.  For each case it stores the arrays a
reference `DGSystem` precomputes (solvers.py:195-341: ww, inv, minv, the
interior / periodic trace arrays and the boundary groups) — the input
contract of `paper_1906_03489_b200.dg.DGOperators` — and the outputs of the
reference's own primitives and right-hand sides on seeded inputs:

  walls     structured_quad_mesh(3,3), P=4, rigid walls; every DGSystem
            primitive (bwd, iproduct, iproduct_deriv, mass_solve,
            trace_minus/plus, lift_interior, lift_boundary) and ape_rhs with a
            non-uniform base flow (pointwise c2 branch), upwind and
            Lax-Friedrichs
  periodic  structured_quad_mesh(4,4), P=5, periodic box; ape_rhs with a
            uniform base flow (element-constant c2 branch) and a pressure
            source; AdvectionOperator.rhs
  mixed     structured_quad_mesh(5,2), P=3; periodic west/east, far field
            south, Dirichlet north; ape_rhs (upwind) and AdvectionOperator.rhs
            with Dirichlet / far-field boundaries
Expressions are plain numpy callables (the reference calls them with
x=, y=, t= keywords); the tests re-create the same callables.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]

from spechp.meshio import structured_quad_mesh  # noqa: E402
from spechp.region import build_elements  # noqa: E402
from spechp.solvers import (AdvectionOperator, DGSystem, ape_rhs,  # noqa: E402
                            make_ape_state)

sys.path.insert(0, str(ROOT / "tests"))
from dg_cases import CASES  # noqa: E402

SEED = 20240801
out = {}


def dump_system(tag, system):
    out[f"{tag}/P"] = np.int64(system.exp.basis_keys[0].num_modes - 1)
    out[f"{tag}/Q"] = np.int64(system.exp.basis_keys[0].points_key.num_points)
    for k in ("ww", "inv", "minv", "xy"):
        out[f"{tag}/{k}"] = np.asarray(getattr(system, k))
    out[f"{tag}/int_li"] = np.asarray(system.int_li, dtype=np.int64)
    out[f"{tag}/int_ri"] = np.asarray(system.int_ri, dtype=np.int64)
    if system.num_interior:
        for k in ("exm", "lm", "exp", "lp", "warc", "nrm", "xy"):
            out[f"{tag}/int_{k}"] = np.asarray(getattr(system, f"int_{k}"))
    names = list(system.bnd)
    out[f"{tag}/bnd_names"] = np.array(names if names else [""])
    for name, grp in system.bnd.items():
        for k in ("li", "exm", "lm", "nrm", "warc", "xy"):
            out[f"{tag}/bnd/{name}/{k}"] = np.asarray(grp[k])


for tag, case in CASES.items():
    mesh = structured_quad_mesh(*case["mesh"])
    elements = build_elements(mesh, orders=case["P"])
    system = DGSystem(mesh, elements, case["bcs"], strategy="sumfac")
    dump_system(tag, system)
    rng = np.random.default_rng(SEED + len(tag))
    E, nm = len(elements), elements[0].num_modes
    npts = system.ww.shape[1]
    if case.get("primitives"):
        c = rng.uniform(-1, 1, (E, nm))
        ph = rng.uniform(-1, 1, (E, npts))
        fx, fy = rng.uniform(-1, 1, (2, E, npts))
        b = rng.uniform(-1, 1, (E, nm))
        out[f"{tag}/in/coeffs"] = c
        out[f"{tag}/in/phys"] = ph
        out[f"{tag}/in/fx"] = fx
        out[f"{tag}/in/fy"] = fy
        out[f"{tag}/in/b"] = b
        out[f"{tag}/out/bwd"] = system.bwd(c)
        out[f"{tag}/out/iproduct"] = system.iproduct(ph)
        out[f"{tag}/out/iproduct_deriv"] = system.iproduct_deriv(fx, fy)
        out[f"{tag}/out/mass_solve"] = system.mass_solve(b)
        if system.num_interior:
            out[f"{tag}/out/trace_minus"] = system.trace_minus(ph)
            out[f"{tag}/out/trace_plus"] = system.trace_plus(ph)
            s = rng.uniform(-1, 1, system.int_warc.shape)
            out[f"{tag}/in/s_int"] = s
            bb = b.copy()
            system.lift_interior(bb, s)
            out[f"{tag}/out/lift_interior"] = bb
        for name, grp in system.bnd.items():
            s = rng.uniform(-1, 1, grp["warc"].shape)
            out[f"{tag}/in/s_bnd/{name}"] = s
            bb = b.copy()
            system.lift_boundary(bb, name, s)
            out[f"{tag}/out/lift_boundary/{name}"] = bb
    for k, ape in enumerate(case.get("ape", [])):
        state = make_ape_state(system, ape["base"], initial=ape["initial"],
                               sources=ape.get("sources"), riemann=ape["riemann"])
        coeffs = state.coeffs + 0.1 * rng.standard_normal(state.coeffs.shape)
        t = ape.get("t", 0.0)
        out[f"{tag}/ape{k}/coeffs"] = coeffs
        out[f"{tag}/ape{k}/c2_constant"] = np.int64(state.c2_elementwise_constant)
        out[f"{tag}/ape{k}/rhs"] = ape_rhs(state, coeffs, t)
    for k, adv in enumerate(case.get("advection", [])):
        op = AdvectionOperator(system, adv["velocity"], adv.get("bcs"))
        coeffs = rng.uniform(-1, 1, (E, nm))
        t = adv.get("t", 0.0)
        out[f"{tag}/adv{k}/coeffs"] = coeffs
        out[f"{tag}/adv{k}/rhs"] = op.rhs(coeffs, t)

path = ROOT / "tests" / "golden" / "reference_dg.npz"
np.savez_compressed(path, **out)
print(f"wrote {path} ({path.stat().st_size / 1e3:.0f} KB, {len(out)} arrays)")
