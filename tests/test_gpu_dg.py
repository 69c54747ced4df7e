"""GPU parity of the DG layer (dg.py / csrc/dg.cu) against the reference's
own DGSystem primitives, ape_rhs and AdvectionOperator.rhs on the committed
fixtures (tests/golden/make_golden_dg.py): every primitive, both Riemann
fluxes, all four boundary kinds, both c2 branches, sources and
time-dependent Dirichlet data.  Tolerance: max-abs normalised by the
output's max-abs < 1e-12; repeated calls bitwise equal."""
import numpy as np
import pytest
import torch

from dg_cases import CASES
from dg_fixture import G, ape_state, system

pytestmark = pytest.mark.gpu

TOL = 1e-12


def close(got, ref):
    got = got.detach().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape
    scale = max(np.max(np.abs(ref)), 1e-300)
    err = np.max(np.abs(got - ref)) / scale
    assert err < TOL, err


@pytest.fixture(scope="module")
def sp():
    import paper_1906_03489_b200 as sp
    return sp


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


@pytest.mark.parametrize("tag", sorted(CASES))
def test_dg_primitives(sp, tag):
    from paper_1906_03489_b200.dg import DGOperators
    ns = system(tag, sp.make_quad)
    d = DGOperators(ns)
    close(d.bwd(dev(G[f"{tag}/in/coeffs"])), G[f"{tag}/out/bwd"])
    close(d.iproduct(dev(G[f"{tag}/in/phys"])), G[f"{tag}/out/iproduct"])
    close(d.iproduct_deriv(dev(G[f"{tag}/in/fx"]), dev(G[f"{tag}/in/fy"])), G[f"{tag}/out/iproduct_deriv"])
    close(d.mass_solve(dev(G[f"{tag}/in/b"])), G[f"{tag}/out/mass_solve"])
    ph = dev(G[f"{tag}/in/phys"])
    if d.num_interior:
        close(d.trace_minus(ph), G[f"{tag}/out/trace_minus"])
        close(d.trace_plus(ph), G[f"{tag}/out/trace_plus"])
        b = dev(G[f"{tag}/in/b"])
        d.lift_interior(b, dev(G[f"{tag}/in/s_int"]))
        close(b, G[f"{tag}/out/lift_interior"])
    for name in d.bnd:
        b = dev(G[f"{tag}/in/b"])
        d.lift_boundary(b, name, dev(G[f"{tag}/in/s_bnd/{name}"]))
        close(b, G[f"{tag}/out/lift_boundary/{name}"])


@pytest.mark.parametrize("tag,k", [(t, k) for t, c in sorted(CASES.items())
                                   for k in range(len(c.get("ape", [])))])
def test_ape_rhs(sp, tag, k):
    from paper_1906_03489_b200.dg import ApeOperator, DGOperators
    ns = system(tag, sp.make_quad)
    st = ape_state(tag, k, ns)
    op = ApeOperator(DGOperators(ns), st["base"], st["base_trace"], st["base_bnd"], ns.bcs,
                     st["riemann"], st["sources"], st["c2_per_element"])
    c = dev(G[f"{tag}/ape{k}/coeffs"])
    r1 = op.rhs(c, st["t"])
    close(r1, G[f"{tag}/ape{k}/rhs"])
    r2 = op.rhs(c, st["t"])
    assert torch.equal(r1, r2)


@pytest.mark.parametrize("tag,k", [(t, k) for t, c in sorted(CASES.items())
                                   for k in range(len(c.get("advection", [])))])
def test_advection_rhs(sp, tag, k):
    from paper_1906_03489_b200.dg import AdvectionOperator, DGOperators
    ns = system(tag, sp.make_quad)
    adv = CASES[tag]["advection"][k]
    op = AdvectionOperator(DGOperators(ns), adv["velocity"], adv.get("bcs"))
    r = op.rhs(dev(G[f"{tag}/adv{k}/coeffs"]), adv.get("t", 0.0))
    close(r, G[f"{tag}/adv{k}/rhs"])


def test_dg_rejects_bad_kinds(sp):
    from paper_1906_03489_b200.dg import ApeOperator, DGOperators, SolverError
    ns = system("walls", sp.make_quad)
    st = ape_state("walls", 0, ns)
    d = DGOperators(ns)
    with pytest.raises(SolverError, match="Riemann"):
        ApeOperator(d, st["base"], st["base_trace"], st["base_bnd"], ns.bcs, "roe")
    bad = dict(ns.bcs, south={"type": "periodic_typo"})
    with pytest.raises(SolverError, match="unsupported"):
        ApeOperator(d, st["base"], st["base_trace"], st["base_bnd"], bad, "upwind")
