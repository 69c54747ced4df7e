"""Host-side checks of the DG device layer (no GPU): the lift CSR built by
dg._csr reproduces the reference's np.add.at accumulation on the golden
fixtures when applied on the CPU, and the fixtures are self-consistent."""
import numpy as np
import pytest

from dg_cases import CASES
from dg_fixture import G, system
from paper_1906_03489_b200 import dg as D
from paper_1906_03489_b200 import make_quad


def cpu_lift(E, rowp, codes, Lm, Lp, w, s, b):
    """Sequential reference semantics of sphp_trace_lift."""
    out = b.copy()
    for e in range(E):
        for c in codes[rowp[e]:rowp[e + 1]]:
            t, plus, neg = c >> 2, (c >> 1) & 1, c & 1
            L = (Lp if plus else Lm)[t]
            v = L @ (w[t] * s[t] if w is not None else s[t])
            out[e] = out[e] - v if neg else out[e] + v
    return out


@pytest.mark.parametrize("tag", sorted(CASES))
def test_lift_csr_matches_reference_add_at(tag):
    ns = system(tag, make_quad)
    E = ns.ww.shape[0]
    b = G[f"{tag}/in/b"]
    if ns.int_li.size:
        rowp, codes = D._csr(E, [(ns.int_li, 0, 0, 1), (ns.int_ri, 0, 1, 0)])
        got = cpu_lift(E, rowp, codes, ns.int_lm, ns.int_lp, ns.int_warc, G[f"{tag}/in/s_int"], b)
        ref = G[f"{tag}/out/lift_interior"]
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    for name, g in ns.bnd.items():
        rowp, codes = D._csr(E, [(g["li"], 0, 0, 1)])
        got = cpu_lift(E, rowp, codes, g["lm"], g["lm"], g["warc"], G[f"{tag}/in/s_bnd/{name}"], b)
        ref = G[f"{tag}/out/lift_boundary/{name}"]
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_csr_orders_groups_then_traces():
    rowp, codes = D._csr(3, [(np.array([2, 0, 2]), 0, 0, 1), (np.array([0, 2]), 10, 1, 0)])
    assert rowp.tolist() == [0, 2, 2, 5]
    assert (codes[:2] >> 2).tolist() == [1, 10]            # element 0: group 0 then group 1
    assert (codes[2:] >> 2).tolist() == [0, 2, 11]         # element 2
    assert (codes[2:] & 3).tolist() == [1, 1, 2]


def test_fixture_cases_cover_every_bc_kind():
    kinds = {spec["type"] for c in CASES.values() for spec in c["bcs"].values()}
    assert kinds == {"rigid_wall", "periodic", "farfield", "dirichlet"}
    assert {a["riemann"] for c in CASES.values() for a in c.get("ape", [])} == {"upwind", "laxfriedrichs"}
    assert any(int(G[f"{t}/ape{k}/c2_constant"]) for t, c in CASES.items() for k in range(len(c.get("ape", []))))
    assert not all(int(G[f"{t}/ape{k}/c2_constant"]) for t, c in CASES.items() for k in range(len(c.get("ape", []))))
