"""GPU against the reference's own outputs (tests/golden/reference_golden.npz,
produced by /root/reference through make_golden.py): the drop-in path —
element objects carrying reference-layout GeomFactors, the reference's
AssemblyMap codes — must reproduce Collection.apply / world Helmholtz /
GlobalSystem.apply to 1e-12."""
from pathlib import Path
from types import SimpleNamespace as NS

import numpy as np
import pytest

from helpers import assert_parity

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
G = np.load(Path(__file__).resolve().parent / "golden" / "reference_golden.npz")


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1906_03489_b200 as sp

    return sp


def _elements(sp, exp, wts, inv):
    return [NS(exp=exp, gf=sp.GeomFactors(None, None, inv[e], wts[e])) for e in range(len(wts))]


@pytest.mark.parametrize("strategy", ["cuda_sumfac", "cuda_stdmat"])
def test_cfg1_reference_outputs(sp, strategy):
    exp = sp.make_quad(4, 6)
    els = _elements(sp, exp, G["cfg1/wts"], G["cfg1/inv"])
    st = sp.Strategy(strategy)
    for op, inp, ref in (("bwdtrans", "cfg1/coeffs", "cfg1/bwd"),
                         ("iproductwrtbase", "cfg1/phys", "cfg1/iprod"),
                         ("physderiv", "cfg1/phys", "cfg1/deriv"),
                         ("helmholtz", "cfg1/coeffs", "cfg1/helm")):
        coll = sp.Collection(els, sp.OperatorKind(op), st, lam=1.0)
        got = coll.apply(G[inp])          # numpy in -> numpy out (host path)
        assert got.shape == G[ref].shape
        assert_parity(got, G[ref], what=f"cfg1 {op} {strategy}")


@pytest.mark.parametrize("P", [2, 5, 8])
def test_standard_elements_reference_outputs(sp, P):
    exp = sp.make_quad(P)                 # reference default quadrature Q = P + 2
    exps = [exp] * 7
    for op, inp, ref in (("bwdtrans", "coeffs", "bwd"), ("iproductwrtbase", "phys", "iprod"),
                         ("physderiv", "phys", "deriv")):
        coll = sp.Collection(exps, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
        got = coll.apply(G[f"std/{P}/{inp}"])
        assert_parity(got, G[f"std/{P}/{ref}"], what=f"std P{P} {op}")


def test_cfg2_curved_reference_outputs(sp):
    exp = sp.make_quad(6, 8)
    els = _elements(sp, exp, G["cfg2/wts"], G["cfg2/inv"])
    for op, inp, ref in (("physderiv", "cfg2/phys", "cfg2/deriv"),
                         ("iproductwrtbase", "cfg2/phys", "cfg2/iprod"),
                         ("helmholtz", "cfg2/coeffs", "cfg2/helm")):
        coll = sp.Collection(els, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC, lam=1.0)
        assert_parity(coll.apply(G[inp]), G[ref], what=f"cfg2 {op}")
    # the analytic device geometry reproduces the injected reference factors
    batch = sp.ElementBatch.structured(exp, 4, kind=sp.GEOM_POINT, mapping=sp.MAP_QUAD_SINE, amp=0.05)
    coll = sp.Collection(batch, sp.OperatorKind.PHYS_DERIV, sp.Strategy.CUDA_SUMFAC)
    got = coll.apply(torch.as_tensor(G["cfg2/phys"], device="cuda")).cpu().numpy()
    assert_parity(got, G["cfg2/deriv"], what="cfg2 analytic geometry")


@pytest.mark.parametrize("alg", ["owner", "colour"])
@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_global_system_apply_reference(sp, tag, alg):
    """GlobalSystem.apply on variable-order meshes with Dirichlet blocks and
    pinned modes, from the reference's AssemblyMap and GeomFactors."""
    nx, ny = (int(v) for v in G[f"amap/{tag}/shape"])
    orders = G[f"amap/{tag}/orders"]
    l2g, sgn = G[f"amap/{tag}/l2g"], G[f"amap/{tag}/signs"]
    wts_all, inv_all = G[f"amap/{tag}/wts"], G[f"amap/{tag}/inv"]
    ng = int(G[f"amap/{tag}/num_global"])
    nmodes = (orders + 1) ** 2
    npts = (orders + 2) ** 2
    mo = np.concatenate([[0], np.cumsum(nmodes)])
    po = np.concatenate([[0], np.cumsum(npts)])
    batches = []
    for P in sorted(set(orders.tolist())):
        ids = np.nonzero(orders == P)[0]
        exp = sp.make_quad(int(P))
        els = [NS(exp=exp, gf=sp.GeomFactors(None, None,
                                              inv_all[4 * po[e]:4 * po[e + 1]].reshape(-1, 2, 2),
                                              wts_all[po[e]:po[e + 1]])) for e in ids]
        coll = sp.Collection(els, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC, lam=1.0)
        amap = sp.AssemblyMap.from_reference(NS(local_to_global=[l2g[mo[e]:mo[e + 1]] for e in ids],
                                                signs=[sgn[mo[e]:mo[e + 1]] for e in ids],
                                                num_global=ng)).set_algorithm(alg)
        batches.append((coll, amap))
    y = sp.GlobalHelmholtz(batches, ng).apply(torch.as_tensor(G[f"amap/{tag}/x"], device="cuda"))
    assert_parity(y.cpu().numpy(), G[f"amap/{tag}/y"], what=f"GlobalSystem.apply {tag} {alg}")


def test_autotune_report_shape(sp):
    """collections.py:285-313 report: {strategy: {median_s, times_s, mac_count}}."""
    exp = sp.make_quad(4, 6)
    batch = sp.ElementBatch.structured(exp, 16, kind=sp.GEOM_AFFINE)
    strat, rep = sp.autotune(batch, sp.OperatorKind.BWD_TRANS, trials=3, warmups=1)
    assert strat in sp.CONCRETE_STRATEGIES
    assert set(rep) == {"cuda_sumfac", "cuda_stdmat"}
    for v in rep.values():
        assert len(v["times_s"]) == 3 and v["median_s"] > 0 and v["mac_count"] > 0
        # the SURVEY §5 extension of the report: rates consistent with the median
        assert v["dof_per_s"] == pytest.approx(16 * 16 * 25 / v["median_s"])
        assert v["hbm_gbs_achieved"] == pytest.approx(v["hbm_bytes"] / v["median_s"] / 1e9)
        assert v["roofline_frac"] == pytest.approx(v["hbm_gbs_achieved"] / sp.collections.hbm_peak_gbs()[0])
    only, rep1 = sp.autotune(batch, sp.OperatorKind.BWD_TRANS, trials=2, warmups=0,
                             candidates=[sp.Strategy.CUDA_STDMAT])
    assert only is sp.Strategy.CUDA_STDMAT and list(rep1) == ["cuda_stdmat"]
    with pytest.raises(sp.CollectionError):
        sp.autotune(batch, sp.OperatorKind.BWD_TRANS, trials=0)
    coll = sp.create_collection(batch, sp.OperatorKind.BWD_TRANS, sp.Strategy.AUTO, trials=2,
                                warmups=1)
    assert coll.strategy in sp.CONCRETE_STRATEGIES


def test_mac_counts_favor_sumfac_at_high_order(sp):
    """test_collections.py:176-190 on the GPU collections."""
    for P, shape in ((8, "quad"), (6, "hex")):
        exp = sp.make_quad(P, P + 2) if shape == "quad" else sp.make_hex(P, P + 2)
        b = sp.ElementBatch.standard(exp, 256)
        sf = sp.Collection(b, sp.OperatorKind.BWD_TRANS, sp.Strategy.CUDA_SUMFAC).mac_count()
        sm = sp.Collection(b, sp.OperatorKind.BWD_TRANS, sp.Strategy.CUDA_STDMAT).mac_count()
        assert sf < sm


def test_specpy_listing1_and_hex(sp):
    """NekPy-style names (specpy/__init__.py:31-106) over the GPU path, plus
    StdHexExp: Listing-1 integral and BwdTrans/PhysDeriv against the oracle."""
    import math

    from paper_1906_03489_b200 import specpy as nek
    from oracle import ops as oo

    pKey = nek.PointsKey(9, nek.PointsType.GaussLobattoLegendre)
    bKey = nek.BasisKey(nek.BasisType.Modified_A, 8, pKey)
    quad = nek.StdQuadExp(bKey, bKey)
    x, y = quad.GetCoords()
    assert abs(quad.Integral(np.cos(x) * np.cos(y)) - 4 * math.sin(1.0) ** 2) < 1e-8
    with pytest.raises(ValueError, match="expected array of length 64"):
        quad.BwdTrans(np.zeros(63))
    hk = nek.BasisKey(nek.BasisType.Modified_A, 5, nek.PointsKey(6, nek.PointsType.GaussLobattoLegendre))
    hexe = nek.StdHexExp(hk, hk, hk)
    c = np.random.default_rng(3).standard_normal(hexe.GetNcoeffs())
    oe = oo.Expansion("hex", 4, 6)
    assert_parity(hexe.BwdTrans(c), oo.bwd(oe, c[None])[0], what="StdHexExp.BwdTrans")
    u = oo.bwd(oe, c[None])[0]
    d = hexe.PhysDeriv(u)
    ref = oo.ref_deriv(oe, u[None])[0]
    for a in range(3):
        assert_parity(d[a], ref[a], what=f"StdHexExp.PhysDeriv[{a}]")
    assert_parity(hexe.IProductWRTBase(u), oo.iprod(oe, u[None], oe.weights)[0],
                  what="StdHexExp.IProductWRTBase")
