"""Triangle collections against the reference's own
outputs (tests/golden/make_golden_tri.py): host tables on CPU, the CUDA
sum-factorisation and StdMat strategies on the GPU, for standard elements
and elements with affine / per-point geometry, P = 1..6."""
from pathlib import Path

import numpy as np
import pytest

import paper_1906_03489_b200 as sp

G = np.load(Path(__file__).resolve().parent / "golden" / "reference_tri.npz")
PS = range(1, 7)
TOL = 1e-12


def close(got, want, tol=TOL):
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert err < tol, err


@pytest.mark.parametrize("P", PS)
def test_tri_tables_match_reference(P):
    exp = sp.make_tri(P)
    assert exp.num_modes == G[f"P{P}/B"].shape[0]
    close(exp.bwd_matrix, G[f"P{P}/B"], 1e-14)
    close(exp.weights, G[f"P{P}/w"], 1e-14)
    for a in range(2):
        close(exp.deriv_matrices[a], G[f"P{P}/D{a}"], 1e-13)
    # the golden std outputs are the dense operators applied to the inputs
    close(G[f"P{P}/coeffs"] @ G[f"P{P}/B"], G[f"P{P}/std/bwd"])


def test_tri_key_validation():
    from paper_1906_03489_b200.basis import BasisKey, BasisType
    from paper_1906_03489_b200.quadrature import PointsKey, PointsType
    pk = PointsKey(5, PointsType.GAUSS_LOBATTO_LEGENDRE)
    with pytest.raises(sp.ExpansionError, match="collapsed-direction"):
        sp.StdExpansion(sp.Shape.TRI, (BasisKey(BasisType.MODIFIED_A, 4, pk),) * 2)
    with pytest.raises(sp.ExpansionError, match="P2 >= P1"):
        sp.make_tri(4, P2=3)


@pytest.mark.gpu
@pytest.mark.parametrize("P", PS)
@pytest.mark.parametrize("strategy", ["cuda_sumfac", "cuda_stdmat"])
def test_gpu_tri_collections(P, strategy):
    import torch

    strat = sp.Strategy(strategy)
    exp = sp.make_tri(P)
    c = torch.as_tensor(G[f"P{P}/coeffs"], device="cuda")
    u = torch.as_tensor(G[f"P{P}/phys"], device="cuda")
    E = c.shape[0]
    std = sp.ElementBatch.standard(exp, E)
    close(sp.Collection(std, sp.OperatorKind.BWD_TRANS, strat).apply(c), G[f"P{P}/std/bwd"])
    close(sp.Collection(std, sp.OperatorKind.IPRODUCT_WRT_BASE, strat).apply(u), G[f"P{P}/std/iprod"])
    close(sp.Collection(std, sp.OperatorKind.PHYS_DERIV, strat).apply(u), G[f"P{P}/std/deriv"])
    wj, inv = G[f"P{P}/wj"], G[f"P{P}/inv"]
    point = sp.ElementBatch(exp, E, sp.geometry.from_factors(exp, wj, inv, kind=sp.GEOM_POINT),
                            sp.GEOM_POINT)
    # AFFINE record per element: [det, inv00, inv01, inv10, inv11, pad]
    det = wj[:, 0] / exp.weights[0]
    aff = np.zeros((E, 6))
    aff[:, 0] = det
    aff[:, 1:5] = inv[:, 0].reshape(E, 4)
    affine = sp.ElementBatch(exp, E, torch.as_tensor(aff, device="cuda"), sp.GEOM_AFFINE)
    for batch in (point, affine):
        close(sp.Collection(batch, sp.OperatorKind.IPRODUCT_WRT_BASE, strat).apply(u), G[f"P{P}/phys/iprod"])
        close(sp.Collection(batch, sp.OperatorKind.PHYS_DERIV, strat).apply(u), G[f"P{P}/phys/deriv"])
    if strategy == "cuda_stdmat":
        f = torch.as_tensor(G[f"P{P}/flux"], device="cuda")
        close(sp.Collection(point, sp.OperatorKind.IPRODUCT_WRT_DERIV_BASE, strat).apply(f),
              G[f"P{P}/phys/ipderiv"])
    # bitwise repeatable
    coll = sp.Collection(point, sp.OperatorKind.PHYS_DERIV, strat)
    assert torch.equal(coll.apply(u), coll.apply(u))
