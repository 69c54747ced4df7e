"""Hex operators pinned to the reference's own outputs.

The reference has no hexahedra, but on an affine brick every hex operator
factors exactly into the reference's quad and segment operators
(tests/golden/make_golden_hexpin.py).  The numpy oracle (CPU) and the CUDA
kernels (GPU) are checked against those Kronecker compositions:
BwdTrans, IProductWRTBase, PhysDeriv and the fused Helmholtz, P = 1..8,
Q = P+2, on the brick [0, 1/2]^3 (the n = 2 structured grid)."""
from pathlib import Path

import numpy as np
import pytest

from oracle import geometry as og
from oracle import ops

G = np.load(Path(__file__).resolve().parent / "golden" / "reference_hexpin.npz")
PS = (1, 2, 3, 4, 5, 6, 7, 8)
H, LAM = float(G["h"]), float(G["lam"])
TOL = 1e-12


def ref(P):
    g = {k: G[f"P{P}/{k}"] for k in ("B2", "W2", "M2", "K2", "Dx2", "Dy2", "B1", "w1", "D1", "M1", "K1")}
    Q = int(G[f"P{P}/Q"])
    I1, I2 = np.eye(Q), np.eye(Q * Q)
    return {
        "Q": Q,
        "B3": np.kron(g["B2"], g["B1"]),
        "W3": np.kron(g["W2"], g["w1"] * H / 2),
        "D3": (np.kron(g["Dx2"], I1), np.kron(g["Dy2"], I1), np.kron(I2, (2.0 / H) * g["D1"])),
        "H3": np.kron(g["K2"], g["M1"]) + np.kron(g["M2"], g["K1"]) + LAM * np.kron(g["M2"], g["M1"]),
    }


def close(got, want):
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert err < TOL, err


def inputs(P, Q, E=2, seed=0):
    rng = np.random.default_rng(seed + P)
    return rng.uniform(-1, 1, (E, (P + 1) ** 3)), rng.uniform(-1, 1, (E, Q ** 3))


@pytest.mark.parametrize("P", PS)
def test_oracle_hex_pinned_to_reference(P):
    r = ref(P)
    exp = ops.Expansion("hex", P, r["Q"])
    c, u = inputs(P, r["Q"])
    _, _, inv, wj = og.factors(exp, 2, [0, 0])
    close(ops.bwd(exp, c), c @ r["B3"])
    close(ops.iprod(exp, u, wj), (u * r["W3"]) @ r["B3"].T)
    d = ops.physderiv(exp, u, inv)
    for a in range(3):
        close(d[:, a], u @ r["D3"][a].T)
    Gm = ops.metric_from_inv(wj, inv)
    close(ops.helmholtz(exp, c, LAM, Gm, wj), c @ r["H3"].T)


@pytest.mark.gpu
@pytest.mark.parametrize("P", PS)
def test_gpu_hex_pinned_to_reference(P):
    import torch

    import paper_1906_03489_b200 as sp

    r = ref(P)
    Q = r["Q"]
    exp = sp.make_hex(P, Q)
    c, u = inputs(P, Q, E=8)
    cd = torch.as_tensor(c, device="cuda")
    ud = torch.as_tensor(u, device="cuda")
    std = sp.ElementBatch.standard(exp, 8)
    close(sp.Collection(std, sp.OperatorKind.BWD_TRANS, sp.Strategy.CUDA_SUMFAC).apply(cd).cpu().numpy(),
          c @ r["B3"])
    for kind in (sp.GEOM_AFFINE, sp.GEOM_POINT):
        b = sp.ElementBatch.structured(exp, 2, kind=kind, mapping=sp.MAP_AFFINE)
        ip = sp.Collection(b, sp.OperatorKind.IPRODUCT_WRT_BASE, sp.Strategy.CUDA_SUMFAC).apply(ud)
        close(ip.cpu().numpy(), (u * r["W3"]) @ r["B3"].T)
        d = sp.Collection(b, sp.OperatorKind.PHYS_DERIV, sp.Strategy.CUDA_SUMFAC).apply(ud).cpu().numpy()
        for a in range(3):
            close(d[:, a], u @ r["D3"][a].T)
    for kind in (sp.GEOM_AFFINE, sp.GEOM_METRIC):
        b = sp.ElementBatch.structured(exp, 2, kind=kind, mapping=sp.MAP_AFFINE)
        for strat in (sp.Strategy.CUDA_SUMFAC, sp.Strategy.CUDA_STDMAT):
            h = sp.Collection(b, sp.OperatorKind.HELMHOLTZ, strat, lam=LAM).apply(cd)
            close(h.cpu().numpy(), c @ r["H3"].T)
