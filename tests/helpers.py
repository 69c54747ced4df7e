"""Shared helpers for the parity tests: build GPU collections on structured
grids and the matching oracle inputs."""
import numpy as np

from oracle import geometry as og
from oracle import ops as oo

OPS = ("bwdtrans", "iproductwrtbase", "physderiv", "iproductwrtderivbase", "helmholtz")


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = max(np.linalg.norm(b), 1e-300)
    return np.linalg.norm(a - b) / den


def max_abs_norm(a, b):
    b = np.asarray(b)
    return np.max(np.abs(np.asarray(a) - b)) / max(np.max(np.abs(b)), 1e-300)


def assert_parity(got, ref, rtol=1e-12, atol_norm=1e-11, what=""):
    r = rel_l2(got, ref)
    m = max_abs_norm(got, ref)
    assert r < rtol and m < atol_norm, f"{what}: rel L2 {r:.3e}, max-abs/max {m:.3e}"


def oracle_geometry(shape, P, Q, n, ids, mapping, amp, lengths=None):
    oe = oo.Expansion(shape, P, Q)
    jac, det, inv, wj = og.factors(oe, n, np.asarray(ids), mapping, amp, lengths)
    return oe, inv, wj


def oracle_apply(op, oe, x, inv, wj, geom, lam=1.0):
    """geom: 'none' (standard elements), 'affine'/'point'/'metric' (physical)."""
    if op == "bwdtrans":
        return oo.bwd(oe, x)
    if op == "iproductwrtbase":
        w = oe.weights[None, :] if geom == "none" else wj
        return oo.iprod(oe, x, w)
    if op == "physderiv":
        return oo.physderiv(oe, x, None if geom == "none" else inv)
    if op == "iproductwrtderivbase":
        E = x.shape[0]
        if geom == "none":
            d = oe.d
            inv = np.broadcast_to(np.eye(d), (E, oe.np, d, d))
            wj = np.broadcast_to(oe.weights, (E, oe.np))
        return oo.ipderiv(oe, x.reshape(E, oe.d, oe.np), wj, inv)
    if op == "helmholtz":
        return oo.helmholtz(oe, x, lam, oo.metric_from_inv(wj, inv), wj)
    raise ValueError(op)


def input_size(op, oe):
    return {"bwdtrans": oe.nm, "iproductwrtbase": oe.np, "physderiv": oe.np,
            "iproductwrtderivbase": oe.d * oe.np, "helmholtz": oe.nm}[op]
