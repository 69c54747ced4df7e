"""Analytic element maps of the BASELINE configs (TEST INFRASTRUCTURE ONLY).

Per-point factors follow geometry.py:115-142: jac[i,k,a] = dx_k/dxi_a,
det, inv[i,a,k] = dxi_a/dx_k, weights_world = w * det.  The reference can
only express polynomial edge curves (geometry.py:59-78), so the analytic
maps named in BASELINE.json are restated here; the CUDA geometry kernel
evaluates the same closed forms.

Structured grids: element (ex, ey[, ez]) has id ex + n*(ey + n*ez)
(meshio.py:400-405 generalised); reference direction 0 <-> x, 1 <-> y, 2 <-> z.
"""
from __future__ import annotations

import numpy as np

from .ops import Expansion

TWO_PI = 2.0 * np.pi

# mapping ids shared with the C ABI (include/spechp_b200.h, SPHP_MAP_*)
MAP_AFFINE = 0          # x' = x
MAP_QUAD_SINE = 1       # cfg2: x' = x + a sin(2 pi y), y' = y + a sin(2 pi x)
MAP_HEX_SINE = 2        # cfg4: x' = x + a sin(2 pi y) sin(2 pi z)


def element_points(exp: Expansion, n, elems, lengths=None):
    """Undeformed world points (E, np, d) of structured-grid elements."""
    d = exp.d
    z = exp.t.z
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    h = L / n
    elems = np.asarray(elems)
    idx = []
    rem = elems.copy()
    for a in range(d):
        idx.append(rem % n)
        rem = rem // n
    grids = np.meshgrid(*([z] * d), indexing="ij")
    out = np.empty((len(elems), exp.np, d))
    for a in range(d):
        out[:, :, a] = (idx[a][:, None] + 0.5 * (grids[a].ravel()[None, :] + 1.0)) * h[a]
    return out


def factors(exp: Expansion, n, elems, mapping=MAP_AFFINE, amp=0.0, lengths=None):
    """Per-point (jac, det, inv, wj) for the structured grid elements."""
    d = exp.d
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    h = L / n
    x = element_points(exp, n, elems, lengths)
    E = x.shape[0]
    jac = np.zeros((E, exp.np, d, d))
    for a in range(d):
        jac[:, :, a, a] = 0.5 * h[a]
    if mapping == MAP_QUAD_SINE:
        X, Y = x[..., 0], x[..., 1]
        # d x'/d y = a 2pi cos(2pi y) ; d y'/d x = a 2pi cos(2pi x)
        jac[:, :, 0, 1] = amp * TWO_PI * np.cos(TWO_PI * Y) * 0.5 * h[1]
        jac[:, :, 1, 0] = amp * TWO_PI * np.cos(TWO_PI * X) * 0.5 * h[0]
    elif mapping == MAP_HEX_SINE:
        Y, Z = x[..., 1], x[..., 2]
        jac[:, :, 0, 1] = amp * TWO_PI * np.cos(TWO_PI * Y) * np.sin(TWO_PI * Z) * 0.5 * h[1]
        jac[:, :, 0, 2] = amp * TWO_PI * np.sin(TWO_PI * Y) * np.cos(TWO_PI * Z) * 0.5 * h[2]
    elif mapping != MAP_AFFINE:
        raise ValueError(mapping)
    det = np.linalg.det(jac)
    if np.any(det <= 0):
        raise ValueError("non-positive Jacobian")
    inv = np.linalg.inv(jac)            # inv[a, k] = dxi_a / dx_k
    wj = exp.weights[None, :] * det
    return jac, det, inv, wj


def world_points(exp: Expansion, n, elems, mapping=MAP_AFFINE, amp=0.0, lengths=None):
    x = element_points(exp, n, elems, lengths)
    if mapping == MAP_QUAD_SINE:
        X, Y = x[..., 0].copy(), x[..., 1].copy()
        x[..., 0] = X + amp * np.sin(TWO_PI * Y)
        x[..., 1] = Y + amp * np.sin(TWO_PI * X)
    elif mapping == MAP_HEX_SINE:
        x[..., 0] = x[..., 0] + amp * np.sin(TWO_PI * x[..., 1]) * np.sin(TWO_PI * x[..., 2])
    return x
