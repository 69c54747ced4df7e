"""Batched elemental operators, numpy restatement (TEST INFRASTRUCTURE ONLY).

Layout (stdregions.py:1-14, :123-133, :189-198, generalised to hex):
  quad coefficient n = p*m2 + q,            point (i, j)    -> i*Q2 + j
  hex  coefficient n = (p*m2 + q)*m3 + r,   point (i, j, k) -> (i*Q2 + j)*Q3 + k
first direction slowest.  Blocks are (E, nm) / (E, np) / (E, d, np) float64.

Operators follow collections.py:
  bwd        u = (B1 x B2 [x B3])^T uhat             collections.py:133-150
  iprod      b = (B1 x B2 [x B3]) (W u)              collections.py:152-167, :215-224
  physderiv  d_a = D_a u ; world: dx_k = sum_a inv[a,k] d_a   collections.py:169-185
  ipderiv    b = sum_a B_a [ W sum_k inv[a,k] f_k ]  geometry.py:163-168 / solvers.py:361-365
  helmholtz  y = sum_ab B_a G_ab B_b^T uhat + lam B wJ B^T uhat
             with G_ab = wJ sum_k inv[a,k] inv[b,k]   geometry.py:171-184, assembly.py:189-191
The sum-factorised forms contract one direction at a time; the dense
(StdMat) forms build the Kronecker operators explicitly (collections.py:203-229).
"""
from __future__ import annotations

import numpy as np

from .tables import GLL, tables


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def dims(shape: str):
    return {"quad": 2, "hex": 3}[shape]


class Expansion:
    """Per-shape reference element of order P with Q points per direction."""

    def __init__(self, shape: str, P: int, Q: int | None = None, ptype: str = GLL):
        self.shape = shape
        self.d = dims(shape)
        self.P = P
        self.m = P + 1
        self.Q = Q if Q is not None else P + 2
        self.t = tables(self.m, self.Q, ptype)
        self.nm = self.m ** self.d
        self.np = self.Q ** self.d

    @property
    def weights(self):
        w = self.t.w
        if self.d == 2:
            return np.outer(w, w).ravel()
        return np.einsum("i,j,k->ijk", w, w, w).ravel()

    # dense Kronecker operators (StdMat) ------------------------------------
    def bwd_matrix(self):
        """B[n, i] = phi_n(xi_i) (stdregions.py:189-198)."""
        B = self.t.B
        if self.d == 2:
            return np.einsum("pi,qj->pqij", B, B).reshape(self.nm, self.np)
        return np.einsum("pi,qj,rk->pqrijk", B, B, B).reshape(self.nm, self.np)

    def deriv_matrices(self):
        """Collocation derivative operators per direction (stdregions.py:218-235)."""
        D, I = self.t.D, np.eye(self.Q)
        if self.d == 2:
            return (np.kron(D, I), np.kron(I, D))
        return (np.kron(np.kron(D, I), I), np.kron(np.kron(I, D), I),
                np.kron(np.kron(I, I), D))

    def deriv_bwd_matrices(self):
        """B_a[n, i] = d(phi_n)/d(xi_a) at point i (stdregions.py:237-240)."""
        B = self.bwd_matrix()
        return tuple(B @ Da.T for Da in self.deriv_matrices())


# ---------------------------------------------------------------------------
# 1D contraction along one direction of an (E, n0, n1[, n2]) tensor
# ---------------------------------------------------------------------------

def _contract(x, A, axis):
    """y[..., o, ...] = sum_i A[i, o] x[..., i, ...] along tensor `axis`
    (axis counted after the element axis)."""
    y = np.tensordot(x, A, axes=([axis + 1], [0]))       # moves new axis last
    return np.moveaxis(y, -1, axis + 1)


def bwd(exp: Expansion, coeffs):
    E = coeffs.shape[0]
    m, Q, B = exp.m, exp.Q, exp.t.B
    x = coeffs.reshape((E,) + (m,) * exp.d)
    for a in reversed(range(exp.d)):            # last direction first, like :140,:149
        x = _contract(x, B, a)
    return x.reshape(E, exp.np)


def iprod_unweighted(exp: Expansion, vals):
    E = vals.shape[0]
    Q, B = exp.Q, exp.t.B
    x = vals.reshape((E,) + (Q,) * exp.d)
    for a in range(exp.d):                      # first direction first, like :157-160
        x = _contract(x, B.T, a)
    return x.reshape(E, exp.nm)


def iprod(exp: Expansion, vals, wts):
    """wts: (np,) standard weights or (E, np) world weights w*|J|."""
    return iprod_unweighted(exp, vals * wts)


def ref_deriv(exp: Expansion, vals):
    """(E, d, np) reference-coordinate collocation derivatives."""
    E = vals.shape[0]
    Q, D = exp.Q, exp.t.D
    x = vals.reshape((E,) + (Q,) * exp.d)
    out = np.empty((E, exp.d, exp.np))
    for a in range(exp.d):
        out[:, a] = _contract(x, D.T, a).reshape(E, exp.np)
    return out


def deriv_transpose(exp: Expansion, flux):
    """sum_a D_a^T flux_a: the adjoint of ref_deriv, (E, d, np) -> (E, np)."""
    E = flux.shape[0]
    Q, D = exp.Q, exp.t.D
    out = np.zeros((E,) + (Q,) * exp.d)
    for a in range(exp.d):
        out += _contract(flux[:, a].reshape((E,) + (Q,) * exp.d), D, a)
    return out.reshape(E, exp.np)


def physderiv(exp: Expansion, vals, inv=None):
    """inv: None (reference derivatives) or (E, np, d, d) with inv[e,i,a,k] =
    dxi_a/dx_k (geometry.py:115-142).  Returns (E, d, np)."""
    d = ref_deriv(exp, vals)
    if inv is None:
        return d
    # dx_k = sum_a inv[a,k] d_a  (collections.py:181-185)
    return np.einsum("eiak,eai->eki", inv, d)


def ipderiv(exp: Expansion, flux, wj, inv):
    """IProductWRTDerivBase (geometry.py:163-168): flux (E, d, np) world
    components, wj (E, np) = w*|J|, inv (E, np, d, d)."""
    g = np.einsum("ei,eiak,eki->eai", wj, inv, flux)
    return iprod_unweighted(exp, deriv_transpose(exp, g))


def metric_from_inv(wj, inv):
    """G_ab = wJ sum_k inv[a,k] inv[b,k]  -> (E, d, d, np)."""
    return np.einsum("ei,eiak,eibk->eabi", wj, inv, inv)


def helmholtz(exp: Expansion, coeffs, lam, G, wj):
    """Fused local Helmholtz by sum-factorisation.
    G: (E, d, d, np) symmetric metric with weights; wj: (E, np)."""
    u = bwd(exp, coeffs)
    du = ref_deriv(exp, u)
    flux = np.einsum("eabi,ebi->eai", G, du)
    t = deriv_transpose(exp, flux) + lam * wj * u
    return iprod_unweighted(exp, t)


def helmholtz_dense(exp: Expansion, coeffs, lam, G, wj):
    """Elemental-matrix form (geometry.py:171-184): per element
    H = sum_ab B_a diag(G_ab) B_b^T + lam B diag(wJ) B^T, symmetrised."""
    B = exp.bwd_matrix()
    Ba = exp.deriv_bwd_matrices()
    out = np.empty((coeffs.shape[0], exp.nm))
    for e in range(coeffs.shape[0]):
        H = lam * (B * wj[e][None, :]) @ B.T
        for a in range(exp.d):
            for b in range(exp.d):
                H += (Ba[a] * G[e, a, b][None, :]) @ Ba[b].T
        H = 0.5 * (H + H.T)
        out[e] = H @ coeffs[e]
    return out


def elemental_helmholtz_matrices(exp: Expansion, lam, G, wj):
    """(E, nm, nm) dense elemental Helmholtz matrices (StdMat strategy)."""
    B = exp.bwd_matrix()
    Ba = exp.deriv_bwd_matrices()
    E = wj.shape[0]
    H = lam * np.einsum("ni,ei,mi->enm", B, wj, B)
    for a in range(exp.d):
        for b in range(exp.d):
            H += np.einsum("ni,ei,mi->enm", Ba[a], G[:, a, b], Ba[b])
    return 0.5 * (H + np.transpose(H, (0, 2, 1)))


# ---------------------------------------------------------------------------
# cost model (collections.py:250-273 generalised)
# ---------------------------------------------------------------------------

def mac_count(shape, op, strategy, P, Q, E, geometry=True):
    d = dims(shape)
    m = P + 1
    nm, npts = m ** d, Q ** d
    if d == 2:
        staged = m * m * Q + m * Q * Q
    else:
        staged = m ** 3 * Q + m * m * Q * Q + m * Q ** 3
    dense = nm * npts
    if op == "bwdtrans":
        per = dense if strategy == "stdmat" else staged
    elif op == "iproductwrtbase":
        per = npts + (dense if strategy == "stdmat" else staged)
    elif op == "physderiv":
        ref = d * npts * npts if strategy == "stdmat" else d * Q ** (d + 1)
        per = ref + (d * d * npts if geometry else 0)
    elif op == "iproductwrtderivbase":
        ref = d * npts * npts + dense if strategy == "stdmat" else d * Q ** (d + 1) + staged
        per = ref + (d * d + d) * npts
    elif op == "helmholtz":
        if strategy == "stdmat":
            per = nm * nm
        else:
            per = 2 * staged + 2 * d * Q ** (d + 1) + (d * d + d + 2) * npts
    else:
        raise ValueError(op)
    return E * per
