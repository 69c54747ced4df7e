"""Reference elements (mirror of spechp.stdregions, stdregions.py:41-399,
generalised to hexahedra).

Storage conventions are the reference's (stdregions.py:1-14): boundary-first
1D modes, coefficient n = p*m2 + q (quad) / (p*m2 + q)*m3 + r (hex), points
flattened C-order with the first direction slowest.  The tables come from
the native library (`sphp_tables_create`), one handle per expansion.

`native_key(exp)` duck-types any StdExpansion-like object — including the
reference's own `spechp.stdregions.StdExpansion` — into the C-ABI key, so
elements built by the reference (`region.build_elements`) can be handed to
the GPU collections unchanged.
"""
from __future__ import annotations

import ctypes as C
from enum import Enum
from functools import cached_property

import numpy as np

from . import _lib
from .basis import BasisKey, BasisType
from .quadrature import PointsKey, PointsType, make_rule


class Shape(Enum):
    SEG = "seg"
    QUAD = "quad"
    TRI = "tri"
    HEX = "hex"


class ExpansionError(ValueError):
    pass


_SHAPE_CODE = {"seg": _lib.SHAPE_SEG, "quad": _lib.SHAPE_QUAD, "tri": _lib.SHAPE_TRI,
               "hex": _lib.SHAPE_HEX}
_DIMS = {"seg": 1, "quad": 2, "tri": 2, "hex": 3}


def _value(x):
    return x.value if hasattr(x, "value") else x


def native_key(exp):
    """(shape code, modes, points, points types, basis types) of any
    StdExpansion-like object (shape + basis_keys with num_modes and
    points_key.{num_points, points_type})."""
    shape = _value(exp.shape)
    if shape not in _SHAPE_CODE:
        raise ExpansionError(f"unknown shape {shape!r}")
    keys = tuple(exp.basis_keys)
    modes = tuple(int(k.num_modes) for k in keys)
    pts = tuple(int(k.points_key.num_points) for k in keys)
    ptypes = tuple(_lib.POINTS[_value(k.points_key.points_type)] for k in keys)
    btypes = tuple(_lib.BASIS[_value(k.basis_type)] for k in keys)
    return _SHAPE_CODE[shape], modes, pts, ptypes, btypes


class NativeTables:
    """Owner of one `sphp_tables` handle."""

    def __init__(self, shape_code, modes, pts, ptypes, btypes):
        n = len(modes)
        arr = C.c_int * n
        self.handle = C.c_void_p()
        rc = _lib.lib.sphp_tables_create(shape_code, arr(*modes), arr(*pts), arr(*ptypes),
                                         arr(*btypes), C.byref(self.handle))
        _lib.check(rc, ExpansionError)
        self.dim = n
        self.modes, self.pts = modes, pts
        self.tri = shape_code == _lib.SHAPE_TRI
        nm = C.c_int64()
        _lib.check(_lib.lib.sphp_tables_sizes(self.handle, C.byref(nm), None, None))
        self.num_modes = nm.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.sphp_tables_destroy(h)
            self.handle = None

    def direction(self, d):
        q, m = self.pts[d], self.modes[d]
        if self.tri and d == 1:  # Modified_B: one row per triangle mode
            m = self.num_modes
        z, w = np.empty(q), np.empty(q)
        B, Bd, D = np.empty((m, q)), np.empty((m, q)), np.empty((q, q))
        _lib.check(_lib.lib.sphp_tables_query(self.handle, d, _lib.ptr(z), _lib.ptr(w),
                                              _lib.ptr(B), _lib.ptr(Bd), _lib.ptr(D)))
        return z, w, B, Bd, D


_table_cache: dict = {}


def native_tables(exp) -> NativeTables:
    key = native_key(exp)
    t = _table_cache.get(key)
    if t is None:
        t = _table_cache.setdefault(key, NativeTables(*key))
    return t


class StdExpansion:
    """A reference element: shape plus one basis key per direction
    (stdregions.py:70-370).  Immutable; derived tables cached."""

    def __init__(self, shape: Shape, basis_keys):
        basis_keys = tuple(basis_keys)
        expected = _DIMS[shape.value]
        if len(basis_keys) != expected:
            raise ExpansionError(
                f"{shape.value} needs {expected} basis keys, got {len(basis_keys)}")
        if shape is Shape.TRI:  # stdregions.py:83-91
            if basis_keys[1].basis_type is not BasisType.MODIFIED_B:
                raise ExpansionError("triangle direction 2 must use the collapsed-direction basis")
            if basis_keys[0].basis_type is not BasisType.MODIFIED_A:
                raise ExpansionError("triangle direction 1 must be modal")
            if basis_keys[1].num_modes < basis_keys[0].num_modes:
                raise ExpansionError("triangle needs P2 >= P1")
        else:
            for key in basis_keys:
                if key.basis_type is BasisType.MODIFIED_B:
                    raise ExpansionError("collapsed-direction basis is only valid on triangles")
        self.shape = shape
        self.basis_keys = basis_keys

    @cached_property
    def native(self) -> NativeTables:
        return native_tables(self)

    @cached_property
    def rules(self):
        return tuple(make_rule(k.points_key) for k in self.basis_keys)

    @property
    def dim(self):
        return len(self.basis_keys)

    @property
    def num_points_dir(self):
        return tuple(k.points_key.num_points for k in self.basis_keys)

    @property
    def num_points(self):
        return int(np.prod(self.num_points_dir))

    @cached_property
    def num_modes(self):
        if self.shape is Shape.TRI:
            return self.native.num_modes
        return int(np.prod([k.num_modes for k in self.basis_keys]))

    @cached_property
    def tables(self):
        """Per-direction (values, derivs) in storage order (stdregions.py:137-148)."""
        return tuple(self.native.direction(d)[2:4] for d in range(self.dim))

    @cached_property
    def weights(self):
        ws = [self.native.direction(d)[1] for d in range(self.dim)]
        if self.shape is Shape.TRI:  # collapse Jacobian in direction 2 (stdregions.py:113-121)
            z2 = self.native.direction(1)[0]
            ws[1] = ws[1] * 0.5 * (1.0 - z2)
        out = ws[0]
        for w in ws[1:]:
            out = np.multiply.outer(out, w)
        return np.asarray(out).ravel()

    @cached_property
    def points(self):
        zs = [self.native.direction(d)[0] for d in range(self.dim)]
        grids = np.meshgrid(*zs, indexing="ij")
        pts = np.stack([g.ravel() for g in grids], axis=1)
        if self.shape is Shape.TRI:  # duffy_collapse (basis.py:187-195)
            xi = pts.copy()
            xi[:, 0] = 0.5 * (1.0 + pts[:, 0]) * (1.0 - pts[:, 1]) - 1.0
            return xi
        return pts

    @cached_property
    def mode_index(self):
        if self.shape is Shape.TRI:  # blocks p, q = 0..P2-p (basis.py:117-157)
            P1, P2 = self.basis_keys[0].num_modes - 1, self.basis_keys[1].num_modes - 1
            return tuple((p, q) for p in range(P1 + 1) for q in range(P2 + 1 - p if p else P2 + 1))
        ms = [k.num_modes for k in self.basis_keys]
        return tuple(np.unravel_index(n, ms) for n in range(self.num_modes))

    @cached_property
    def _collapse_factors(self):
        """Chain-rule factors f = 2/(1-eta2), g = (1+eta1)/(1-eta2) (stdregions.py:210-217)."""
        eta1, eta2 = self.native.direction(0)[0], self.native.direction(1)[0]
        return 2.0 / (1.0 - eta2)[None, :], (1.0 + eta1)[:, None] / (1.0 - eta2)[None, :]

    @cached_property
    def bwd_matrix(self):
        """Dense B[n, i] = phi_n(xi_i) (stdregions.py:189-208)."""
        if self.shape is Shape.TRI:
            a1, b2 = self.tables[0][0], self.tables[1][0]
            rows = []
            for n, (p, q) in enumerate(self.mode_index):
                m = np.outer(a1[p], b2[n])
                if (p, q) == (0, 1):
                    m = m + np.outer(a1[1], b2[n])
                rows.append(m.ravel())
            return np.array(rows)
        out = self.tables[0][0]
        for d in range(1, self.dim):
            out = np.einsum("ni,pj->npij", out, self.tables[d][0]).reshape(
                out.shape[0] * self.tables[d][0].shape[0], -1)
        return out

    @cached_property
    def deriv_matrices(self):
        """Collocation derivative operators per direction (stdregions.py:218-235)."""
        Ds = [self.native.direction(d)[4] for d in range(self.dim)]
        out = []
        for a in range(self.dim):
            k = np.ones((1, 1))
            for d in range(self.dim):
                k = np.kron(k, Ds[d] if d == a else np.eye(len(Ds[d])))
            out.append(k)
        if self.shape is Shape.TRI:  # collapsed chain rule (stdregions.py:221-235)
            f, g = self._collapse_factors
            q1, q2 = self.num_points_dir
            fr = np.broadcast_to(f, (q1, q2)).ravel()
            return (fr[:, None] * out[0], g.ravel()[:, None] * out[0] + out[1])
        return tuple(out)

    @cached_property
    def deriv_bwd_matrices(self):
        return tuple(self.bwd_matrix @ d.T for d in self.deriv_matrices)


def _gll(n):
    return PointsKey(n, PointsType.GAUSS_LOBATTO_LEGENDRE)


def make_seg(P, num_points=None, basis=BasisType.MODIFIED_A):
    pk = _gll(num_points or P + 2)
    return StdExpansion(Shape.SEG, (BasisKey(basis, P + 1, pk),))


def make_quad(P, num_points=None, basis=BasisType.MODIFIED_A, P2=None):
    """stdregions.py:391-399 (default Q = P+2 points, one more than modes)."""
    m1, m2 = P + 1, (P2 if P2 is not None else P) + 1
    pk1 = _gll(num_points or m1 + 1)
    pk2 = _gll(num_points or m2 + 1)
    return StdExpansion(Shape.QUAD, (BasisKey(basis, m1, pk1), BasisKey(basis, m2, pk2)))


def make_tri(P, num_points=None, P2=None):
    """stdregions.py:402-408: Modified_A on GLL x Modified_B on Gauss-Radau."""
    m1, m2 = P + 1, (P2 if P2 is not None else P) + 1
    pk1 = PointsKey(num_points or m1 + 1, PointsType.GAUSS_LOBATTO_LEGENDRE)
    pk2 = PointsKey(num_points or m2 + 1, PointsType.GAUSS_RADAU_M_LEGENDRE)
    return StdExpansion(Shape.TRI, (BasisKey(BasisType.MODIFIED_A, m1, pk1),
                                    BasisKey(BasisType.MODIFIED_B, m2, pk2)))


def make_hex(P, num_points=None, basis=BasisType.MODIFIED_A):
    """The hexahedral generalisation: three identical Modified_A keys."""
    pk = _gll(num_points or P + 2)
    return StdExpansion(Shape.HEX, (BasisKey(basis, P + 1, pk),) * 3)


def make_expansion(shape, P, num_points=None, basis=BasisType.MODIFIED_A):
    if shape is Shape.SEG:
        return make_seg(P, num_points, basis)
    if shape is Shape.QUAD:
        return make_quad(P, num_points, basis)
    if shape is Shape.HEX:
        return make_hex(P, num_points, basis)
    if shape is Shape.TRI:
        return make_tri(P, num_points)
    raise ExpansionError(f"unsupported shape {shape}")
