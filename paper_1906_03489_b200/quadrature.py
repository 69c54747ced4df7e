"""Quadrature keys and rules (mirror of spechp.quadrature, quadrature.py:19-260).

Rules and collocation matrices are computed by the native library
(csrc/tables.cpp) and cached per key, read-only like the reference's
(quadrature.py:188-214).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib


class PointsType(Enum):
    GAUSS_LEGENDRE = "gauss_legendre"
    GAUSS_LOBATTO_LEGENDRE = "gauss_lobatto_legendre"
    GAUSS_RADAU_M_LEGENDRE = "gauss_radau_m_legendre"


class QuadratureError(ValueError):
    pass


@dataclass(frozen=True)
class PointsKey:
    """Descriptor of a 1D rule (quadrature.py:30-45)."""

    num_points: int
    points_type: PointsType

    def __post_init__(self):
        if not isinstance(self.num_points, int) or self.num_points < 1:
            raise QuadratureError(
                f"num_points must be a positive integer, got {self.num_points!r}")
        if (self.points_type is PointsType.GAUSS_LOBATTO_LEGENDRE
                and self.num_points < 2):
            raise QuadratureError(
                "Gauss-Lobatto-Legendre needs at least 2 points "
                f"(got {self.num_points})")


@dataclass(frozen=True)
class QuadratureRule:
    key: PointsKey
    points: np.ndarray
    weights: np.ndarray


_cache: dict = {}
_lock = threading.Lock()


def _seg_tables(q: int, ptype: str):
    """(z, w, D) from the native library for a Q-point rule."""
    handle = C.c_void_p()
    one = (C.c_int * 1)
    rc = _lib.lib.sphp_tables_create(_lib.SHAPE_SEG, one(2), one(q), one(_lib.POINTS[ptype]),
                                     one(_lib.BASIS["modified_a"]), C.byref(handle))
    _lib.check(rc, QuadratureError)
    z = np.empty(q)
    w = np.empty(q)
    D = np.empty((q, q))
    try:
        _lib.check(_lib.lib.sphp_tables_query(handle, 0, _lib.ptr(z), _lib.ptr(w), None, None,
                                              _lib.ptr(D)))
    finally:
        _lib.lib.sphp_tables_destroy(handle)
    return z, w, D


def make_rule(key: PointsKey) -> QuadratureRule:
    """Cached rule for `key` (quadrature.py:188-214)."""
    with _lock:
        rule = _cache.get(key)
    if rule is not None:
        return rule[0]
    z, w, D = _seg_tables(key.num_points, key.points_type.value)
    for a in (z, w, D):
        a.setflags(write=False)
    rule = QuadratureRule(key, z, w)
    with _lock:
        rule = _cache.setdefault(key, (rule, D))[0]
    return rule


def diff_matrix(rule) -> np.ndarray:
    """Collocation derivative matrix on the rule's points (quadrature.py:246-260)."""
    if isinstance(rule, QuadratureRule):
        make_rule(rule.key)
        return _cache[rule.key][1].copy()
    raise QuadratureError("diff_matrix expects a QuadratureRule")
