"""Device-resident geometric factors (geometry.py:115-142 semantics).

The reference stores per-element `GeomFactors` (jac, det, inv,
weights_world) as numpy arrays and stacks them per collection
(collections.py:110-129).  On the B200 the factors of a whole element batch
live in HBM in one of four encodings (include/spechp_b200.h SPHP_GEOM_*):

  NONE    standard elements (reference weights only)
  AFFINE  per element [det, inv(d x d)]        - constant-Jacobian elements
  POINT   per element, SoA over points [wJ, inv_ak]
  METRIC  per element, SoA over points [G_ab (symmetric), wJ]   (Helmholtz)

with each per-point component padded to an even count of doubles so every
element record is 16-byte aligned for the TMA bulk copies.

`ElementBatch` is the batch descriptor the north star asks for: shape/key,
element count and the geometry tensor, so a 262,144-element mesh never
becomes 262,144 Python objects.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .stdregions import native_tables

GEOM_NONE, GEOM_AFFINE, GEOM_POINT, GEOM_METRIC = (
    _lib.GEOM_NONE, _lib.GEOM_AFFINE, _lib.GEOM_POINT, _lib.GEOM_METRIC)
MAP_AFFINE, MAP_QUAD_SINE, MAP_HEX_SINE = _lib.MAP_AFFINE, _lib.MAP_QUAD_SINE, _lib.MAP_HEX_SINE


class GeometryError(ValueError):
    pass


@dataclass(frozen=True)
class GeomFactors:
    """Per-quadrature-point mapping factors of one element (geometry.py:115-122)."""

    jac: np.ndarray
    det: np.ndarray
    inv: np.ndarray
    weights_world: np.ndarray


def geom_stride(exp, kind) -> int:
    return int(_lib.lib.sphp_geom_stride(native_tables(exp).handle, kind))


def structured_geometry(exp, n, kind=GEOM_METRIC, mapping=MAP_AFFINE, amp=0.0, lengths=None,
                        elem_ids=None, e0=0, num_elements=None, device=None, stream=None):
    """Geometry of elements of the structured n^d grid on [0, L]^d with an
    analytic map, evaluated on the device.  Element id = ex + n*(ey + n*ez)."""
    t = native_tables(exp)
    dim = t.dim
    if elem_ids is not None:
        ids = torch.as_tensor(elem_ids, dtype=torch.int64, device=device or "cuda")
        E = ids.numel()
    else:
        ids = None
        E = n ** dim - e0 if num_elements is None else num_elements
    stride = geom_stride(exp, kind)
    out = torch.empty((E, stride), dtype=torch.float64, device=device or "cuda")
    L = (ctypes_doubles(lengths or [1.0] * 3))
    rc = _lib.lib.sphp_geom_analytic(t.handle, kind, mapping, n, L, float(amp), e0, E,
                                     _lib.ptr(ids), _lib.ptr(out), _lib.stream_ptr(stream))
    _lib.check(rc, GeometryError)
    return out


def ctypes_doubles(vals):
    import ctypes as C

    arr = (C.c_double * 3)(*([float(v) for v in vals] + [1.0] * (3 - len(vals))))
    return arr


def from_factors(exp, weights_world, inv, kind=GEOM_POINT, device=None, stream=None):
    """Encode reference-layout factors — weights_world (E, np) and inv
    (E, np, d, d) — as POINT or METRIC on the device."""
    t = native_tables(exp)
    dev = device or "cuda"
    wj = torch.as_tensor(np.ascontiguousarray(weights_world, dtype=np.float64)
                         if not torch.is_tensor(weights_world) else weights_world,
                         dtype=torch.float64, device=dev).contiguous()
    iv = torch.as_tensor(np.ascontiguousarray(inv, dtype=np.float64)
                         if not torch.is_tensor(inv) else inv,
                         dtype=torch.float64, device=dev).contiguous()
    E = wj.shape[0]
    out = torch.empty((E, geom_stride(exp, kind)), dtype=torch.float64, device=dev)
    rc = _lib.lib.sphp_geom_from_factors(t.handle, kind, E, _lib.ptr(wj), _lib.ptr(iv),
                                         _lib.ptr(out), _lib.stream_ptr(stream))
    _lib.check(rc, GeometryError)
    return out


class ElementBatch:
    """A homogeneous batch of E elements sharing one expansion, with its
    geometry tensor already on the device (or none for standard elements)."""

    def __init__(self, exp, num_elements, geometry=None, geom_kind=GEOM_NONE, elem_ids=None):
        self.exp = exp
        self.num_elements = int(num_elements)
        self.geometry = geometry
        self.geom_kind = geom_kind if geometry is not None else GEOM_NONE
        self.elem_ids = elem_ids
        if geometry is not None:
            want = geom_stride(exp, self.geom_kind)
            if tuple(geometry.shape) != (self.num_elements, want):
                raise GeometryError(
                    f"geometry shape {tuple(geometry.shape)} != ({self.num_elements}, {want})")
            if geometry.dtype != torch.float64 or not geometry.is_cuda or not geometry.is_contiguous():
                raise GeometryError("geometry must be a contiguous float64 CUDA tensor")

    def __len__(self):
        return self.num_elements

    @classmethod
    def structured(cls, exp, n, kind=GEOM_METRIC, mapping=MAP_AFFINE, amp=0.0, lengths=None,
                   elem_ids=None, device=None):
        g = structured_geometry(exp, n, kind, mapping, amp, lengths, elem_ids, device=device)
        return cls(exp, g.shape[0], g, kind, elem_ids)

    @classmethod
    def standard(cls, exp, num_elements):
        return cls(exp, num_elements)
