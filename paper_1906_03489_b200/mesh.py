"""Mesh ingestion straight into device batches.

The reference builds one Python `Element` per mesh face — expansion, an
`ElementGeom` with the coordinate map as a modal expansion (vertex modes +
fitted edge-curve bubbles, geometry.py:43-95), and `geom_factors` evaluated
per element (geometry.py:125-142) — about 10 s per 65k quads
(region.py:54-81).  Here the per-element host work is only gathering vertex
coordinates (and fitting the few curved edges); the map is evaluated on the
device for the whole batch:

  coordinate map coefficients (E, nm_geo) for x and y
    -> BwdTrans at the solution expansion's points (geometry basis of order
       p_geo on the solution's quadrature rule)
    -> PhysDeriv (reference directions; exact since p_geo <= Q-1, with the
       collapsed chain rule on triangles)
    -> jac, det, inv, w det -> POINT / METRIC records (sphp_geom_from_jacobian)

`mesh` is any object with the reference MeshGraph interface
(meshio.py:23-64: elements(), local_vertices(), face_edges(), segs, curves,
verts) — e.g. the reference's own `read_mesh` / `structured_quad_mesh`
output.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .basis import BasisKey, BasisType
from .collections import Collection, OperatorKind, Strategy
from .geometry import ElementBatch, GeometryError
from .stdregions import Shape, StdExpansion, make_quad, make_seg, make_tri

__all__ = ["element_coordinates", "geometry_from_vertices", "mesh_batch"]

# local-edge mode-axis endpoints (local vertex ids), stdregions.py:271-302
_EDGE_ENDS = {"quad": ((0, 1), (1, 2), (3, 2), (0, 3)), "tri": ((0, 1), (1, 2), (0, 2))}


def element_coordinates(mesh, kind="quad"):
    """Domain elements of `kind` in mesh.elements() order: (ids, vertex
    coordinates (E, nv, 2), curves {row: {local edge: nodes (n, 2)}}), the
    curve nodes oriented along the local edge's mode axis as build_elements
    does (region.py:64-77)."""
    rows = [eid for k, eid in mesh.elements() if k == kind]
    nv = 4 if kind == "quad" else 3
    verts = np.empty((len(rows), nv, 2))
    curves = {}
    mcurves = getattr(mesh, "curves", None) or {}
    for r, eid in enumerate(rows):
        loop = mesh.local_vertices(kind, eid)
        verts[r] = [mesh.verts[v][:2] for v in loop]
        if mcurves:
            for le, sid in enumerate(mesh.face_edges(kind, eid)):
                if sid in mcurves:
                    fwd = mesh.segs[sid][0] == loop[_EDGE_ENDS[kind][le][0]]
                    nodes = np.array([p[:2] for p in mcurves[sid]], dtype=float)
                    curves.setdefault(r, {})[le] = nodes if fwd else nodes[::-1]
    return np.asarray(rows), verts, curves


def _geom_expansion(exp, p_geo):
    """Coordinate-map basis of order p_geo on the solution's quadrature rule."""
    keys = exp.basis_keys
    if exp.shape is Shape.QUAD:
        return StdExpansion(Shape.QUAD, (BasisKey(BasisType.MODIFIED_A, p_geo + 1, keys[0].points_key),
                                         BasisKey(BasisType.MODIFIED_A, p_geo + 1, keys[1].points_key)))
    return StdExpansion(Shape.TRI, (BasisKey(BasisType.MODIFIED_A, p_geo + 1, keys[0].points_key),
                                    BasisKey(BasisType.MODIFIED_B, p_geo + 1, keys[1].points_key)))


def _mode_layout(shape, m):
    """vertex modes and per-edge bubble modes (stdregions.py:260-302) for a
    geometry expansion with m modes per direction."""
    if shape is Shape.QUAD:
        flat = lambda p, q: p * m + q  # noqa: E731
        return ((0, m, m + 1, 1),
                ([flat(k, 0) for k in range(2, m)], [flat(1, k) for k in range(2, m)],
                 [flat(k, 1) for k in range(2, m)], [flat(0, k) for k in range(2, m)]))
    bs = np.cumsum([0] + [m] + [m - p for p in range(1, m)])[:m]  # block starts
    return ((0, int(bs[1]), 1),
            ([int(bs[k]) for k in range(2, m)], [int(bs[1]) + k for k in range(1, m - 1)],
             list(range(2, m))))


def _fit_curve(nodes):
    """Boundary-first modal coefficients of a curve sampled at GLL
    parameters (geometry.py:27-37)."""
    n = len(nodes)
    if n < 2:
        raise GeometryError("curve needs at least 2 nodes")
    B = make_seg(n - 1, num_points=n).tables[0][0]   # (modes, n)
    return np.linalg.solve(B.T, nodes)


def geometry_from_vertices(exp, verts, curves=None, kind=_lib.GEOM_POINT, device=None, ids=None):
    """Device geometry records (E, stride) of the elements whose vertices
    (E, nv, 2) and optional curved edges {row: {edge: nodes}} are given."""
    dev = torch.device(device or "cuda")
    shape = exp.shape
    verts = np.asarray(verts, dtype=float)
    E = verts.shape[0]
    curves = curves or {}
    p_geo = 1
    for cs in curves.values():
        for nodes in cs.values():
            p_geo = max(p_geo, len(nodes) - 1)
    gexp = _geom_expansion(exp, p_geo)
    vmodes, emodes = _mode_layout(shape, p_geo + 1)
    coeffs = np.zeros((2, E, gexp.num_modes))
    for v, mode in enumerate(vmodes):
        coeffs[:, :, mode] = verts[:, v, :].T
    for r, cs in curves.items():
        for le, nodes in cs.items():
            c1d = _fit_curve(np.asarray(nodes, float))
            ends = verts[r, list(_EDGE_ENDS["quad" if shape is Shape.QUAD else "tri"][le])]
            if np.max(np.abs(c1d[:2] - ends)) > 1e-8:
                eid = ids[r] if ids is not None else r
                raise GeometryError(f"element {eid}: curve on edge {le} does not meet the element vertices")
            for k, mode in enumerate(emodes[le]):
                if k + 2 < len(c1d):
                    coeffs[:, r, mode] = c1d[k + 2]
    c = torch.as_tensor(coeffs.reshape(2 * E, -1), device=dev)
    # the map at the points, then its reference-direction derivatives
    bwd = Collection(ElementBatch.standard(gexp, 2 * E), OperatorKind.BWD_TRANS, Strategy.CUDA_STDMAT)
    xy = bwd.apply(c)
    der = Collection(ElementBatch.standard(exp, 2 * E), OperatorKind.PHYS_DERIV,
                     Strategy.CUDA_SUMFAC if _fast(exp) else Strategy.CUDA_STDMAT).apply(xy)
    der = der.reshape(2, E, 2, -1)
    stride = _lib.lib.sphp_geom_stride(exp.native.handle, kind)
    out = torch.empty((E, stride), dtype=torch.float64, device=dev)
    import ctypes as C
    bad = C.c_int64()
    rc = _lib.lib.sphp_geom_from_jacobian(exp.native.handle, kind, E, _lib.ptr(der[0].contiguous()),
                                          _lib.ptr(der[1].contiguous()), _lib.ptr(out), C.byref(bad),
                                          _lib.stream_ptr())
    if rc != _lib.OK:
        msg = _lib.last_error()
        if bad.value >= 0 and ids is not None:
            msg = msg.replace(f"element {bad.value}:", f"element {ids[bad.value]}:", 1)
        raise GeometryError(msg)
    return out


def _fast(exp):
    try:
        Collection(ElementBatch.standard(exp, 1), OperatorKind.PHYS_DERIV, Strategy.CUDA_SUMFAC)
        return True
    except Exception:
        return False


def mesh_batch(mesh, P, num_points=None, kind="quad", geom_kind=_lib.GEOM_POINT, device=None):
    """build_elements (region.py:54-81) for a uniform-order mesh as one
    device ElementBatch: (element ids, batch)."""
    exp = make_quad(P, num_points) if kind == "quad" else make_tri(P, num_points)
    ids, verts, curves = element_coordinates(mesh, kind)
    geom = geometry_from_vertices(exp, verts, curves, geom_kind, device, ids=ids)
    return ids, ElementBatch(exp, len(ids), geom, geom_kind)
