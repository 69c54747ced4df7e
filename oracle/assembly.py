"""C0 assembly maps and signed gather/scatter (TEST INFRASTRUCTURE ONLY).

Restates assembly.py:72-160 over an explicit element topology and
generalises it to hexahedra:

  numbering  Dirichlet block first (vertices by id, then (edge, degree));
             free vertices by id; free edge dofs by (edge id, degree);
             [hex] face dofs by (face id, degree1, degree2);
             interiors element by element in local flat order
             (assembly.py:89-133).
  conformity edge order = min over the elements sharing the edge
             (assembly.py:74-79); [hex] face order = min over the two
             elements sharing the face; excess modes pinned (gid -1,
             sign 0; assembly.py:124-127).
  signs      -1 on odd-degree bubbles of edges traversed against their
             segment (assembly.py:126-127).  Structured grids traverse every
             edge forward, so their signs are all +1 (test_assembly.py:132-140).

Structured topologies:
  quad  exactly meshio.structured_quad_mesh (meshio.py:377-413): vertex
        j*(nx+1)+i, horizontal segments first, element j*nx+i.
  hex   periodic n^3 grid (cfg4/cfg5): vertex / x-edge / x-face id
        i + n*(j + n*k) (indices mod n); y-edges and y-faces offset by n^3,
        z-edges and z-faces by 2 n^3; element ex + n*(ey + n*ez).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# local mode topology
# ---------------------------------------------------------------------------

def quad_local(m):
    """(vertex modes, edge bubble lists, interior) for a quad with m modes per
    direction (stdregions.py:259-307)."""
    flat = lambda p, q: p * m + q
    verts = (0, m, m + 1, 1)
    edges = ([flat(k, 0) for k in range(2, m)], [flat(1, k) for k in range(2, m)],
             [flat(k, 1) for k in range(2, m)], [flat(0, k) for k in range(2, m)])
    on = set(verts).union(*map(set, edges))
    interior = [n for n in range(m * m) if n not in on]
    return verts, edges, interior


def hex_local(m):
    """Hex local topology: vertices (a,b,c) lexicographic; 12 edges as
    (direction, fixed pair); 6 faces as (normal, side)."""
    flat = lambda p, q, r: (p * m + q) * m + r
    verts = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]
    vmodes = [flat(*v) for v in verts]
    edges = []
    for d in range(3):
        for s in (0, 1):
            for t in (0, 1):
                modes = []
                for k in range(2, m):
                    idx = [s, t]
                    idx.insert(d, k)
                    modes.append(flat(*idx))
                edges.append((d, s, t, modes))
    faces = []
    for d in range(3):
        for side in (0, 1):
            modes = []   # (mode, deg1, deg2) ordered by (deg1, deg2)
            for k1 in range(2, m):
                for k2 in range(2, m):
                    idx = [k1, k2]
                    idx.insert(d, side)
                    modes.append((flat(*idx), k1, k2))
            faces.append((d, side, modes))
    interior = [flat(p, q, r) for p in range(2, m) for q in range(2, m)
                for r in range(2, m)]
    return verts, vmodes, edges, faces, interior


# ---------------------------------------------------------------------------
# generic map over explicit topology
# ---------------------------------------------------------------------------

@dataclass
class ElementTopo:
    order: int
    nmodes: int
    vertex: list          # [(mode, global vertex id)]
    edges: list           # [(edge id, forward, [bubble modes by degree])]
    faces: list           # [(face id, [(mode, d1, d2)])]
    interior: list        # [mode]


@dataclass
class AssemblyMap:
    local_to_global: list
    signs: list
    num_global: int
    num_dirichlet: int
    edge_orders: dict
    face_orders: dict


def build_map(elements, dirichlet_vertices=(), dirichlet_edges=()):
    """assembly.py:72-138 generalised (faces between edges and interiors)."""
    edge_orders, face_orders = {}, {}
    for el in elements:
        for eid, _, _ in el.edges:
            edge_orders[eid] = min(edge_orders.get(eid, el.order), el.order)
        for fid, _ in el.faces:
            face_orders[fid] = min(face_orders.get(fid, el.order), el.order)
    d_verts, d_edges = set(dirichlet_vertices), set(dirichlet_edges)
    used_verts = sorted({v for el in elements for _, v in el.vertex})
    used_edge = sorted((e, d) for e, p in edge_orders.items() for d in range(2, p + 1))
    used_face = sorted((f, a, b) for f, p in face_orders.items()
                       for a in range(2, p + 1) for b in range(2, p + 1))
    vgid, egid, fgid = {}, {}, {}
    gid = 0
    for v in used_verts:
        if v in d_verts:
            vgid[v] = gid
            gid += 1
    for e, d in used_edge:
        if e in d_edges:
            egid[(e, d)] = gid
            gid += 1
    ndir = gid
    for v in used_verts:
        if v not in d_verts:
            vgid[v] = gid
            gid += 1
    for e, d in used_edge:
        if e not in d_edges:
            egid[(e, d)] = gid
            gid += 1
    for f, a, b in used_face:
        fgid[(f, a, b)] = gid
        gid += 1
    l2g_all, sgn_all = [], []
    for el in elements:
        l2g = np.full(el.nmodes, -1, dtype=np.int64)
        sgn = np.zeros(el.nmodes)
        for mode, v in el.vertex:
            l2g[mode] = vgid[v]
            sgn[mode] = 1.0
        for eid, fwd, modes in el.edges:
            pe = edge_orders[eid]
            for pos, mode in enumerate(modes):
                deg = pos + 2
                if deg > pe:
                    continue
                l2g[mode] = egid[(eid, deg)]
                sgn[mode] = 1.0 if (fwd or deg % 2 == 0) else -1.0
        for fid, modes in el.faces:
            pf = face_orders[fid]
            for mode, a, b in modes:
                if a > pf or b > pf:
                    continue
                l2g[mode] = fgid[(fid, a, b)]
                sgn[mode] = 1.0
        for mode in el.interior:
            l2g[mode] = gid
            sgn[mode] = 1.0
            gid += 1
        l2g_all.append(l2g)
        sgn_all.append(sgn)
    return AssemblyMap(l2g_all, sgn_all, gid, ndir, edge_orders, face_orders)


def assemble(amap, local):
    """Signed gather-sum in element order (assembly.py:141-147)."""
    out = np.zeros(amap.num_global)
    for l2g, sgn, vec in zip(amap.local_to_global, amap.signs, local):
        ok = l2g >= 0
        np.add.at(out, l2g[ok], sgn[ok] * np.asarray(vec)[ok])
    return out


def scatter(amap, x):
    """Signed scatter; pinned modes -> 0 (assembly.py:150-160)."""
    out = []
    for l2g, sgn in zip(amap.local_to_global, amap.signs):
        v = np.zeros(len(l2g))
        ok = l2g >= 0
        v[ok] = sgn[ok] * x[l2g[ok]]
        out.append(v)
    return out


def element_codes(amap, e):
    """C-ABI codes of one element: gid (sign +1), -1 pinned, -(gid+2) sign -1."""
    l2g, sgn = amap.local_to_global[e], amap.signs[e]
    c = l2g.copy()
    neg = sgn < 0
    c[neg] = -(l2g[neg] + 2)
    return c


def pack_map(amap):
    """(E, nm) int64 codes in the C-ABI encoding: gid (sign +1), -1 pinned,
    -(gid+2) for sign -1.  Requires a uniform mode count."""
    rows = []
    for l2g, sgn in zip(amap.local_to_global, amap.signs):
        c = l2g.copy()
        neg = sgn < 0
        c[neg] = -(l2g[neg] + 2)
        rows.append(c)
    return np.stack(rows)


# ---------------------------------------------------------------------------
# structured topologies
# ---------------------------------------------------------------------------

def quad_structured(nx, ny, orders):
    """Topology of meshio.structured_quad_mesh(nx, ny) (meshio.py:377-413).
    orders: int or sequence per element id (j*nx + i).
    Returns (elements, boundary) with boundary[name] = (vertex ids, seg ids)."""
    vid = lambda i, j: j * (nx + 1) + i
    hseg = lambda i, j: j * nx + i
    vseg = lambda i, j: (ny + 1) * nx + j * (nx + 1) + i
    els = []
    for j in range(ny):
        for i in range(nx):
            e = j * nx + i
            P = orders if np.isscalar(orders) else int(orders[e])
            m = P + 1
            vm, em, interior = quad_local(m)
            loop = [vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)]
            segs = [hseg(i, j), vseg(i + 1, j), hseg(i, j + 1), vseg(i, j)]
            els.append(ElementTopo(
                P, m * m, list(zip(vm, loop)),
                [(s, True, em[k]) for k, s in enumerate(segs)], [], interior))
    bnd = {
        "south": ([vid(i, 0) for i in range(nx + 1)], [hseg(i, 0) for i in range(nx)]),
        "east": ([vid(nx, j) for j in range(ny + 1)], [vseg(nx, j) for j in range(ny)]),
        "north": ([vid(i, ny) for i in range(nx + 1)], [hseg(i, ny) for i in range(nx)]),
        "west": ([vid(0, j) for j in range(ny + 1)], [vseg(0, j) for j in range(ny)]),
    }
    return els, bnd


def quad_structured_map(nx, ny, orders, dirichlet=()):
    els, bnd = quad_structured(nx, ny, orders)
    dv, de = set(), set()
    for name in dirichlet:
        v, s = bnd[name]
        dv.update(v)
        de.update(s)
    return build_map(els, dv, de)


def hex_periodic(n, orders):
    """Periodic n^3 hex topology; orders int or per element id."""
    N3 = n ** 3
    vid = lambda i, j, k: (i % n) + n * ((j % n) + n * (k % n))
    els = []
    for ez in range(n):
        for ey in range(n):
            for ex in range(n):
                e = ex + n * (ey + n * ez)
                P = orders if np.isscalar(orders) else int(orders[e])
                m = P + 1
                verts, vmodes, edges, faces, interior = hex_local(m)
                vert = [(mode, vid(ex + a, ey + b, ez + c))
                        for mode, (a, b, c) in zip(vmodes, verts)]
                eds = []
                for d, s, t, modes in edges:
                    off = [ex, ey, ez]
                    o = [s, t]
                    o.insert(d, 0)
                    eid = d * N3 + vid(off[0] + o[0], off[1] + o[1], off[2] + o[2])
                    eds.append((eid, True, modes))
                fcs = []
                for d, side, modes in faces:
                    off = [ex, ey, ez]
                    off[d] += side
                    fcs.append((d * N3 + vid(*off), modes))
                els.append(ElementTopo(P, m ** 3, vert, eds, fcs, interior))
    return els


def hex_periodic_map(n, orders):
    return build_map(hex_periodic(n, orders))


# ---------------------------------------------------------------------------
# vectorised periodic hex numbering (BASELINE sizes: 64^3, 48^3)
# ---------------------------------------------------------------------------

def hex_periodic_codes(n, orders):
    """build_map(hex_periodic(n, orders)) without per-element Python objects.

    The same numbering rules (assembly.py:89-133 generalised): on the periodic
    grid every vertex and every edge/face is used and there is no Dirichlet
    block, so vertex gid = vertex id; edge dofs follow in (edge id, degree)
    order, edge order = min over the 4 sharing elements (assembly.py:74-79);
    face dofs in (face id, deg1, deg2) order, face order = min over the 2
    sharing elements; interiors element by element in local flat order;
    excess modes pinned (-1).  Signs are all +1 (every edge traversed
    forward), so a code is the gid.  `tests/test_oracle.py` pins this to
    `build_map` at small n; it exists so the 64^3 / 48^3 maps can be
    compared bit for bit with the native ones.

    Returns (num_global, offsets (n^3 + 1,), codes (sum m_e^3,)) with element
    e's codes at codes[offsets[e]:offsets[e+1]] in local flat order
    (p*m + q)*m + r.
    """
    N3 = n ** 3
    orders = np.broadcast_to(np.asarray(orders, dtype=np.int64).ravel(), (N3,)) \
        if np.ndim(orders) == 0 else np.asarray(orders, dtype=np.int64).ravel()
    if orders.size != N3:
        raise ValueError(f"need {N3} orders")
    e = np.arange(N3, dtype=np.int64)
    b = (e % n, (e // n) % n, e // (n * n))

    def vid(o):
        return ((b[0] + o[0]) % n) + n * (((b[1] + o[1]) % n) + n * ((b[2] + o[2]) % n))

    def edge_id(d, s, t):
        o = [s, t]
        o.insert(d, 0)
        return d * N3 + vid(o)

    def face_id(d, side):
        o = [0, 0, 0]
        o[d] = side
        return d * N3 + vid(o)

    big = np.iinfo(np.int64).max
    eord = np.full(3 * N3, big, dtype=np.int64)
    ford = np.full(3 * N3, big, dtype=np.int64)
    for d in range(3):
        for s in (0, 1):
            for t in (0, 1):
                np.minimum.at(eord, edge_id(d, s, t), orders)
        for side in (0, 1):
            np.minimum.at(ford, face_id(d, side), orders)
    eoff = np.concatenate([[0], np.cumsum(np.maximum(eord - 1, 0))])
    foff = np.concatenate([[0], np.cumsum(np.maximum(ford - 1, 0) ** 2)])
    ebase = N3
    fbase = ebase + eoff[-1]
    ibase = fbase + foff[-1]
    nint = np.maximum(orders - 1, 0) ** 3
    ioff = ibase + np.concatenate([[0], np.cumsum(nint)])[:-1]
    offsets = np.concatenate([[0], np.cumsum((orders + 1) ** 3)])
    uniform = np.all(orders == orders[0])
    codes = None if uniform else np.empty(offsets[-1], dtype=np.int64)
    for P in np.unique(orders):
        ids = np.nonzero(orders == P)[0]
        m = int(P) + 1
        bl = tuple(x[ids] for x in b)

        def vid_l(o):
            return ((bl[0] + o[0]) % n) + n * (((bl[1] + o[1]) % n) + n * ((bl[2] + o[2]) % n))

        out = np.empty((ids.size, m ** 3), dtype=np.int64)
        interior_rank = 0
        for p in range(m):
            for q in range(m):
                for r in range(m):
                    idx = (p, q, r)
                    nb = (p >= 2) + (q >= 2) + (r >= 2)
                    col = (p * m + q) * m + r
                    if nb == 0:
                        out[:, col] = vid_l(idx)
                    elif nb == 1:
                        d = 0 if p >= 2 else (1 if q >= 2 else 2)
                        o = [idx[a] if a != d else 0 for a in range(3)]
                        eid = d * N3 + vid_l(o)
                        deg = idx[d]
                        out[:, col] = np.where(deg <= eord[eid], ebase + eoff[eid] + (deg - 2), -1)
                    elif nb == 2:
                        d = 0 if p < 2 else (1 if q < 2 else 2)
                        o = [idx[a] if a == d else 0 for a in range(3)]
                        fid = d * N3 + vid_l(o)
                        k1, k2 = [idx[a] for a in range(3) if a != d]
                        pf = ford[fid]
                        ok = (k1 <= pf) & (k2 <= pf)
                        out[:, col] = np.where(ok, fbase + foff[fid] + (k1 - 2) * (pf - 1) + (k2 - 2), -1)
                    else:
                        out[:, col] = ioff[ids] + interior_rank
                        interior_rank += 1
        if uniform:
            codes = out.reshape(-1)
        else:
            flat_idx = (offsets[ids][:, None] + np.arange(m ** 3)[None, :]).ravel()
            codes[flat_idx] = out.ravel()
    return int(ibase + nint.sum()), offsets, codes
