"""Reference geometric factors for mesh ingestion.

    python tests/golden/make_golden_mesh.py  ->  tests/golden/reference_mesh.npz

Two meshes built with the reference's meshio, vertices perturbed and a few
edges curved (curve nodes at GLL parameters, endpoints on the vertices):
a 5x4 quad mesh (P = 3, 5) and a 3x3 triangle mesh (P = 3).  Stored: the
MeshGraph tables (verts, segs, faces, domain element order, curves) and the
reference build_elements GeomFactors (weights_world, inv) per element.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from spechp.meshio import structured_quad_mesh, structured_tri_mesh  # noqa: E402
from spechp.quadrature import PointsKey, PointsType, make_rule  # noqa: E402
from spechp.region import build_elements  # noqa: E402

out = {}


def perturb_and_curve(mesh, amp, curved, seed):
    rng = np.random.default_rng(seed)
    xs = np.array([v[0] for v in mesh.verts.values()])
    ys = np.array([v[1] for v in mesh.verts.values()])
    x0, x1, y0, y1 = xs.min(), xs.max(), ys.min(), ys.max()
    for vid, (x, y, z) in list(mesh.verts.items()):
        if x0 < x < x1 and y0 < y < y1:  # interior vertices only
            mesh.verts[vid] = (x + amp * rng.uniform(-1, 1), y + amp * rng.uniform(-1, 1), z)
    for sid, nn in curved:
        a, b = mesh.segs[sid]
        pa, pb = np.array(mesh.verts[a][:2]), np.array(mesh.verts[b][:2])
        t = 0.5 * (make_rule(PointsKey(nn, PointsType.GAUSS_LOBATTO_LEGENDRE)).points + 1.0)
        d = pb - pa
        nrm = np.array([-d[1], d[0]]) / np.linalg.norm(d)
        pts = pa[None, :] + t[:, None] * d[None, :] + 0.04 * np.sin(np.pi * t)[:, None] * nrm[None, :]
        mesh.curves[sid] = [(float(p[0]), float(p[1]), 0.0) for p in pts]


def dump(tag, mesh, kind, Ps):
    vids = sorted(mesh.verts)
    out[f"{tag}/vert_ids"] = np.array(vids)
    out[f"{tag}/verts"] = np.array([mesh.verts[v] for v in vids])
    sids = sorted(mesh.segs)
    out[f"{tag}/seg_ids"] = np.array(sids)
    out[f"{tag}/segs"] = np.array([mesh.segs[s] for s in sids])
    faces = mesh.quads if kind == "quad" else mesh.tris
    fids = sorted(faces)
    out[f"{tag}/face_ids"] = np.array(fids)
    out[f"{tag}/faces"] = np.array([faces[f] for f in fids])
    out[f"{tag}/elements"] = np.array([eid for k, eid in mesh.elements()])
    out[f"{tag}/curve_ids"] = np.array(sorted(mesh.curves) or [-1])
    for sid in sorted(mesh.curves):
        out[f"{tag}/curve/{sid}"] = np.array(mesh.curves[sid])
    for P in Ps:
        els = build_elements(mesh, orders=P)
        out[f"{tag}/elem_verts"] = np.stack([e.geom.verts for e in els])
        out[f"{tag}/P{P}/wj"] = np.stack([e.gf.weights_world for e in els])
        out[f"{tag}/P{P}/inv"] = np.stack([e.gf.inv for e in els])
    out[f"{tag}/Ps"] = np.array(Ps)


q = structured_quad_mesh(5, 4)
perturb_and_curve(q, 0.03, [(0, 4), (7, 3), (12, 5)], 1)
dump("quad", q, "quad", [3, 5])
t = structured_tri_mesh(3, 3)
perturb_and_curve(t, 0.04, [(0, 3), (5, 4)], 2)
dump("tri", t, "tri", [3])

path = Path(__file__).resolve().parent / "reference_mesh.npz"
np.savez_compressed(path, **out)
print(f"wrote {path} ({path.stat().st_size / 1024:.0f} KB, {len(out)} arrays)")
