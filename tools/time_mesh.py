"""Mesh ingestion at cfg2 scale: a 256x256 quad mesh (perturbed interior
vertices) -> device ElementBatch with POINT geometry, P = 6, Q = 8.
Host vertex gathering and the device map/factors are timed separately."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402
from paper_1906_03489_b200 import mesh as M  # noqa: E402


class GridMesh:
    """nx x ny quads with the MeshGraph interface (own numbering)."""

    def __init__(self, nx, ny, amp=0.2, seed=0):
        rng = np.random.default_rng(seed)
        vid = lambda i, j: j * (nx + 1) + i  # noqa: E731
        self.verts = {}
        for j in range(ny + 1):
            for i in range(nx + 1):
                x, y = i / nx, j / ny
                if 0 < i < nx and 0 < j < ny:
                    x += amp / nx * rng.uniform(-1, 1)
                    y += amp / ny * rng.uniform(-1, 1)
                self.verts[vid(i, j)] = (x, y, 0.0)
        self.segs, hseg, vseg = {}, {}, {}
        for j in range(ny + 1):
            for i in range(nx):
                hseg[i, j] = len(self.segs)
                self.segs[hseg[i, j]] = (vid(i, j), vid(i + 1, j))
        for j in range(ny):
            for i in range(nx + 1):
                vseg[i, j] = len(self.segs)
                self.segs[vseg[i, j]] = (vid(i, j), vid(i, j + 1))
        self.quads = {j * nx + i: (hseg[i, j], vseg[i + 1, j], hseg[i, j + 1], vseg[i, j])
                      for j in range(ny) for i in range(nx)}
        self.curves = {}

    def elements(self):
        return [("quad", e) for e in range(len(self.quads))]

    def face_edges(self, kind, eid):
        return self.quads[eid]

    def local_vertices(self, kind, eid):
        pairs = [self.segs[e] for e in self.quads[eid]]
        return [a if b in pairs[(i + 1) % 4] else b for i, (a, b) in enumerate(pairs)]


mesh = GridMesh(256, 256)
exp = sp.make_quad(6)
t0 = time.perf_counter()
ids, verts, curves = M.element_coordinates(mesh, "quad")
t1 = time.perf_counter()
M.geometry_from_vertices(exp, verts[:8], curves)   # warm-up (tables, kernels)
torch.cuda.synchronize()
t2 = time.perf_counter()
g = M.geometry_from_vertices(exp, verts, curves, sp.GEOM_POINT)
torch.cuda.synchronize()
t3 = time.perf_counter()
print(f"65536 quads P=6: host vertex gathering {t1 - t0:.3f} s, device map + factors {1e3 * (t3 - t2):.1f} ms "
      f"(geometry {tuple(g.shape)})")
