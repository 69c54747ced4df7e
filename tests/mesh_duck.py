"""A minimal object with the reference MeshGraph interface (meshio.py:23-64),
rebuilt from tests/golden/reference_mesh.npz, for the mesh-ingestion tests."""
from pathlib import Path

import numpy as np

G = np.load(Path(__file__).resolve().parent / "golden" / "reference_mesh.npz")


class DuckMesh:
    def __init__(self, tag, kind):
        self.kind = kind
        self.verts = {int(i): tuple(v) for i, v in zip(G[f"{tag}/vert_ids"], G[f"{tag}/verts"])}
        self.segs = {int(i): tuple(int(x) for x in s) for i, s in zip(G[f"{tag}/seg_ids"], G[f"{tag}/segs"])}
        self.faces = {int(i): tuple(int(x) for x in f) for i, f in zip(G[f"{tag}/face_ids"], G[f"{tag}/faces"])}
        self.order = [int(e) for e in G[f"{tag}/elements"]]
        self.curves = {int(c): [tuple(p) for p in G[f"{tag}/curve/{int(c)}"]]
                       for c in G[f"{tag}/curve_ids"] if int(c) >= 0}

    def elements(self):
        return [(self.kind, e) for e in self.order]

    def face_edges(self, kind, eid):
        return self.faces[eid]

    def local_vertices(self, kind, eid):
        """Vertex loop: for edge i, the end not shared with edge i+1 is
        followed by the shared one, so V0 starts edge 0's traversal."""
        pairs = [self.segs[e] for e in self.faces[eid]]
        loop = []
        for i, (a, b) in enumerate(pairs):
            nxt = pairs[(i + 1) % len(pairs)]
            loop.append(a if b in nxt else b)
        return loop
