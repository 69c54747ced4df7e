"""Mesh ingestion into device batches: element vertex
gathering on the host, the coordinate map and geometric factors on the
device, against the reference's build_elements GeomFactors
(tests/golden/make_golden_mesh.py): perturbed quad and triangle meshes with
curved edges."""
import numpy as np
import pytest

from mesh_duck import DuckMesh, G
from paper_1906_03489_b200 import mesh as M

CASES = [("quad", "quad", 3), ("quad", "quad", 5), ("tri", "tri", 3)]


@pytest.mark.parametrize("tag,kind", [("quad", "quad"), ("tri", "tri")])
def test_element_coordinates_match_reference(tag, kind):
    ids, verts, curves = M.element_coordinates(DuckMesh(tag, kind), kind)
    assert np.array_equal(verts, G[f"{tag}/elem_verts"])
    assert len(curves) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("tag,kind,P", CASES)
def test_mesh_geometry_matches_reference(tag, kind, P):
    import paper_1906_03489_b200 as sp

    ids, batch = M.mesh_batch(DuckMesh(tag, kind), P, kind=kind, geom_kind=sp.GEOM_POINT)
    g = batch.geometry.cpu().numpy()
    E, npts = G[f"{tag}/P{P}/wj"].shape
    cs = (npts + 1) & ~1
    wj = g[:, :npts]
    inv = np.stack([g[:, (1 + c) * cs:(1 + c) * cs + npts] for c in range(4)], axis=-1).reshape(E, npts, 2, 2)
    for got, ref in ((wj, G[f"{tag}/P{P}/wj"]), (inv, G[f"{tag}/P{P}/inv"])):
        err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
        assert err < 1e-12, err


@pytest.mark.gpu
def test_mesh_geometry_rejects_inverted_element():
    import paper_1906_03489_b200 as sp

    exp = sp.make_quad(3)
    verts = np.array([[[0, 0], [1, 0], [1, 1], [0, 1]], [[0, 0], [0, 1], [1, 1], [1, 0]]], float)
    with pytest.raises(sp.geometry.GeometryError, match="element 11: non-positive Jacobian"):
        M.geometry_from_vertices(exp, verts, ids=[10, 11])
