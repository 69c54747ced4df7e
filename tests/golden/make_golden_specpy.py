"""Reference outputs of the NekPy-style binding (specpy) for the scripting
layer's parity tests.

    python tests/golden/make_golden_specpy.py -> tests/golden/reference_specpy.npz

The reference's own specpy StdQuadExp (specpy/__init__.py:76-102 over
stdregions.py) is built for (nModes, nPts) in the binding tests' pairs and
FwdTrans / BwdTrans / IProductWRTBase-free Integral are evaluated on seeded
inputs (FwdTrans = the Galerkin projection of stdregions.py:484-498).
"""
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/specpy/src")

import specpy as rs  # noqa: E402

SEED = 20240801
out = {}
for nmodes, npts in ((3, 4), (4, 5), (4, 6), (6, 7), (8, 9), (8, 10)):
    pk = rs.PointsKey(npts, rs.PointsType.GaussLobattoLegendre)
    bk = rs.BasisKey(rs.BasisType.Modified_A, nmodes, pk)
    q = rs.StdQuadExp(bk, bk)
    rng = np.random.default_rng(SEED + 10 * nmodes + npts)
    u = rng.uniform(-1, 1, q.GetTotPoints())
    c = rng.uniform(-1, 1, q.GetNcoeffs())
    pre = f"m{nmodes}q{npts}/"
    out[pre + "phys"] = u
    out[pre + "coeffs"] = c
    out[pre + "fwd"] = np.asarray(q.FwdTrans(u))
    out[pre + "bwd"] = np.asarray(q.BwdTrans(c))
    out[pre + "integral"] = np.array(q.Integral(u))
np.savez_compressed("tests/golden/reference_specpy.npz", **out)
print("wrote", len(out), "arrays")
