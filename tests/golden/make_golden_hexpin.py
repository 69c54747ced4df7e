"""Reference outputs that pin the 3D (hex) path by exact Kronecker identities.

The reference has no hexahedra, but on an affine brick
element [0,h]^3 every hex operator factors into the reference's own 2D
(quad, [0,h]^2) and 1D (segment) operators, with the hex index conventions
of this repository (mode (p*m+q)*m+r, point (i*Q+j)*Q+k: 2D index slow, the
third direction fast):

  BwdTrans        B3 = kron(B2, B1)
  IProduct        b  = kron(B2, B1) (kron(W2, W1) * u)
  PhysDeriv       d/dx = kron(Dx2, I), d/dy = kron(Dy2, I), d/dz = kron(I2, (2/h) D1)
  Helmholtz       H3 = kron(K2, M1) + kron(M2, K1) + lam kron(M2, M1)

where B2, W2, M2 = world_mass_matrix, K2 = world_stiffness_matrix and the
world derivative matrices Dx2/Dy2 (reference Collection PHYS_DERIV applied
to the identity) come from the reference's quad element on [0,h]^2, and
B1, w1, D1 from its segment expansion (make_seg), with M1 = B1 diag(w1 h/2)
B1^T and K1 = (2/h) Bd1 diag(w1) Bd1^T the 1D world mass / stiffness.

    python tests/golden/make_golden_hexpin.py   ->  tests/golden/reference_hexpin.npz
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from spechp.collections import Collection, OperatorKind, Strategy  # noqa: E402
from spechp.geometry import world_mass_matrix, world_stiffness_matrix  # noqa: E402
from spechp.meshio import structured_quad_mesh  # noqa: E402
from spechp.region import build_elements  # noqa: E402
from spechp.stdregions import make_seg  # noqa: E402

H = 0.5
LAM = 1.3
out = {"h": np.float64(H), "lam": np.float64(LAM)}
for P in (1, 2, 3, 4, 5, 6, 7, 8):
    Q = P + 2
    mesh = structured_quad_mesh(1, 1, x1=H, y1=H)
    el = build_elements(mesh, orders=P, num_points=Q)[0]
    exp2, gf = el.exp, el.gf
    np2 = exp2.num_points
    # world derivative matrices: column j = PhysDeriv of the j-th unit vector
    cols = [Collection([el], OperatorKind.PHYS_DERIV, Strategy.STD_MAT).apply(np.eye(np2)[j][None, :])[0]
            for j in range(np2)]
    cols = np.stack(cols, axis=-1)          # (2, np2, np2): [a, i, j] = d_a e_j at i
    seg = make_seg(P, num_points=Q)
    B1, w1, D1 = seg.bwd_matrix, seg.weights, seg.deriv_matrices[0]
    Bd1 = seg.deriv_bwd_matrices[0]
    M1 = B1 @ ((w1 * H / 2)[None, :] * B1).T
    K1 = (2.0 / H) * (Bd1 @ (w1[None, :] * Bd1).T)
    pre = f"P{P}/"
    out[pre + "Q"] = np.int64(Q)
    out[pre + "B2"] = exp2.bwd_matrix
    out[pre + "W2"] = gf.weights_world
    out[pre + "M2"] = world_mass_matrix(exp2, gf)
    out[pre + "K2"] = world_stiffness_matrix(exp2, gf)
    out[pre + "Dx2"] = cols[0]
    out[pre + "Dy2"] = cols[1]
    out[pre + "B1"] = B1
    out[pre + "w1"] = w1
    out[pre + "D1"] = D1
    out[pre + "M1"] = 0.5 * (M1 + M1.T)
    out[pre + "K1"] = 0.5 * (K1 + K1.T)

path = Path(__file__).resolve().parent / "reference_hexpin.npz"
np.savez_compressed(path, **out)
print(f"wrote {path} ({path.stat().st_size / 1024:.0f} KB, {len(out)} arrays)")
