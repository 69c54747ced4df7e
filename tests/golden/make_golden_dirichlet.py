"""Reference Helmholtz solve with NON-ZERO Dirichlet data (the lifting
branch of helmholtz_solve, assembly.py:274-354), for the device solver's
parity test.

    python tests/golden/make_golden_dirichlet.py -> tests/golden/reference_dirichlet.npz

4 x 4 structured quads on [0,1]^2, -lap u + lam u = f with the exact
solution u = exp(x) cos(y) + x y (so f = lam u and the boundary data are the
trace of u), Dirichlet on all four sides (and on south/west only, Neumann
data then being absent: the weak form's natural condition, solved as-is by
both sides), orders P = 2..6.  Stored per case: the lifted boundary vector
u_d (dirichlet_values), the global solution, the assembled load b, and the
reference's L2 error of the solution.
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from spechp.assembly import (assemble, build_assembly_map, dirichlet_values,  # noqa: E402
                             helmholtz_solve)
from spechp.geometry import integral_world, iproduct_world, x_map  # noqa: E402
from spechp.meshio import structured_quad_mesh  # noqa: E402
from spechp.region import build_elements  # noqa: E402
from spechp.stdregions import bwd_trans  # noqa: E402

LAM = 1.0


def exact(x, y):
    return np.exp(x) * np.cos(y) + x * y


out = {}
for sides in (("south", "east", "north", "west"), ("south", "west")):
    tag = "all" if len(sides) == 4 else "sw"
    for P in range(2, 7):
        mesh = structured_quad_mesh(4, 4)
        elements = build_elements(mesh, orders=P)
        forcing = []
        for el in elements:
            xy = x_map(el.geom, el.exp.points)
            forcing.append(LAM * exact(xy[:, 0], xy[:, 1]))   # -lap(e^x cos y + x y) = 0
        specs = {n: exact for n in sides}
        coeffs, info = helmholtz_solve(mesh, elements, LAM, forcing, specs, tol=1e-13, max_iter=6000)
        amap = info["amap"]
        u_d = dirichlet_values(mesh, amap, specs)
        b = assemble(amap, [iproduct_world(el.exp, el.gf, f) for el, f in zip(elements, forcing)])
        num = den = 0.0
        for el, c in zip(elements, coeffs):
            xy = x_map(el.geom, el.exp.points)
            ex = exact(xy[:, 0], xy[:, 1])
            num += integral_world(el.exp, el.gf, (bwd_trans(el.exp, c) - ex) ** 2)
            den += integral_world(el.exp, el.gf, ex ** 2)
        pre = f"{tag}/P{P}/"
        out[pre + "u_d"] = u_d
        out[pre + "x"] = info["global"]
        out[pre + "b"] = b
        out[pre + "nd"] = np.array(info["num_dirichlet"])
        out[pre + "err"] = np.array(math.sqrt(num / den))
        print(tag, P, info["num_dirichlet"], math.sqrt(num / den))
path = Path(__file__).resolve().parent / "reference_dirichlet.npz"
np.savez_compressed(path, **out)
print("wrote", path)
