"""The reference's own cost model, Collection.mac_count() (collections.py:
250-273), for every (shape, order, operator, strategy, geometry) the GPU
collections build, so the native counts (sphp_collection_info) are pinned
to it.

    python tests/golden/make_golden_macs.py -> tests/golden/reference_macs.json
"""
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from spechp.collections import Collection, OperatorKind, Strategy  # noqa: E402
from spechp.geometry import GeomFactors  # noqa: E402
from spechp.stdregions import make_quad, make_tri  # noqa: E402

E = 5
rows = []
for shape, orders, mk in (("quad", range(1, 9), make_quad), ("tri", range(1, 7), make_tri)):
    for P in orders:
        for npts in (None, P + 3):
            exp = mk(P) if npts is None else mk(P, num_points=npts)
            n = exp.num_points
            jac = np.broadcast_to(np.eye(2) * 0.5, (n, 2, 2)).copy()
            det = np.full(n, 0.25)
            gf = GeomFactors(jac, det, np.broadcast_to(np.eye(2) * 2.0, (n, 2, 2)).copy(), exp.weights * det)
            for geo in (False, True):
                els = [SimpleNamespace(exp=exp, gf=gf)] * E if geo else [exp] * E
                for op in (OperatorKind.BWD_TRANS, OperatorKind.IPRODUCT_WRT_BASE, OperatorKind.PHYS_DERIV):
                    for strat in (Strategy.SUM_FAC, Strategy.STD_MAT):
                        c = Collection(els, op, strat)
                        rows.append({"shape": shape, "P": P, "npts": exp.num_points_dir, "geometry": geo,
                                     "op": op.value, "strategy": strat.value, "E": E,
                                     "mac_count": int(c.mac_count())})
path = Path(__file__).resolve().parent / "reference_macs.json"
path.write_text(json.dumps(rows, indent=0))
print(f"wrote {path} ({len(rows)} rows)")
