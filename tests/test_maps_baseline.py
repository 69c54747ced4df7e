"""Assembly index maps at the BASELINE sizes, bit for bit (CPU).

north_star: "assembly index maps must be bit-exact".  The native periodic
map of cfg4 (64^3, P = 2..8) and the variable-order map of cfg5 (48^3,
P_e in {3..7}) are compared entry by entry with the oracle's numbering of
assembly.py:72-138 (generalised to hex faces).  The oracle's vectorised
numbering (`hex_periodic_codes`) is itself pinned to the element-by-element
restatement (`build_map`) at small n first.
"""
import numpy as np
import pytest

import paper_1906_03489_b200 as sp
from oracle import assembly as oa
from paper_1906_03489_b200 import configs


@pytest.mark.parametrize("n,orders", [
    (2, 1), (2, 3), (3, 2), (4, 4), (4, 5),
    (2, "rand1-4"), (3, "rand2-6"), (4, "rand3-7"), (5, "rand1-3"),
])
def test_vectorised_numbering_equals_build_map(n, orders):
    if isinstance(orders, str):
        lo, hi = (int(v) for v in orders[4:].split("-"))
        orders = np.random.default_rng(n * 10 + lo).integers(lo, hi + 1, n ** 3)
    ng, off, codes = oa.hex_periodic_codes(n, orders)
    om = oa.hex_periodic_map(n, orders)
    assert ng == om.num_global
    ref = np.concatenate([oa.element_codes(om, e) for e in range(n ** 3)])
    assert np.array_equal(off[1:] - off[:-1], [len(c) for c in om.local_to_global])
    assert np.array_equal(codes, ref)


@pytest.mark.parametrize("P", configs.CFG4["orders"])
def test_cfg4_periodic_map_bit_exact(P):
    """cfg4's 64^3 periodic map, the one the benchmarked apply uses."""
    n = configs.CFG4["n"]
    am = sp.AssemblyMap.hex_periodic(n, P)
    ng, off, ref = oa.hex_periodic_codes(n, P)
    assert am.num_global == ng == (n * P) ** 3
    got = am.codes()
    assert got.shape == (n ** 3, (P + 1) ** 3)
    assert np.array_equal(got.reshape(-1), ref)
    del got, ref


def test_cfg5_variable_map_bit_exact():
    """cfg5's 48^3 variable-order map (min rule on edges and faces, pinned
    excess modes) with the bench's own orders."""
    n = configs.CFG5["n"]
    orders = configs.cfg5_orders()
    ng, off, codes = sp.hex_variable_codes(n, orders)
    rng_, roff, ref = oa.hex_periodic_codes(n, orders)
    assert ng == rng_
    assert np.array_equal(off, roff)
    assert np.array_equal(codes, ref)
    # per-order batches keep each element's row intact
    ng2, maps = sp.hex_variable_maps(n, orders)
    assert ng2 == ng
    for P, (ids, amap) in maps.items():
        rows = amap.codes()
        pick = np.linspace(0, ids.size - 1, 64).astype(int)
        for k in pick:
            e = ids[k]
            assert np.array_equal(rows[k], ref[roff[e]:roff[e + 1]])
