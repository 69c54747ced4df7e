"""CPU (no GPU): the C-ABI library loads and exports every symbol of
include/spechp_b200.h; its host-side logic — tables, keys, assembly-map
numbering, error wording — matches the reference (golden fixtures) and the
oracle bit for bit where integer."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1906_03489_b200 as sp
from paper_1906_03489_b200 import _lib
from oracle import assembly as oa

ROOT = Path(__file__).resolve().parent.parent
G = np.load(ROOT / "tests" / "golden" / "reference_golden.npz")


def test_library_exports_every_declared_symbol():
    hdr = (ROOT / "include" / "spechp_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(sphp_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert declared == set(_lib.EXPORTED)
    assert _lib.abi_version() == 1


def test_hex_helmholtz_plan_query():
    """sphp_hex_helmholtz_plan: one of the three stage plans for every fast
    key (Q = M + 1 or M + 2, M = 2..9), -1 elsewhere; the BASELINE orders
    P = 2..5 (Q = P + 2) run the i-column plan."""
    plan = _lib.lib.sphp_hex_helmholtz_plan
    for m in range(2, 10):
        for q in (m + 1, m + 2):
            assert plan(m, q) in (0, 1, 3), (m, q)
    assert [plan(p + 1, p + 2) for p in (2, 3, 4, 5)] == [3, 3, 3, 3]
    assert plan(7, 8) == 1 and plan(9, 10) == 0
    assert plan(5, 9) == -1 and plan(12, 13) == -1 and plan(1, 2) == -1


def test_fast_divn_identity():
    """The class launch's fast_divn (pipeline.cuh): q = umulhi(x, floor(2^32 / n))
    is x // n or one less, so one correction step gives the exact quotient
    and remainder — for every mesh size the maps accept (n <= 1024) and
    every element index below 2^31 (edges of each quotient bucket included)."""
    rng = np.random.default_rng(7)
    for n in list(range(2, 130)) + [255, 256, 257, 511, 512, 1000, 1023, 1024]:
        magic = (1 << 32) // n
        top = min(n ** 3, 2 ** 31 - 1)
        x = np.concatenate([rng.integers(0, top, 4000), np.arange(0, min(top, 4 * n)),
                            np.arange(n, top, max(1, top // 2000)) - 1,
                            np.arange(n, top, max(1, top // 2000)), [top - 1, top]]).astype(np.uint64)
        q = (x * np.uint64(magic)) >> np.uint64(32)
        r = x - q * np.uint64(n)
        assert np.all((q == x // np.uint64(n)) | (q + np.uint64(1) == x // np.uint64(n))), n
        fix = r >= n
        q, r = q + fix, r - fix * np.uint64(n)
        assert np.array_equal(q, x // np.uint64(n)) and np.array_equal(r, x % np.uint64(n)), n


def test_autotune_roofline_peak_source():
    """hbm_peak_gbs(): SPHP_HBM_PEAK_GBS overrides; otherwise the driver's
    MEASURED_PEAKS.json at the repository root, else the 8 TB/s nominal."""
    import os
    from paper_1906_03489_b200.collections import hbm_peak_gbs
    old = os.environ.pop("SPHP_HBM_PEAK_GBS", None)
    try:
        gbs, kind = hbm_peak_gbs()
        assert kind in ("measured", "nominal") and 1000.0 < gbs <= 8000.0
        os.environ["SPHP_HBM_PEAK_GBS"] = "7000"
        assert hbm_peak_gbs() == (7000.0, "env")
    finally:
        os.environ.pop("SPHP_HBM_PEAK_GBS", None)
        if old is not None:
            os.environ["SPHP_HBM_PEAK_GBS"] = old


def test_library_is_in_tree_sm100a():
    assert _lib.LIB_PATH.parent == ROOT / "paper_1906_03489_b200"
    blob = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in blob or b"sm_100" in blob


@pytest.mark.parametrize("name,ptype,qs", [("gll", sp.PointsType.GAUSS_LOBATTO_LEGENDRE, range(2, 14)),
                                           ("gl", sp.PointsType.GAUSS_LEGENDRE, range(1, 13)),
                                           ("radau", sp.PointsType.GAUSS_RADAU_M_LEGENDRE, range(1, 13))])
def test_native_rules_match_reference(name, ptype, qs):
    for q in qs:
        r = sp.make_rule(sp.PointsKey(q, ptype))
        assert np.max(np.abs(r.points - G[f"tables/{name}/{q}/z"])) < 1e-14
        assert np.max(np.abs(r.weights - G[f"tables/{name}/{q}/w"])) < 1e-14
        D = sp.diff_matrix(r)
        ref = G[f"tables/{name}/{q}/D"]
        assert np.max(np.abs(D - ref)) <= 1e-13 * max(1, np.max(np.abs(ref)))


def test_native_modified_a_matches_reference():
    for P in range(1, 11):
        for q in (P + 1, P + 2, P + 3):
            exp = sp.make_hex(P, q)
            B, Bd = exp.tables[0]
            assert np.max(np.abs(B - G[f"tables/moda/{P}/{q}/B"])) < 1e-14
            assert np.max(np.abs(Bd - G[f"tables/moda/{P}/{q}/Bd"])) < 1e-12


def test_keys_validation_mirrors_reference():
    with pytest.raises(sp.QuadratureError):
        sp.PointsKey(0, sp.PointsType.GAUSS_LEGENDRE)
    with pytest.raises(sp.QuadratureError):
        sp.PointsKey(1, sp.PointsType.GAUSS_LOBATTO_LEGENDRE)
    with pytest.raises(sp.BasisError):
        sp.BasisKey(sp.BasisType.MODIFIED_A, 1, sp.PointsKey(3, sp.PointsType.GAUSS_LOBATTO_LEGENDRE))
    with pytest.warns(UserWarning):
        sp.BasisKey(sp.BasisType.MODIFIED_A, 5, sp.PointsKey(3, sp.PointsType.GAUSS_LOBATTO_LEGENDRE))


def test_expansion_shapes():
    q = sp.make_quad(4)                      # reference default: Q = P + 2
    assert (q.num_modes, q.num_points, q.num_points_dir) == (25, 36, (6, 6))
    h = sp.make_hex(4, 6)
    assert (h.num_modes, h.num_points) == (125, 216)
    assert h.bwd_matrix.shape == (125, 216)
    assert abs(h.weights.sum() - 8.0) < 1e-13


def test_reference_expansion_duck_typing():
    """Elements built by the reference (any object with shape/basis_keys)
    map to the same native key as ours."""
    from types import SimpleNamespace as NS

    from paper_1906_03489_b200.stdregions import native_key

    pk = NS(num_points=6, points_type=NS(value="gauss_lobatto_legendre"))
    bk = NS(num_modes=5, points_key=pk, basis_type=NS(value="modified_a"))
    ref_like = NS(shape=NS(value="quad"), basis_keys=(bk, bk))
    assert native_key(ref_like) == native_key(sp.make_quad(4, 6))


@pytest.mark.parametrize("n,P", [(2, 1), (2, 3), (4, 2), (4, 4), (6, 3)])
def test_periodic_map_bit_exact(n, P):
    am = sp.AssemblyMap.hex_periodic(n, P)
    assert am.num_global == (n * P) ** 3
    assert np.array_equal(am.codes(), oa.pack_map(oa.hex_periodic_map(n, P)))


@pytest.mark.parametrize("n,lo,hi,seed", [(2, 1, 4, 0), (4, 3, 7, 1), (4, 2, 5, 2)])
def test_variable_order_map_bit_exact(n, lo, hi, seed):
    orders = np.random.default_rng(seed).integers(lo, hi + 1, n ** 3)
    ng, off, codes = sp.hex_variable_codes(n, orders)
    om = oa.hex_periodic_map(n, orders)
    assert ng == om.num_global
    for e in range(n ** 3):
        assert np.array_equal(codes[off[e]:off[e + 1]], oa.element_codes(om, e)), e


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_explicit_map_from_reference_roundtrip(tag):
    """The reference's own AssemblyMap (golden) goes through the C ABI
    unchanged: codes round-trip bit-exactly, colours are a valid colouring."""
    nx, ny = (int(v) for v in G[f"amap/{tag}/shape"])
    orders = G[f"amap/{tag}/orders"]
    l2g, sgn = G[f"amap/{tag}/l2g"], G[f"amap/{tag}/signs"]
    ng = int(G[f"amap/{tag}/num_global"])
    # equal-order batches, as the collections require
    off = np.concatenate([[0], np.cumsum((orders + 1) ** 2)])
    for P in sorted(set(orders.tolist())):
        ids = np.nonzero(orders == P)[0]
        rows = np.stack([oa.element_codes(type("M", (), {"local_to_global": [l2g[off[e]:off[e + 1]]],
                                                         "signs": [sgn[off[e]:off[e + 1]]]})(), 0)
                         for e in ids])
        am = sp.AssemblyMap.explicit(rows, ng)
        assert np.array_equal(am.codes(), rows)
        assert 1 <= am.num_colours <= 8


def test_default_assembly_algorithm():
    """Periodic maps default to the class-range algorithm (split at P = 7,
    where it measures faster; owner without bubbles), explicit maps to
    owner; set_algorithm round-trips through the C ABI and class-range
    assembly is refused on explicit maps."""
    assert sp.AssemblyMap.hex_periodic(8, 4).algorithm == "class"
    assert sp.AssemblyMap.hex_periodic(6, 4).algorithm == "class"   # runtime fallback: split
    assert sp.AssemblyMap.hex_periodic(8, 7).algorithm == "class"
    assert sp.AssemblyMap.hex_periodic(8, 1).algorithm == "owner"   # no bubbles
    per = sp.AssemblyMap.hex_periodic(8, 3)
    for alg in ("colour", "split", "owner", "class"):
        assert per.set_algorithm(alg).algorithm == alg
    am = sp.AssemblyMap.explicit(np.array([[0, 1, 2], [2, 3, 0]]), 4)
    assert am.algorithm == "owner"
    for alg in ("colour", "split", "owner"):
        assert am.set_algorithm(alg).algorithm == alg
    with pytest.raises(sp.AssemblyError, match="periodic"):
        am.set_algorithm("class")
    with pytest.raises(KeyError):
        am.set_algorithm("atomic")


def test_explicit_map_rejects_bad_codes():
    with pytest.raises(sp.AssemblyError, match="outside"):
        sp.AssemblyMap.explicit(np.array([[0, 1, 5]]), 5)


def test_collection_errors_before_device_use():
    """Argument errors use the reference's wording (collections.py:63-81)."""
    exp = sp.make_hex(3, 5)
    with pytest.raises(sp.CollectionError, match="strategy must be concrete"):
        sp.Collection(sp.ElementBatch.standard(exp, 4), sp.OperatorKind.BWD_TRANS, sp.Strategy.AUTO)
    with pytest.raises(sp.CollectionError, match="reference CPU path"):
        sp.Collection(sp.ElementBatch.standard(exp, 4), sp.OperatorKind.BWD_TRANS, sp.Strategy.SUM_FAC)
    with pytest.raises(sp.CollectionError, match="empty element group"):
        sp.Collection([], sp.OperatorKind.BWD_TRANS, sp.Strategy.CUDA_SUMFAC)
    with pytest.raises(sp.CollectionError, match="heterogeneous"):
        sp.Collection([sp.make_quad(3), sp.make_quad(4)], sp.OperatorKind.BWD_TRANS,
                      sp.Strategy.CUDA_SUMFAC)


def test_c_abi_rejects_bad_keys():
    h = C.c_void_p()
    one = C.c_int * 3
    # a triangle needs Modified_B in direction 2 (stdregions.py:83-86)
    rc = _lib.lib.sphp_tables_create(_lib.SHAPE_TRI, one(3, 3, 3), one(4, 4, 4), one(1, 1, 1),
                                     one(0, 0, 0), C.byref(h))
    assert rc == _lib.ERR_BAD_ARG and "collapsed-direction" in _lib.last_error()
    rc = _lib.lib.sphp_tables_create(_lib.SHAPE_HEX, one(3, 3, 3), one(1, 4, 4), one(1, 1, 1),
                                     one(0, 0, 0), C.byref(h))
    assert rc == _lib.ERR_BAD_ARG and "Lobatto" in _lib.last_error()


def test_mac_count_formula():
    """collections.py:250-273 staged counts, generalised."""
    from oracle.ops import mac_count

    assert mac_count("quad", "bwdtrans", "sumfac", 4, 6, 1) == 330
    assert mac_count("quad", "iproductwrtbase", "sumfac", 4, 6, 1) == 366
    assert mac_count("quad", "physderiv", "sumfac", 4, 6, 1, geometry=False) == 432
    assert mac_count("hex", "bwdtrans", "sumfac", 4, 6, 1) == 125 * 6 + 25 * 36 + 5 * 216


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_native_quad_map_matches_reference(tag):
    """sphp_quadmap_structured == the reference's build_assembly_map
    (assembly.py:72-138) on structured_quad_mesh, bit for bit: Dirichlet
    block, min edge order, pinned modes, numbering."""
    nx, ny = (int(v) for v in G[f"amap/{tag}/shape"])
    orders = G[f"amap/{tag}/orders"]
    dn = tuple(d for d in G[f"amap/{tag}/dirichlet"] if d)
    ng, nd, batches, (offsets, codes) = sp.quad_structured_maps(nx, ny, orders, dn)
    assert ng == int(G[f"amap/{tag}/num_global"])
    assert nd == int(G[f"amap/{tag}/num_dirichlet"])
    assert np.array_equal(codes, G[f"amap/{tag}/l2g"])          # signs all +1 / pinned -1
    assert np.array_equal(np.where(codes >= 0, 1.0, 0.0), G[f"amap/{tag}/signs"])
    for P, (ids, amap) in batches.items():
        assert np.all(orders[ids] == P) and amap.nmodes == (P + 1) ** 2
