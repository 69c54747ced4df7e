"""The C-ABI boundary contract (include/spechp_b200.h, collections.py:76-90,
SPEC.md:465, specpy/tests/test_bindings.py:119-164):

* one handle applied concurrently on distinct streams (from distinct host
  threads) gives bitwise the serial results — every apply's scratch lives in
  a per-stream workspace;
* a reserved stream's assembled apply can be captured into a CUDA graph and
  replayed; an unreserved one is refused instead of allocating mid-capture;
* no device or host memory growth over 1e5 applies and over repeated
  create / apply / destroy cycles;
* the specpy scripting layer's FwdTrans / BwdTrans / Integral match the
  reference's own binding (fixture from tests/golden/make_golden_specpy.py).
"""
import threading
import tracemalloc
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_specpy.npz"


@pytest.fixture(scope="module")
def sp():
    import paper_1906_03489_b200 as sp

    return sp


def _helm(sp, n, P, strategy=None):
    exp = sp.make_hex(P, P + 2)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, strategy or sp.Strategy.CUDA_SUMFAC, lam=1.0)
    return batch, coll


@pytest.mark.parametrize("alg", ["class", "split", "owner"])
def test_assembled_concurrent_streams_bitwise(sp, alg):
    n, P = 16, 4
    _, coll = _helm(sp, n, P)
    amap = sp.AssemblyMap.hex_periodic(n, P).set_algorithm(alg)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    rng = np.random.default_rng(7)
    xs = [torch.as_tensor(rng.uniform(-1, 1, amap.num_global), device="cuda") for _ in range(2)]
    ref = [op.apply(x).clone() for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [torch.empty_like(x) for x in xs]

    def run(k):
        with torch.cuda.stream(streams[k]):
            for _ in range(20):
                op.apply(xs[k], outs[k], stream=streams[k])

    threads = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    for k in range(2):
        assert torch.equal(outs[k], ref[k]), f"stream {k} differs from the serial apply"


def test_local_and_stdmat_concurrent_streams_bitwise(sp):
    n, P = 8, 3
    batch, coll = _helm(sp, n, P)
    exp = sp.make_hex(P, P + 2)
    b2 = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_POINT, mapping=sp.MAP_HEX_SINE, amp=0.03)
    ipd = sp.Collection(b2, sp.OperatorKind.IPRODUCT_WRT_BASE, sp.Strategy.CUDA_STDMAT)
    rng = np.random.default_rng(3)
    jobs = []
    for c in (coll, ipd):
        blocks = [torch.as_tensor(rng.uniform(-1, 1, (c.num_elements, c.input_size)), device="cuda")
                  for _ in range(2)]
        jobs.append((c, blocks, [c.apply(b).clone() for b in blocks]))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    for c, blocks, ref in jobs:
        outs = [torch.empty(c.output_shape, dtype=torch.float64, device="cuda") for _ in range(2)]
        for _ in range(10):
            for k in range(2):
                c.apply(blocks[k], outs[k], stream=streams[k])
        torch.cuda.synchronize()
        for k in range(2):
            assert torch.equal(outs[k], ref[k])


@pytest.mark.parametrize("alg", ["class", "split"])
def test_assembled_graph_capture_after_reserve(sp, alg):
    n, P = 16, 4
    _, coll = _helm(sp, n, P)
    amap = sp.AssemblyMap.hex_periodic(n, P).set_algorithm(alg)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    x = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, amap.num_global), device="cuda")
    ref = op.apply(x).clone()
    side = torch.cuda.Stream()
    # not reserved on `side`: capturing its first apply must be refused
    y = torch.empty_like(x)
    g = torch.cuda.CUDAGraph()
    with pytest.raises(sp.AssemblyError, match="not reserved"):
        with torch.cuda.graph(g, stream=side):
            op.apply(x, y, stream=side)
    side2 = torch.cuda.Stream()
    op.reserve(stream=side2)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=side2):
        for _ in range(3):
            op.apply(x, y, stream=side2)
    y.zero_()
    g2.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, ref)


def test_no_memory_growth_over_repeated_applies(sp):
    """1e5 applies of one handle: no device memory and no host memory
    growth (test_bindings.py:152-164)."""
    q = sp.make_quad(4, 6)
    b = sp.ElementBatch.structured(q, 4, kind=sp.GEOM_AFFINE)
    c = sp.Collection(b, sp.OperatorKind.IPRODUCT_WRT_BASE, sp.Strategy.CUDA_SUMFAC)
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (16, 36)), device="cuda")
    y = torch.empty(c.output_shape, dtype=torch.float64, device="cuda")
    for _ in range(1000):
        c.apply(x, y)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    tracemalloc.start()
    base, _ = tracemalloc.get_traced_memory()
    for _ in range(100_000):
        c.apply(x, y)
    torch.cuda.synchronize()
    current, _ = tracemalloc.get_traced_memory()
    tracemalloc.stop()
    free1, _ = torch.cuda.mem_get_info()
    assert current - base < 2_000_000
    assert abs(free0 - free1) < 4 << 20


def test_no_memory_growth_over_create_destroy(sp):
    """Handles (tables, collections, maps, assembled applies with their
    per-stream workspaces) created, applied and destroyed repeatedly
    release their device memory."""
    import gc

    def cycle():
        _, coll = _helm(sp, 4, 3)
        amap = sp.AssemblyMap.hex_periodic(4, 3)
        op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
        x = torch.ones(amap.num_global, dtype=torch.float64, device="cuda")
        op.apply(x)
        del op, coll, amap, x

    for _ in range(20):
        cycle()
    gc.collect()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(300):
        cycle()
    gc.collect()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 16 << 20


@pytest.mark.parametrize("key", ["m3q4", "m4q5", "m4q6", "m6q7", "m8q9", "m8q10"])
def test_specpy_matches_reference_binding(sp, key):
    from paper_1906_03489_b200 import specpy as bp

    g = np.load(GOLDEN)
    nm, nq = (int(v) for v in key[1:].split("q"))
    pk = bp.PointsKey(nq, bp.PointsType.GaussLobattoLegendre)
    bk = bp.BasisKey(bp.BasisType.Modified_A, nm, pk)
    q = bp.StdQuadExp(bk, bk)
    u, c = g[f"{key}/phys"], g[f"{key}/coeffs"]
    fwd = q.FwdTrans(u)
    ref = g[f"{key}/fwd"]
    assert np.max(np.abs(fwd - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(q.BwdTrans(c) - g[f"{key}/bwd"])) <= 1e-13
    assert abs(q.Integral(u) - float(g[f"{key}/integral"])) <= 1e-13
    # projection: FwdTrans(BwdTrans(c)) == c (Modified_A spans the polynomials)
    assert np.max(np.abs(q.FwdTrans(q.BwdTrans(c)) - c)) <= 1e-11


def test_mac_count_matches_reference_cost_model(sp):
    """Native sphp_collection_info MAC counts == the reference's own
    Collection.mac_count() (collections.py:250-273) for every quad / tri
    order, point count, operator, strategy, with and without geometry
    (fixture: tests/golden/make_golden_macs.py)."""
    import json

    rows = json.loads((Path(__file__).resolve().parent / "golden" / "reference_macs.json").read_text())
    strat = {"sumfac": sp.Strategy.CUDA_SUMFAC, "stdmat": sp.Strategy.CUDA_STDMAT}
    cache = {}
    checked = 0
    for r in rows:
        P, (q1, q2), E = r["P"], r["npts"], r["E"]
        if r["shape"] == "quad":
            exp = sp.make_quad(P, q1 if q1 != P + 2 else None)
        else:
            exp = sp.make_tri(P, q1 if q1 != P + 2 else None)
        assert exp.num_points_dir == tuple(r["npts"])
        key = (r["shape"], P, q1, r["geometry"])
        if key not in cache:
            if r["geometry"]:
                n = exp.num_points
                d = 0.5 * np.ones((E, n))
                inv = np.broadcast_to(2.0 * np.eye(2), (E, n, 2, 2)).copy()
                wj = d * 0.5 * np.asarray(exp.weights)[None, :]
                cache[key] = sp.ElementBatch(exp, E, sp.geometry.from_factors(exp, wj, inv, kind=sp.GEOM_POINT),
                                             sp.GEOM_POINT)
            else:
                cache[key] = sp.ElementBatch.standard(exp, E)
        c = sp.Collection(cache[key], sp.OperatorKind(r["op"]), strat[r["strategy"]])
        assert c.mac_count() == r["mac_count"], r
        checked += 1
    assert checked == len(rows) == 336
