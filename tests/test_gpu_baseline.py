"""GPU parity at the BASELINE.json sizes (cfg1-cfg5), against the oracle.

Every configuration is applied by the CUDA path at its full stated size and
compared with the CPU oracle (tests/helpers.py tolerances: relative L2 <
1e-12, max-abs / max < 1e-11):

  cfg1  32^2 affine quads P=4: BwdTrans, IProductWRTBase — every element
  cfg2  256^2 curved quads P=6: PhysDeriv, Helmholtz — every element
  cfg3  64^3 affine hexes P=4: BwdTrans, IProductWRTBase, PhysDeriv —
        every element (oracle chunked over a process pool)
  cfg4  64^3 deformed periodic hexes, P=2..8: the fused local Helmholtz on
        the whole mesh, 8192 elements checked (first and last 2048 — the
        first and last tiles of every CTA schedule — and 4096 random);
        the assembled apply (default class-range algorithm, the benchmarked path)
        checked exactly on the global dofs of 48 sampled elements (their
        values need only the 27-element neighbourhoods); at P=4 the whole
        assembled vector against a chunked oracle
  cfg5  48^3 variable order P in {3..7}: the whole assembled vector

The oracle is test infrastructure; it only checks the CUDA results.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

from helpers import assert_parity
from oracle import assembly as oa
from oracle import geometry as og
from oracle import ops as oo

pytestmark = [pytest.mark.gpu,
              pytest.mark.filterwarnings("ignore:This process .* is multi-threaded:DeprecationWarning")]
torch = pytest.importorskip("torch")

SEED = int(os.environ.get("SPECHP_SEED", "20240801"))
WORKERS = max(1, min(16, (os.cpu_count() or 2)))


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1906_03489_b200 as sp

    return sp


# ---------------------------------------------------------------------------
# oracle workers (fork pool: numpy only in the children)
# ---------------------------------------------------------------------------
def _oracle_chunk(args):
    kind, shape, P, Q, n, ids, mapping, amp, data, lam = args
    oe = oo.Expansion(shape, P, Q)
    _, _, inv, wj = og.factors(oe, n, ids, mapping, amp)
    if kind == "helmholtz":
        return oo.helmholtz(oe, data, lam, oo.metric_from_inv(wj, inv), wj)
    if kind == "bwdtrans":
        return oo.bwd(oe, data)
    if kind == "iproductwrtbase":
        return oo.iprod(oe, data, wj)
    if kind == "physderiv":
        return oo.physderiv(oe, data, inv)
    raise ValueError(kind)


def _pool_apply(kind, shape, P, Q, n, ids, mapping, amp, data, lam=1.0, chunk=8192):
    ids = np.asarray(ids)
    jobs = [(kind, shape, P, Q, n, ids[s:s + chunk], mapping, amp, data[s:s + chunk], lam)
            for s in range(0, ids.size, chunk)]
    if len(jobs) == 1 or WORKERS == 1:
        return np.concatenate([_oracle_chunk(j) for j in jobs])
    with mp.get_context("fork").Pool(min(WORKERS, len(jobs))) as pool:
        return np.concatenate(pool.map(_oracle_chunk, jobs))


def _assemble_ref(codes, yl, ng):
    """assemble (assembly.py:141-147): signed sum in element order; every
    structured-grid code is a gid (+1) or pinned (-1)."""
    ok = codes >= 0
    return np.bincount(codes[ok], weights=yl[ok], minlength=ng)


def _gather(codes, x):
    return np.where(codes >= 0, x[np.maximum(codes, 0)], 0.0)


# ---------------------------------------------------------------------------
# 2D: cfg1, cfg2 (every element)
# ---------------------------------------------------------------------------
def test_cfg1_full(sp):
    n, P, Q = 32, 4, 6
    E = n * n
    exp = sp.make_quad(P, Q)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_AFFINE)
    rng = np.random.default_rng(SEED)
    ids = np.arange(E)
    for op, size in (("bwdtrans", (P + 1) ** 2), ("iproductwrtbase", Q * Q)):
        x = rng.uniform(-1, 1, (E, size))
        coll = sp.Collection(batch, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
        got = coll.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
        ref = _oracle_chunk((op, "quad", P, Q, n, ids, og.MAP_AFFINE, 0.0, x, 1.0))
        assert_parity(got, ref, what=f"cfg1 {op}")


def test_cfg2_full(sp):
    n, P, Q = 256, 6, 8
    E = n * n
    exp = sp.make_quad(P, Q)
    rng = np.random.default_rng(SEED)
    ids = np.arange(E)
    u = rng.uniform(-1, 1, (E, Q * Q))
    bp = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_POINT, mapping=sp.MAP_QUAD_SINE, amp=0.05)
    got = sp.Collection(bp, sp.OperatorKind.PHYS_DERIV, sp.Strategy.CUDA_SUMFAC).apply(
        torch.as_tensor(u, device="cuda")).cpu().numpy()
    ref = _pool_apply("physderiv", "quad", P, Q, n, ids, og.MAP_QUAD_SINE, 0.05, u)
    assert_parity(got, ref, what="cfg2 physderiv")
    c = rng.uniform(-1, 1, (E, (P + 1) ** 2))
    bm = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_QUAD_SINE, amp=0.05)
    got = sp.Collection(bm, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC, lam=1.0).apply(
        torch.as_tensor(c, device="cuda")).cpu().numpy()
    ref = _pool_apply("helmholtz", "quad", P, Q, n, ids, og.MAP_QUAD_SINE, 0.05, c)
    assert_parity(got, ref, what="cfg2 helmholtz")


# ---------------------------------------------------------------------------
# cfg3: 64^3 affine hexes, every element
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("op", ["bwdtrans", "iproductwrtbase", "physderiv"])
def test_cfg3_full(sp, op):
    n, P, Q = 64, 4, 6
    E = n ** 3
    exp = sp.make_hex(P, Q)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_AFFINE)
    size = (P + 1) ** 3 if op == "bwdtrans" else Q ** 3
    x = np.random.default_rng(SEED).standard_normal((E, size))
    coll = sp.Collection(batch, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
    got = coll.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
    ref = _pool_apply(op, "hex", P, Q, n, np.arange(E), og.MAP_AFFINE, 0.0, x, chunk=16384)
    assert_parity(got, ref.reshape(got.shape), what=f"cfg3 {op} 64^3")


# ---------------------------------------------------------------------------
# cfg4: 64^3 deformed periodic hexes, P = 2..8
# ---------------------------------------------------------------------------
def _cfg4(sp, P, n=64):
    exp = sp.make_hex(P, P + 2)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC, lam=1.0)
    return batch, coll


def _sample_ids(E, rng, k_end=2048, k_mid=4096):
    mid = rng.choice(np.arange(k_end, E - k_end), k_mid, replace=False)
    return np.unique(np.concatenate([np.arange(k_end), np.arange(E - k_end, E), mid]))


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7, 8])
def test_cfg4_local_helmholtz_64(sp, P):
    n = 64
    E = n ** 3
    batch, coll = _cfg4(sp, P, n)
    rng = np.random.default_rng(SEED + P)
    c = torch.empty((E, (P + 1) ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    y = coll.apply(c)
    ids = _sample_ids(E, rng)
    idt = torch.as_tensor(ids, device="cuda")
    got = y.index_select(0, idt).cpu().numpy()
    cs = c.index_select(0, idt).cpu().numpy()
    del c, y
    ref = _pool_apply("helmholtz", "hex", P, P + 2, n, ids, og.MAP_HEX_SINE, 0.03, cs, chunk=1024)
    assert_parity(got, ref, what=f"cfg4 local P{P} 64^3 ({ids.size} sampled elements)")


def _neighbourhood(n, sample):
    """Elements sharing a vertex with any sampled element (periodic)."""
    ex, ey, ez = sample % n, (sample // n) % n, sample // (n * n)
    out = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                out.append(((ex + dx) % n) + n * (((ey + dy) % n) + n * ((ez + dz) % n)))
    return np.unique(np.concatenate(out))


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7, 8])
def test_cfg4_assembled_64_sampled(sp, P):
    """The benchmarked assembled apply (64^3, default algorithm) on every P:
    y is exact on the dofs of 48 sampled elements given the oracle's local
    outputs of their neighbourhoods; the map is the oracle's numbering."""
    n = 64
    E = n ** 3
    batch, coll = _cfg4(sp, P, n)
    amap = sp.AssemblyMap.hex_periodic(n, P)
    assert amap.algorithm == "class"
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    ng = amap.num_global
    x = np.random.default_rng(SEED + 10 * P).uniform(-1, 1, ng)
    y = op.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
    _, _, codes = oa.hex_periodic_codes(n, P)
    codes = codes.reshape(E, -1)
    rng = np.random.default_rng(P)
    sample = np.unique(np.concatenate([[0, 1, n - 1, E - n, E - 1],
                                       rng.choice(E, 43, replace=False)]))
    nb = _neighbourhood(n, sample)
    yl = _pool_apply("helmholtz", "hex", P, P + 2, n, nb, og.MAP_HEX_SINE, 0.03,
                     _gather(codes[nb], x), chunk=512)
    yref = _assemble_ref(codes[nb], yl, ng)
    dofs = np.unique(codes[sample])
    assert_parity(y[dofs], yref[dofs], what=f"cfg4 assembled P{P} 64^3 ({dofs.size} dofs)")


@pytest.mark.parametrize("alg", ["class", "split"])
def test_cfg4_assembled_64_full_p4(sp, alg):
    """The headline apply (P=4, 64^3; class = the default and benchmarked
    algorithm, split its fallback) against the whole oracle vector."""
    n, P = 64, 4
    E = n ** 3
    batch, coll = _cfg4(sp, P, n)
    amap = sp.AssemblyMap.hex_periodic(n, P).set_algorithm(alg)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    ng = amap.num_global
    x = np.random.default_rng(SEED).uniform(-1, 1, ng)
    y = op.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
    _, _, codes = oa.hex_periodic_codes(n, P)
    codes = codes.reshape(E, -1)
    yl = _pool_apply("helmholtz", "hex", P, P + 2, n, np.arange(E), og.MAP_HEX_SINE, 0.03,
                     _gather(codes, x), chunk=8192)
    yref = _assemble_ref(codes, yl, ng)
    assert_parity(y, yref, what=f"cfg4 assembled P4 64^3 (full vector, {alg})")


# ---------------------------------------------------------------------------
# cfg5: 48^3 variable order, whole assembled vector
# ---------------------------------------------------------------------------
def test_cfg5_assembled_48_full(sp):
    from paper_1906_03489_b200 import configs

    n = 48
    orders = configs.cfg5_orders()
    ng, maps = sp.hex_variable_maps(n, orders)
    batches = []
    for P, (ids, amap) in maps.items():
        exp = sp.make_hex(P, P + 2)
        bb = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE,
                                        amp=0.03, elem_ids=ids)
        batches.append((sp.Collection(bb, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC), amap))
    op = sp.GlobalHelmholtz(batches, ng)
    x = np.random.default_rng(SEED).uniform(-1, 1, ng)
    y = op.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
    rng_, off, codes = oa.hex_periodic_codes(n, orders)
    assert rng_ == ng
    yref = np.zeros(ng)
    for P in sorted(set(orders.tolist())):
        ids = np.nonzero(orders == P)[0]
        m3 = (P + 1) ** 3
        rows = codes[(off[ids][:, None] + np.arange(m3)[None, :])]
        yl = _pool_apply("helmholtz", "hex", P, P + 2, n, ids, og.MAP_HEX_SINE, 0.03,
                         _gather(rows, x), chunk=2048)
        yref += _assemble_ref(rows, yl, ng)
    assert_parity(y, yref, what="cfg5 assembled 48^3 variable order (full vector)")
