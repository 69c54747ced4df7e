"""GPU parity: every operator x shape x order x geometry encoding x strategy
against the CPU oracle (rel L2 < 1e-12, max-abs/max < 1e-11 — the
north-star FP64 tolerance).  Element subsets of odd length exercise partial
tiles and the synchronous (non-TMA) input path."""
import numpy as np
import pytest

from helpers import OPS, assert_parity, input_size, oracle_apply, oracle_geometry

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1906_03489_b200 as sp

    return sp


GEOMS = {  # op -> encodings that op accepts
    "bwdtrans": ("none",),
    "iproductwrtbase": ("none", "affine", "point"),
    "physderiv": ("none", "affine", "point"),
    "iproductwrtderivbase": ("none", "affine", "point"),
    "helmholtz": ("affine", "metric"),
}


def _build(sp, shape, P, Q, n, ids, op, geom, strategy, lam=1.0):
    exp = sp.make_hex(P, Q) if shape == "hex" else sp.make_quad(P, Q)
    kinds = {"affine": sp.GEOM_AFFINE, "point": sp.GEOM_POINT, "metric": sp.GEOM_METRIC}
    if geom == "none":
        if op == "helmholtz":
            raise ValueError
        batch = sp.ElementBatch.standard(exp, len(ids))
        mapping, amp, lengths = 0, 0.0, None
    elif geom == "affine":
        mapping, amp = 0, 0.0
        lengths = [1.0, 2.0, 0.5][: (3 if shape == "hex" else 2)]
        batch = sp.ElementBatch.structured(exp, n, kind=kinds[geom], mapping=mapping,
                                           lengths=lengths, elem_ids=ids)
    else:
        mapping = sp.MAP_HEX_SINE if shape == "hex" else sp.MAP_QUAD_SINE
        amp = 0.03 if shape == "hex" else 0.05
        lengths = None
        batch = sp.ElementBatch.structured(exp, n, kind=kinds[geom], mapping=mapping, amp=amp,
                                           elem_ids=ids)
    opk = sp.OperatorKind(op)
    strat = sp.Strategy(strategy)
    coll = sp.Collection(batch, opk, strat, lam=lam)
    oe, inv, wj = oracle_geometry(shape, P, Q, n, ids, mapping, amp, lengths)
    return coll, oe, inv, wj


CASES = []
for shape, Ps in (("hex", range(1, 9)), ("quad", range(1, 10))):
    for P in Ps:
        for Q in (P + 2, P + 3):
            CASES.append((shape, P, Q))


@pytest.mark.parametrize("shape,P,Q", CASES)
@pytest.mark.parametrize("op", OPS)
def test_sumfac_parity(sp, shape, P, Q, op):
    n = 4 if shape == "hex" else 8
    E = n ** (3 if shape == "hex" else 2)
    rng = np.random.default_rng(1000 * P + Q)
    for geom in GEOMS[op]:
        for ids in (np.arange(E), np.arange(3, 3 + 37 if E >= 40 else E - 3)):
            coll, oe, inv, wj = _build(sp, shape, P, Q, n, ids, op, geom, "cuda_sumfac")
            x = rng.uniform(-1, 1, (len(ids), input_size(op, oe)))
            got = coll.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
            ref = oracle_apply(op, oe, x, inv, wj, geom)
            assert_parity(got.reshape(ref.shape), ref, what=f"{shape} P{P} Q{Q} {op} {geom} E{len(ids)}")


@pytest.mark.parametrize("shape,P", [("hex", 2), ("hex", 4), ("quad", 3), ("quad", 6)])
@pytest.mark.parametrize("op", OPS)
def test_stdmat_parity(sp, shape, P, op):
    n = 3 if shape == "hex" else 6
    E = n ** (3 if shape == "hex" else 2)
    ids = np.arange(E)
    rng = np.random.default_rng(7)
    for geom in GEOMS[op]:
        coll, oe, inv, wj = _build(sp, shape, P, P + 2, n, ids, op, geom, "cuda_stdmat")
        x = rng.standard_normal((E, input_size(op, oe)))
        got = coll.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
        ref = oracle_apply(op, oe, x, inv, wj, geom)
        assert_parity(got.reshape(ref.shape), ref, what=f"stdmat {shape} P{P} {op} {geom}")


def test_host_buffers_roundtrip(sp):
    """numpy in -> numpy out through sphp_apply_host (the e2e C-ABI path)."""
    n, P = 4, 4
    coll, oe, inv, wj = _build(sp, "hex", P, P + 2, n, np.arange(n ** 3), "helmholtz", "metric",
                               "cuda_sumfac")
    x = np.random.default_rng(3).uniform(-1, 1, (n ** 3, oe.nm))
    got = coll.apply(x)
    assert isinstance(got, np.ndarray)
    assert_parity(got, oracle_apply("helmholtz", oe, x, inv, wj, "metric"), what="apply_host")


def test_repeated_apply_bitwise(sp):
    """test_collections.py:193-201: repeated applies are bitwise equal."""
    n, P = 4, 5
    for op in OPS:
        geom = "metric" if op == "helmholtz" else "point" if op != "bwdtrans" else "none"
        coll, oe, _, _ = _build(sp, "hex", P, P + 2, n, np.arange(n ** 3), op, geom, "cuda_sumfac")
        x = torch.as_tensor(np.random.default_rng(5).standard_normal((n ** 3, input_size(op, oe))),
                            device="cuda")
        a = coll.apply(x).cpu().numpy()
        b = coll.apply(x).cpu().numpy()
        assert a.tobytes() == b.tobytes(), op


def test_shape_error_message(sp):
    exp = sp.make_hex(3, 5)
    coll = sp.Collection(sp.ElementBatch.standard(exp, 5), sp.OperatorKind.BWD_TRANS,
                         sp.Strategy.CUDA_SUMFAC)
    with pytest.raises(sp.CollectionError, match=r"block shape \(4, 64\) does not match \(5, 64\)"):
        coll.apply(torch.zeros((4, 64), dtype=torch.float64, device="cuda"))
    with pytest.raises(sp.CollectionError, match="block shape"):
        coll.apply(np.zeros((5, 63)))


def test_zero_input_zero_output(sp):
    exp = sp.make_quad(4, 6)
    for op in OPS:
        if op == "helmholtz":
            continue
        coll = sp.Collection(sp.ElementBatch.standard(exp, 7), sp.OperatorKind(op),
                             sp.Strategy.CUDA_SUMFAC)
        out = coll.apply(np.zeros((7, coll.input_size)))
        assert np.all(out == 0)


@pytest.mark.parametrize("PQ", [(2, 4), (3, 5), (4, 6), (7, 9)])
@pytest.mark.parametrize("op", OPS)
def test_unaligned_and_tiny_inputs(sp, op, PQ):
    """Inputs not 16-byte aligned take the synchronous (non-TMA) load path;
    E = 1 and E = 2 exercise single partial tiles.  Orders cover the skewed
    i-column plan at three tile sizes, the rotated even-M rows (P=3, 7) and
    the K-row plan."""
    shape, (P, Q) = "hex", PQ
    n = 4
    for E in (1, 2, 37):
        ids = np.arange(E)
        geom = "metric" if op == "helmholtz" else ("point" if op != "bwdtrans" else "none")
        coll, oe, inv, wj = _build(sp, shape, P, Q, n, ids, op, geom, "cuda_sumfac")
        isz = input_size(op, oe)
        x = np.random.default_rng(E).uniform(-1, 1, (E, isz))
        buf = torch.zeros(E * isz + 1, dtype=torch.float64, device="cuda")
        view = buf[1:].view(E, isz)          # 8-byte offset: misaligned for TMA
        view.copy_(torch.as_tensor(x, device="cuda"))
        assert view.data_ptr() % 16 == 8
        got = coll.apply(view).cpu().numpy()
        ref = oracle_apply(op, oe, x, inv, wj, geom)
        assert_parity(got.reshape(ref.shape), ref, what=f"unaligned {op} P{P} E{E}")
        # an output not 16-byte aligned: the store loop instead of the TMA
        # bulk write-back, bitwise the same values
        osz = got.size // E
        obuf = torch.zeros(E * osz + 1, dtype=torch.float64, device="cuda")
        oview = obuf[1:].view(got.shape)
        assert oview.data_ptr() % 16 == 8
        coll.apply(view, oview)
        assert np.array_equal(oview.cpu().numpy(), got)


def test_multi_tile_walk_small_grid(sp):
    """Cap the persistent grid (SPHP_MAX_GRID is read once per process, so
    run in a subprocess) and check every operator still matches."""
    import subprocess
    import sys
    code = r"""
import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, torch
import paper_1906_03489_b200 as sp
from helpers import OPS, assert_parity, input_size, oracle_apply, oracle_geometry
from test_gpu_parity import _build
for op in OPS:
    # hex P = 2, 4, 5: the other tile sizes of the i-column plan (Helmholtz only)
    for shape, P in (("hex", 3), ("hex", 6), ("quad", 5)) + ((("hex", 2), ("hex", 4), ("hex", 5)) if op == "helmholtz" else ()):
        n = 4 if shape == "hex" else 8
        E = n ** (3 if shape == "hex" else 2)
        geom = "metric" if op == "helmholtz" else ("point" if op != "bwdtrans" else "none")
        coll, oe, inv, wj = _build(sp, shape, P, P + 2, n, np.arange(E), op, geom, "cuda_sumfac")
        x = np.random.default_rng(P).uniform(-1, 1, (E, input_size(op, oe)))
        got = coll.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
        ref = oracle_apply(op, oe, x, inv, wj, geom)
        assert_parity(got.reshape(ref.shape), ref, what=f"grid-capped {shape} P{P} {op}")
print("ok")
"""
    import os
    env = dict(os.environ, SPHP_MAX_GRID="3")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0 and "ok" in res.stdout, res.stdout + res.stderr
