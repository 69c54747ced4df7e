"""GPU: the device Helmholtz solve against the
reference — assembled diagonal == GlobalSystem.diag, and the reference's own
acceptance problem (test_acceptance.py:93-125: 4x4 quads, -lap u + u = f,
u = sin(pi x) sin(pi y), Dirichlet 0) reproduces the reference's L2 errors
for P = 2..8 (pkg/test_output.txt:12: 4.58e-3 / 2.61e-7 / 3.83e-12)."""
from pathlib import Path
from types import SimpleNamespace as NS

import numpy as np
import pytest

from helpers import assert_parity

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
G = np.load(Path(__file__).resolve().parent / "golden" / "reference_golden.npz")


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1906_03489_b200 as sp

    return sp


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_assembled_diagonal_matches_reference(sp, tag):
    nx, ny = (int(v) for v in G[f"amap/{tag}/shape"])
    orders = G[f"amap/{tag}/orders"]
    dn = tuple(d for d in G[f"amap/{tag}/dirichlet"] if d)
    ng, nd, maps, _ = sp.quad_structured_maps(nx, ny, orders, dn)
    wts_all, inv_all = G[f"amap/{tag}/wts"], G[f"amap/{tag}/inv"]
    po = np.concatenate([[0], np.cumsum((orders + 2) ** 2)])
    batches = []
    for P, (ids, amap) in maps.items():
        exp = sp.make_quad(P)
        els = [NS(exp=exp, gf=sp.GeomFactors(None, None, inv_all[4 * po[e]:4 * po[e + 1]].reshape(-1, 2, 2),
                                              wts_all[po[e]:po[e + 1]])) for e in ids]
        batches.append((sp.Collection(els, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC, lam=1.0),
                        amap))
    diag = sp.assembled_diagonal(batches, ng)
    assert_parity(diag.cpu().numpy(), G[f"amap/{tag}/diag"], what=f"diag {tag}")


def _solve_acceptance(sp, P, tol=1e-13):
    from oracle import geometry as og
    from oracle import ops as oo

    n = 4
    E = n * n
    ng, nd, maps, _ = sp.quad_structured_maps(n, n, P, ("south", "east", "north", "west"))
    ids, amap = maps[P]
    exp = sp.make_quad(P)                                   # reference default Q = P + 2
    helm = sp.Collection(sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC), sp.OperatorKind.HELMHOLTZ,
                         sp.Strategy.CUDA_SUMFAC, lam=1.0)
    ipb = sp.Collection(sp.ElementBatch.structured(exp, n, kind=sp.GEOM_POINT),
                        sp.OperatorKind.IPRODUCT_WRT_BASE, sp.Strategy.CUDA_SUMFAC)
    bwd = sp.Collection(sp.ElementBatch.standard(exp, E), sp.OperatorKind.BWD_TRANS, sp.Strategy.CUDA_SUMFAC)
    oe = oo.Expansion("quad", P, P + 2)
    X = og.world_points(oe, n, np.arange(E))
    exact = np.sin(np.pi * X[..., 0]) * np.sin(np.pi * X[..., 1])
    f = torch.as_tensor((2 * np.pi ** 2 + 1.0) * exact, device="cuda")
    b = sp.assemble(amap, ipb.apply(f))                      # iproduct_world + assemble
    solver = sp.HelmholtzSolver([(helm, amap)], ng, nd)
    x = solver.solve(b, tol=tol, max_iter=6000)
    u = bwd.apply(sp.scatter(amap, x)).cpu().numpy()         # scatter + bwd_trans
    _, _, _, wj = og.factors(oe, n, np.arange(E))
    err = np.sqrt(np.sum(wj * (u - exact) ** 2) / np.sum(wj * exact ** 2))
    return err, x


@pytest.mark.parametrize("P", range(2, 9))
def test_spectral_convergence_matches_reference(sp, P):
    err, _ = _solve_acceptance(sp, P)
    ref = G["helm_conv/errors"][P - 2]
    # discretisation error identical up to the CG stopping point
    assert abs(err - ref) <= max(1e-3 * ref, 2e-13), (P, err, ref)


def test_solve_bitwise_reproducible(sp):
    _, x1 = _solve_acceptance(sp, 5)
    _, x2 = _solve_acceptance(sp, 5)
    assert x1.cpu().numpy().tobytes() == x2.cpu().numpy().tobytes()


def test_pcg_raises_convergence_error(sp):
    n = 64
    rhs = torch.ones(n, dtype=torch.float64, device="cuda")
    diag = torch.ones_like(rhs)

    def apply(p, out):
        out.copy_(p * torch.arange(1, n + 1, dtype=torch.float64, device="cuda"))
        return out

    x = sp.solve_pcg(apply, rhs, tol=1e-12, max_iter=200, diag=diag)
    assert torch.allclose(x, 1.0 / torch.arange(1, n + 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(sp.ConvergenceError) as ei:
        sp.solve_pcg(apply, rhs, tol=1e-14, max_iter=3, diag=diag)
    assert len(ei.value.residuals) == 4


GD = np.load(Path(__file__).resolve().parent / "golden" / "reference_dirichlet.npz")


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("tag", ["all", "sw"])
@pytest.mark.parametrize("P", range(2, 7))
def test_nonzero_dirichlet_lifting_matches_reference(sp, P, tag, graph):
    """The lifting branch of helmholtz_solve (assembly.py:316-354) with
    non-zero boundary data: b_free = b - A u_d, CG on the free block, the
    Dirichlet block set to u_d.  Inputs are the reference's own load vector
    and lifted boundary values (tests/golden/make_golden_dirichlet.py); the
    device solve (host-checked every 8 iterations, or replayed from one CUDA
    graph) reproduces the reference's global solution."""
    pre = f"{tag}/P{P}/"
    sides = ("south", "east", "north", "west") if tag == "all" else ("south", "west")
    ng, nd, maps, _ = sp.quad_structured_maps(4, 4, P, sides)
    assert nd == int(GD[pre + "nd"]) and ng == GD[pre + "x"].size
    ids, amap = maps[P]
    exp = sp.make_quad(P)
    helm = sp.Collection(sp.ElementBatch.structured(exp, 4, kind=sp.GEOM_METRIC), sp.OperatorKind.HELMHOLTZ,
                         sp.Strategy.CUDA_SUMFAC, lam=1.0)
    solver = sp.HelmholtzSolver([(helm, amap)], ng, nd)
    b = torch.as_tensor(GD[pre + "b"], device="cuda")
    ud = torch.as_tensor(GD[pre + "u_d"], device="cuda")
    x = solver.solve(b, u_dirichlet=ud, tol=1e-13, max_iter=6000, graph=graph).cpu().numpy()
    ref = GD[pre + "x"]
    assert np.array_equal(x[:nd], ref[:nd])
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref), (P, tag)


def test_device_scalar_cg_matches_host_scalar_loop(sp):
    """The device-scalar CG (alpha, beta, residual test in the kernels)
    converges to the per-iteration host loop's solution (the reductions'
    summation orders differ, so to rounding)."""
    n = 200
    rng = np.random.default_rng(0)
    d = torch.as_tensor(rng.uniform(1, 10, n), device="cuda")
    rhs = torch.as_tensor(rng.standard_normal(n), device="cuda")

    def apply(p, out):
        out.copy_(d * p)
        out[1:] += 0.3 * p[:-1]
        out[:-1] += 0.3 * p[1:]
        return out

    x = sp.solve_pcg(apply, rhs, tol=1e-13, max_iter=500, diag=d)
    # host loop, same kernels' arithmetic (assembly.py:218-266)
    xh = torch.zeros_like(rhs)
    dinv = 1.0 / d
    r = rhs.clone()
    z = dinv * r
    p = z.clone()
    rz = float((r * z).sum())
    rn = float(torch.sqrt((r * r).sum()))
    ap = torch.empty_like(p)
    for _ in range(500):
        apply(p, ap)
        alpha = rz / float((p * ap).sum())
        xh += alpha * p
        r -= alpha * ap
        z = dinv * r
        rz_new = float((r * z).sum())
        if float(torch.sqrt((r * r).sum())) / rn <= 1e-13:
            break
        p = z + (rz_new / rz) * p
        rz = rz_new
    assert torch.allclose(x, xh, rtol=0, atol=1e-12 * float(xh.abs().max()))
