"""Device Helmholtz solve: preconditioned CG on the fused assembled operator
(reference `solve_pcg` / `helmholtz_solve`,
assembly.py:218-354).

The operator is `GlobalHelmholtz` (gather -> fused elemental Helmholtz ->
deterministic C0 sum); the Jacobi preconditioner is the assembled diagonal
of the elemental matrices (`GlobalSystem.diag`, assembly.py:208-214),
evaluated on the device by `sphp_helmholtz_diagonal`; the CG vector updates
and dot products are deterministic CUDA kernels (`sphp_cg_*`, fixed
reduction order), so a solve is bitwise reproducible.  Dirichlet dofs are the
leading block of the numbering (assembly.py:89-103): they are pinned by
masking, exactly the reference's restriction to free dofs.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .assembly import AssemblyError, AssemblyMap, GlobalHelmholtz, assemble


class ConvergenceError(RuntimeError):
    """assembly.py:33-36: carries the residual history."""

    def __init__(self, message, residuals):
        super().__init__(message)
        self.residuals = residuals


def _ws(device):
    return torch.empty(int(_lib.lib.sphp_reduction_workspace()), dtype=torch.float64, device=device)


def assembled_diagonal(batches, num_global, device=None):
    """Assembled diagonal of A^T H A over per-order batches (signs square away)."""
    diag = None
    for coll, amap in batches:
        loc = torch.empty((coll.num_elements, amap.nmodes), dtype=torch.float64,
                          device=device or "cuda")
        _lib.check(_lib.lib.sphp_helmholtz_diagonal(coll._handle, _lib.ptr(loc),
                                                    _lib.stream_ptr()))
        part = assemble(amap, loc)
        diag = part if diag is None else diag + part
    return diag


def solve_pcg(apply, rhs, tol=1e-12, max_iter=2000, diag=None):
    """Jacobi-preconditioned CG (assembly.py:218-266) on device vectors.

    apply(p, out) writes A p into out.  Returns x; raises ConvergenceError
    with the residual history when max_iter is reached."""
    if diag is None:
        dinv = torch.ones_like(rhs)
    else:  # inv_diag = 1 / where(diag == 0, 1, diag)   (assembly.py:242)
        dinv = 1.0 / torch.where(diag == 0, torch.ones_like(diag), diag)
    return _solve_with_dinv(apply, rhs, dinv, tol, max_iter)


class HelmholtzSolver:
    """-lap(u) + lam u = f with the first `num_dirichlet` global dofs pinned
    (helmholtz_solve, assembly.py:316-354), on per-order batches
    [(Collection(HELMHOLTZ), AssemblyMap)]."""

    def __init__(self, batches, num_global, num_dirichlet=0):
        self.op = GlobalHelmholtz(batches, num_global)
        self.batches = list(batches)
        self.num_global = int(num_global)
        self.nd = int(num_dirichlet)
        self.diag = assembled_diagonal(self.batches, self.num_global)
        self._buf = torch.empty(self.num_global, dtype=torch.float64, device=self.diag.device)
        self._graph_stream = None

    def _apply_free(self, v, out):
        # A restricted to the free block: Dirichlet entries of the input and
        # of the result are zero (v's Dirichlet part is zero already)
        self.op.apply(v, out)
        out[: self.nd] = 0.0
        return out

    def solve(self, rhs, u_dirichlet=None, tol=1e-12, max_iter=3000, graph=False, check_every=8):
        """rhs: assembled load vector (num_global); u_dirichlet: lifted
        boundary values (num_global, Dirichlet block used) or None (zero).
        graph=True replays chunks of `check_every` CG iterations from one
        CUDA graph (no host work per iteration)."""
        b = rhs.clone()
        if u_dirichlet is not None and self.nd:
            ud = torch.zeros_like(b)
            ud[: self.nd] = u_dirichlet[: self.nd]
            b -= self.op.apply(ud, self._buf)
        b[: self.nd] = 0.0
        diag = self.diag.clone()
        diag[: self.nd] = 0.0
        # zero preconditioner on pinned dofs keeps CG in the free subspace
        dinv = torch.where(diag == 0, torch.zeros_like(diag), 1.0 / torch.where(diag == 0,
                                                                             torch.ones_like(diag), diag))
        cs = None
        if graph:
            if self._graph_stream is None:
                self._graph_stream = torch.cuda.Stream(device=b.device)
                self.op.reserve(stream=self._graph_stream)
            cs = self._graph_stream
        x = _solve_with_dinv(self._apply_free, b, dinv, tol, max_iter, check_every=check_every, graph=cs)
        if u_dirichlet is not None and self.nd:
            x[: self.nd] = u_dirichlet[: self.nd]
        return x


def _solve_with_dinv(apply, rhs, dinv, tol, max_iter, check_every=8, graph=None):
    """solve_pcg with an explicit inverse diagonal (zeros allowed).

    The CG scalars stay on the device (sphp_cg_init_dev / sphp_cg_step_dev:
    alpha = rz / pAp, beta = rz' / rz and the residual test run in the
    update kernels), so the host only looks at the state every
    `check_every` iterations; steps after convergence are no-ops, so x is
    bitwise the per-iteration loop's.  `graph`: a (CUDAGraph, stream)
    factory key — when given, one chunk of `check_every` iterations is
    captured once and replayed (the operator must be reserved on that
    stream, GlobalHelmholtz.reserve)."""
    n = rhs.numel()
    dev = rhs.device
    x, r, z, p, ap = (torch.empty_like(rhs) for _ in range(5))
    st = torch.zeros(int(_lib.lib.sphp_cg_state_size(max_iter)), dtype=torch.float64, device=dev)

    def step(stream=None):
        apply(p, ap)
        _lib.check(_lib.lib.sphp_cg_step_dev(n, _lib.ptr(p), _lib.ptr(ap), _lib.ptr(x), _lib.ptr(r),
                                             _lib.ptr(dinv), _lib.ptr(z), _lib.ptr(st), max_iter,
                                             _lib.stream_ptr(stream)))

    _lib.check(_lib.lib.sphp_cg_init_dev(n, _lib.ptr(rhs), _lib.ptr(dinv), _lib.ptr(x), _lib.ptr(r),
                                         _lib.ptr(z), _lib.ptr(p), _lib.ptr(st), max_iter, float(tol),
                                         _lib.stream_ptr()))
    if float(st[5].item()) == 0.0:
        return x
    chunk = None
    if graph is not None and max_iter >= check_every:
        cs = graph
        cs.wait_stream(torch.cuda.current_stream(dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(check_every):
                step(cs)
        torch.cuda.current_stream(dev).wait_stream(cs)
        chunk = g
    done_iters = 0
    while done_iters < max_iter:
        k = min(check_every, max_iter - done_iters)
        if chunk is not None and k == check_every:
            chunk.replay()
        else:
            for _ in range(k):
                step()
        done_iters += k
        done, iters = st[7:9].tolist()
        if done:
            return x
    iters = int(st[8].item())
    residuals = [1.0] + st[9:9 + iters].tolist()
    raise ConvergenceError(f"PCG did not reach {tol} in {max_iter} iterations "
                           f"(final residual {residuals[-1]:.3e})", residuals)


def quad_structured_maps(nx, ny, orders, dirichlet=()):
    """build_assembly_map (assembly.py:72-138) for structured_quad_mesh(nx, ny)
    on the native library, split into per-order batches.
    Returns (num_global, num_dirichlet, {P: (elem_ids, AssemblyMap)})."""
    import ctypes as C

    orders = np.ascontiguousarray(np.broadcast_to(np.asarray(orders, dtype=np.int32), (nx * ny,)))
    mask = 0
    for name in dirichlet:
        mask |= {"south": 1, "east": 2, "north": 4, "west": 8}[name]
    ng, nd = C.c_int64(), C.c_int64()
    offsets = np.empty(nx * ny + 1, dtype=np.int64)
    codes = np.empty(int(np.sum((orders.astype(np.int64) + 1) ** 2)), dtype=np.int64)
    _lib.check(_lib.lib.sphp_quadmap_structured(nx, ny, _lib.ptr(orders), mask, C.byref(ng),
                                                C.byref(nd), _lib.ptr(offsets), _lib.ptr(codes)),
               AssemblyError)
    out = {}
    for P in sorted(set(int(v) for v in orders)):
        ids = np.nonzero(orders == P)[0]
        nm = (P + 1) ** 2
        rows = np.stack([codes[offsets[e]:offsets[e] + nm] for e in ids])
        out[P] = (ids, AssemblyMap.explicit(rows, ng.value))
    return ng.value, nd.value, out, (offsets, codes)
