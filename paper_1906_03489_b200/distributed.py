"""Element-sharded assembled Helmholtz over several GPUs.

The periodic n^3 hex mesh is cut into z-slabs, one per rank.  Each rank
renumbers the global dofs its elements touch (sorted by global id), applies
the fused gather -> elemental Helmholtz -> owner-computes sum on its own
elements (explicit local map, one GPU), and then performs the single
exchange step the assembled operator needs: the partial sums on the two
interface planes are swapped with the neighbouring ranks (point-to-point,
NCCL over NVLink on GPUs, gloo on CPUs) and added in rank order, so both
copies of an interface dof are bitwise identical and independent of which
rank computed them.  0.5 MB per neighbour at P=4, n=64 (one z-plane of dofs).
Each rank builds only its slab's rows of the map (the periodic numbering in
closed form, sphp_hexmap_periodic_codes) and its neighbours' adjacent
element layers; the exchange's pack / combine run as our kernels.

Dot products for CG count every dof once (owned = lowest rank touching it)
and are all-reduced.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


def slab_codes(n, P, e0, e1):
    """Rows [e0, e1) of the periodic map's codes (sphp_hexmap_periodic_codes:
    the analytic numbering, no n^3 table)."""
    nm = (P + 1) ** 3
    out = np.empty((e1 - e0, nm), dtype=np.int64)
    _lib.check(_lib.lib.sphp_hexmap_periodic_codes(int(n), int(P), int(e0), int(e1), _lib.ptr(out)))
    return out


class SlabPartition:
    """Rank `rank`'s z-slab of the periodic n^3 grid with order P.  Only the
    slab's own rows of the map are built, plus the one element layer of each
    neighbour that touches it (its interface planes)."""

    def __init__(self, n, P, rank, world):
        if n % world or n // world < 2:
            raise ValueError(f"need n divisible by world with >= 2 layers per rank (n={n}, world={world})")
        self.n, self.P, self.rank, self.world = n, P, rank, world
        nz = n // world
        n2 = n * n
        self.z0, self.z1 = rank * nz, (rank + 1) * nz
        self.e0, self.e1 = self.z0 * n2, self.z1 * n2
        self.num_global_total = (n * P) ** 3
        mine = slab_codes(n, P, self.e0, self.e1)
        self.gids = np.unique(mine)                       # local -> global, sorted
        self.local_codes = np.searchsorted(self.gids, mine).astype(np.int64)
        self.num_local = self.gids.size
        # interface dofs shared with each neighbour rank (ring), sorted by
        # gid: the neighbour's element layer adjacent to this slab (below:
        # its top layer z0 - 1; above: its bottom layer z1)
        below, above = (rank - 1) % world, (rank + 1) % world
        layers = {}
        for nb, z in ((below, (self.z0 - 1) % n), (above, self.z1 % n)):
            if nb == rank:
                continue
            layers.setdefault(nb, []).append(slab_codes(n, P, z * n2, (z + 1) * n2))
        self.shared = {}
        for nb, rows in layers.items():
            theirs = np.unique(np.concatenate([r.ravel() for r in rows]))
            common = np.intersect1d(self.gids, theirs, assume_unique=True)
            self.shared[nb] = np.searchsorted(self.gids, common)
        # ownership for reductions: lowest rank touching the dof
        owner_rank = np.full(self.num_local, rank)
        for nb, idx in self.shared.items():
            owner_rank[idx] = np.minimum(owner_rank[idx], nb)
        self.owned = owner_rank == rank


class DistributedHelmholtz:
    """y = A^T H A x on the sharded mesh.  `local_apply(x_local, y_local)`
    applies the slab's own elements (partial sums on interface dofs);
    defaults to the GPU path built by `from_gpu`."""

    def __init__(self, part: SlabPartition, local_apply, device):
        self.part = part
        self.local_apply = local_apply
        self.device = device
        self._idx = {nb: torch.as_tensor(i, dtype=torch.int64, device=device)
                     for nb, i in part.shared.items()}
        self._owned = torch.as_tensor(part.owned, device=device)

    @classmethod
    def from_gpu(cls, part: SlabPartition, lam=1.0, amp=0.03, device=None, algorithm="split"):
        from . import (GEOM_METRIC, MAP_HEX_SINE, AssemblyMap, Collection, ElementBatch,
                       GlobalHelmholtz, OperatorKind, Strategy, make_hex)
        from .geometry import structured_geometry

        dev = device or torch.device("cuda", torch.cuda.current_device())
        exp = make_hex(part.P, part.P + 2)
        g = structured_geometry(exp, part.n, GEOM_METRIC, MAP_HEX_SINE, amp, e0=part.e0,
                                num_elements=part.e1 - part.e0, device=dev)
        coll = Collection(ElementBatch(exp, part.e1 - part.e0, g, GEOM_METRIC), OperatorKind.HELMHOLTZ,
                          Strategy.CUDA_SUMFAC, lam=lam)
        # split: explicit scatter -> fused operator on the local block ->
        # CSR owner sum (faster than the gathering owner path on slabs)
        amap = AssemblyMap.explicit(part.local_codes, part.num_local).set_algorithm(algorithm)
        op = GlobalHelmholtz([(coll, amap)], part.num_local)
        obj = cls(part, lambda x, y: op.apply(x, y), dev)
        obj._keep = (exp, g, coll, amap, op)
        return obj

    def apply(self, x_local, y_local=None):
        if y_local is None:
            y_local = torch.empty_like(x_local)
        self.local_apply(x_local, y_local)
        self.exchange_add(y_local)
        return y_local

    def exchange_add(self, y_local):
        """The one exchange step: swap interface partial sums with each
        neighbour, add in rank order (identical bits on both sides).  On the
        GPU the pack and the combine are our kernels (sphp_index_gather /
        sphp_index_sum2) and the swap is NCCL point-to-point over NVLink."""
        if not self._idx:
            return y_local
        cuda = y_local.is_cuda
        ops, bufs = [], {}
        for nb, idx in sorted(self._idx.items()):
            send = torch.empty(idx.numel(), dtype=y_local.dtype, device=y_local.device)
            if cuda:
                _lib.check(_lib.lib.sphp_index_gather(idx.numel(), _lib.ptr(idx), _lib.ptr(y_local), _lib.ptr(send),
                                                      _lib.stream_ptr()))
            else:
                torch.index_select(y_local, 0, idx, out=send)
            recv = torch.empty_like(send)
            bufs[nb] = (idx, send, recv)
            ops.append(dist.P2POp(dist.isend, send, nb))
            ops.append(dist.P2POp(dist.irecv, recv, nb))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for nb, (idx, send, recv) in sorted(bufs.items()):
            lo, hi = (recv, send) if nb < self.part.rank else (send, recv)
            if cuda:
                _lib.check(_lib.lib.sphp_index_sum2(idx.numel(), _lib.ptr(idx), _lib.ptr(lo), _lib.ptr(hi),
                                                    _lib.ptr(y_local), _lib.stream_ptr()))
            else:
                y_local.index_copy_(0, idx, lo + hi)
        return y_local

    def dot(self, a, b):
        """Global dot product, every dof counted once."""
        s = torch.sum(torch.where(self._owned, a * b, torch.zeros_like(a)))
        t = s.reshape(1).clone()
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(t)
        return t

    def to_local(self, x_global):
        return x_global[torch.as_tensor(self.part.gids, device=x_global.device)]
