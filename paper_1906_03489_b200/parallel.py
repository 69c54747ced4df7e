"""Multi-GPU plumbing: one process per GPU, torch.distributed for the
control plane.

The elemental operators are independent per element, so the hot path
shards by element with no data-path exchange: `shard_range` gives each rank
a contiguous block of element ids (strong scaling) and `bench.py` runs one
independent mesh per rank (weak scaling).  Timings are reduced as the max
over ranks; `replica_checksum` verifies that ranks fed identical inputs
produced bitwise-identical outputs (the kernels are deterministic).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend=None):
    """Initialise the default process group from the environment (no-op for
    a single process).  MASTER_ADDR defaults to 127.0.0.1."""
    rank, world, local = env_world()
    if world == 1 or dist.is_initialized():
        return rank, world, local
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29512")
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(local)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def shard_range(num_elements, rank, world):
    """Contiguous element block [lo, hi) of `rank`; blocks differ in size by at
    most one element and cover 0..num_elements-1 exactly once."""
    base, rem = divmod(int(num_elements), int(world))
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def max_over_ranks(value, device=None):
    """Max of a scalar over all ranks (the benchmark's step time)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_checksum(tensor):
    """(min, max) over ranks of a bit-level checksum of `tensor`; equal
    values mean every rank holds bitwise-identical data."""
    raw = tensor.detach().contiguous().view(torch.int64)
    h = torch.bitwise_xor(raw, raw.roll(1)).sum(dtype=torch.int64)
    h = h.reshape(1).to(torch.float64) if raw.numel() else torch.zeros(1, dtype=torch.float64,
                                                                       device=tensor.device)
    if not dist.is_initialized() or dist.get_world_size() == 1:
        v = float(h.item())
        return v, v
    lo = h.clone()
    hi = h.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    return float(lo.item()), float(hi.item())
