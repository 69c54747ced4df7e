"""CPU, world_size 2 over gloo: the multi-process plumbing bench.py uses
(element sharding, max-over-ranks timing, replica checksums), and that an
element-sharded elemental operator reassembles to the unsharded result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1906_03489_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle import geometry as og
    from oracle import ops as oo

    try:
        r, w, _ = parallel.init("gloo")
        out = {}
        # sharding covers every element exactly once
        E = 37
        lo, hi = parallel.shard_range(E, r, w)
        ranges = [None] * w
        dist.all_gather_object(ranges, (lo, hi))
        cover = np.zeros(E, int)
        for a, b in ranges:
            cover[a:b] += 1
        out["cover"] = bool(np.all(cover == 1))
        out["max"] = parallel.max_over_ranks(float(r) * 2.5)
        same = torch.arange(100, dtype=torch.float64) * 0.5
        out["same"] = parallel.replica_checksum(same)
        out["diff"] = parallel.replica_checksum(same + r)
        # sharded elemental Helmholtz == unsharded (hex P=3, deformed map)
        oe = oo.Expansion("hex", 3, 5)
        n = 3
        Et = n ** 3
        ids = np.arange(Et)
        _, _, inv, wj = og.factors(oe, n, ids, og.MAP_HEX_SINE, 0.03)
        G = oo.metric_from_inv(wj, inv)
        c = np.random.default_rng(0).uniform(-1, 1, (Et, oe.nm))
        a, b = parallel.shard_range(Et, r, w)
        part = oo.helmholtz(oe, c[a:b], 1.0, G[a:b], wj[a:b])
        parts = [None] * w
        dist.all_gather_object(parts, part)
        full = np.concatenate(parts)
        ref = oo.helmholtz(oe, c, 1.0, G, wj)
        out["sharded_err"] = float(np.max(np.abs(full - ref)))
        q.put((r, out))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, {"error": repr(exc)}))


@pytest.mark.timeout(120)
def test_gloo_world2_plumbing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
    for r in range(world):
        assert "error" not in res[r], res[r]
        assert res[r]["cover"]
        assert res[r]["max"] == 2.5
        lo, hi = res[r]["same"]
        assert lo == hi
        lo, hi = res[r]["diff"]
        assert lo != hi
        assert res[r]["sharded_err"] == 0.0
