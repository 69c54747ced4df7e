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


def _dist_worker(rank, world, port, q, n, P):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle import assembly as oa
    from oracle import geometry as og
    from oracle import ops as oo
    from paper_1906_03489_b200.distributed import DistributedHelmholtz, SlabPartition

    try:
        parallel.init("gloo")
        part = SlabPartition(n, P, rank, world)
        oe = oo.Expansion("hex", P, P + 2)
        ids = np.arange(part.e0, part.e1)
        _, _, inv, wj = og.factors(oe, n, ids, og.MAP_HEX_SINE, 0.03)
        G = oo.metric_from_inv(wj, inv)

        def local_apply(x, y):  # oracle stand-in for the GPU slab operator
            xl = x.numpy()
            loc = xl[part.local_codes]
            yl = oo.helmholtz(oe, loc, 1.0, G, wj)
            out = np.zeros(part.num_local)
            np.add.at(out, part.local_codes.ravel(), yl.ravel())
            y.copy_(torch.as_tensor(out))
            return y

        op = DistributedHelmholtz(part, local_apply, torch.device("cpu"))
        x_global = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, part.num_global_total))
        y_local = op.apply(op.to_local(x_global))
        # reference: full (unsharded) oracle assembled apply
        om = oa.hex_periodic_map(n, P)
        Eall = n ** 3
        _, _, inv_a, wj_a = og.factors(oe, n, np.arange(Eall), og.MAP_HEX_SINE, 0.03)
        G_a = oo.metric_from_inv(wj_a, inv_a)
        locs = np.stack(oa.scatter(om, x_global.numpy()))
        ref = oa.assemble(om, list(oo.helmholtz(oe, locs, 1.0, G_a, wj_a)))
        err = float(np.max(np.abs(y_local.numpy() - ref[part.gids])) / np.max(np.abs(ref)))
        d = float(op.dot(y_local, y_local))
        q.put((rank, {"err": err, "dot": d, "dot_ref": float(ref @ ref),
                      "shared": {int(k): len(v) for k, v in part.shared.items()}}))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n,P", [(2, 4, 2), (2, 4, 3), (3, 6, 2), (4, 8, 2)])
def test_sharded_assembled_operator(world, n, P):
    """z-slab sharding with the one interface exchange per apply (SURVEY
    §8(e)): the gathered distributed result equals the unsharded assembled
    operator, interface planes hold n^2 P^2 dofs per neighbour, and the
    owner-masked dot product equals the global one."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, q, n, P)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=200) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
    for r in range(world):
        assert "error" not in res[r], res[r]["error"] if "error" in res[r] else ""
        assert res[r]["err"] < 1e-13
        assert abs(res[r]["dot"] - res[r]["dot_ref"]) <= 1e-10 * res[r]["dot_ref"]
        if world == 2:
            # both planes are shared with the single other rank: 2 n^2 P^2 dofs
            assert list(res[r]["shared"].values()) == [2 * n * n * P * P]
        else:
            # two distinct ring neighbours, one interface plane each
            assert sorted(res[r]["shared"]) == sorted({(r - 1) % world, (r + 1) % world})
            assert list(res[r]["shared"].values()) == [n * n * P * P] * 2


def test_slab_codes_match_full_map():
    """The per-slab map rows (closed form) equal the full periodic map's."""
    from paper_1906_03489_b200.assembly import hex_variable_codes
    from paper_1906_03489_b200.distributed import slab_codes

    n, P = 6, 3
    ng, off, codes = hex_variable_codes(n, np.full(n ** 3, P, dtype=np.int32))
    full = codes.reshape(n ** 3, -1)
    assert ng == (n * P) ** 3
    for e0, e1 in ((0, 36), (36, 108), (180, 216), (0, 216)):
        assert np.array_equal(slab_codes(n, P, e0, e1), full[e0:e1])
