"""Bidirectional PCIe copy patterns of the cfg4 P=4 global vector (134 MB
each way, pinned host buffers): the host pipeline's current per-slab region
pieces vs one contiguous range per slab (what a slab-major numbering would
allow), for several slab counts.  Prints ms per pattern (median of 7)."""
import statistics

import torch

n, b = 64, 3
N3, n2 = n ** 3, n * n
szs = [1, b, b, b, b * b, b * b, b * b, b ** 3]
ng = N3 * sum(szs)
base, acc = [], 0
for s_ in szs:
    base.append(acc)
    acc += N3 * s_
hx = torch.empty(ng, dtype=torch.float64).pin_memory()
hy = torch.empty(ng, dtype=torch.float64).pin_memory()
dx = torch.empty(ng, dtype=torch.float64, device="cuda")
dy = torch.empty(ng, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def slabs(K):
    if K == 13:
        pl = [1, 1, 2] + [8] * 7 + [2, 1, 1]
    else:
        pl = [n // K] * K
    zb = [0]
    for p in pl:
        zb.append(zb[-1] + p)
    return zb


def regions(zb, d, h, to_dev):
    for k in range(len(zb) - 1):
        z0, z1 = zb[k], zb[k + 1]
        for r, s_ in enumerate(szs):
            o, c = base[r] + z0 * n2 * s_, (z1 - z0) * n2 * s_
            if to_dev:
                d[o:o + c].copy_(h[o:o + c], non_blocking=True)
            else:
                h[o:o + c].copy_(d[o:o + c], non_blocking=True)


def contig(zb, d, h, to_dev):
    for k in range(len(zb) - 1):
        o, c = zb[k] * n2 * sum(szs), (zb[k + 1] - zb[k]) * n2 * sum(szs)
        if to_dev:
            d[o:o + c].copy_(h[o:o + c], non_blocking=True)
        else:
            h[o:o + c].copy_(d[o:o + c], non_blocking=True)


def both(fn, zb):
    with torch.cuda.stream(s1):
        fn(zb, dx, hx, True)
    with torch.cuda.stream(s2):
        fn(zb, dy, hy, False)


def t(f):
    ts = []
    for _ in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        f()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts[1:])


print(f"one copy each way: {t(lambda: both(contig, [0, n])):.3f} ms")
for K in (4, 8, 13, 16, 32):
    zb = slabs(K)
    print(f"K={K}: region pieces {t(lambda: both(regions, zb)):.3f} ms, contiguous slabs {t(lambda: both(contig, zb)):.3f} ms",
          flush=True)
