"""PCIe copy bandwidth on this box: H2D alone, D2H alone, both at once
(pinned host buffers, 134 MB = the cfg4 P=4 global vector)."""
import torch

n = 16777216
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  ({8 * n / ms / 1e6:.1f} GB/s per direction)")

# the slab pipeline's copy pattern: K slabs x 8 region pieces (P=4, n=64)
nn, b = 64, 3
N3, n2 = nn ** 3, nn * nn
szs = [1, b, b, b, b * b, b * b, b * b, b ** 3]
base, acc = [], 0
for s_ in szs:
    base.append(acc)
    acc += N3 * s_
for K in (4, 8, 16):
    zs = nn // K

    def pieces(K=K, zs=zs):
        with torch.cuda.stream(s1):
            for k in range(K):
                for r, s_ in enumerate(szs):
                    o, c = base[r] + k * zs * n2 * s_, zs * n2 * s_
                    d1[o:o + c].copy_(h1[o:o + c], non_blocking=True)

    def pieces_both(K=K, zs=zs):
        pieces(K, zs)
        with torch.cuda.stream(s2):
            for k in range(K):
                for r, s_ in enumerate(szs):
                    o, c = base[r] + k * zs * n2 * s_, zs * n2 * s_
                    h2[o:o + c].copy_(d2[o:o + c], non_blocking=True)

    print(f"K={K}: {8 * K} H2D pieces {t(pieces):.3f} ms; both directions {t(pieces_both):.3f} ms")
