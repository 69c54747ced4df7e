"""Per-call host overhead of Collection.apply on the cfg1 workload (1024
affine quads, P=4): wall time per call over many calls (one sync at the end)
against the device time per apply (CUDA-graph replay of 20 applies)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1906_03489_b200 as sp  # noqa: E402

q = sp.make_quad(4, 6)
b = sp.ElementBatch.structured(q, 32, kind=sp.GEOM_AFFINE)
for op, size in (("bwdtrans", 25), ("iproductwrtbase", 36)):
    c = sp.Collection(b, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (1024, size)), device="cuda")
    y = torch.empty(c.output_shape, dtype=torch.float64, device="cuda")
    for _ in range(2000):
        c.apply(x, y)
    torch.cuda.synchronize()
    N = 20000
    t0 = time.perf_counter()
    for _ in range(N):
        c.apply(x, y)
    torch.cuda.synchronize()
    per_call = (time.perf_counter() - t0) / N * 1e6
    side = torch.cuda.Stream()
    c.reserve(stream=side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(20):
            c.apply(x, y)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / (50 * 20) * 1e3
    print(f"cfg1 {op}: {per_call:.2f} us per Python call, device {dev:.2f} us per apply (graph replay)",
          flush=True)
