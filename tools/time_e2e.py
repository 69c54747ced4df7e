"""End-to-end apply through the C ABI with pinned host vectors
(sphp_helmholtz_assembled_host) at P=4, n=64, for several host-slab sizes
(SPHP_HOST_SLABS is read once per process, so each size runs in its own
process) next to the PCIe floor (both directions at once)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    import paper_1906_03489_b200 as sp
    from paper_1906_03489_b200 import _lib

    P, n = 4, 64
    exp = sp.make_hex(P, P + 2)
    batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=0.03)
    coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC)
    amap = sp.AssemblyMap.hex_periodic(n, P)
    ng = amap.num_global
    xh = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, ng)).pin_memory()
    yh = torch.empty(ng, dtype=torch.float64).pin_memory()
    st = torch.cuda.current_stream()

    def step():
        _lib.check(_lib.lib.sphp_helmholtz_assembled_host(coll._handle, amap._h, _lib.ptr(xh), _lib.ptr(yh),
                                                          _lib.stream_ptr(st)))
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    print(f"slabs={os.environ.get('SPHP_HOST_SLAB_LIST', os.environ.get('SPHP_HOST_SLABS', 'default'))}: "
          f"e2e {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
else:
    lists = sys.argv[1:] or ["", "1,1,2,4,8,8,8,8,8,4,2,1,1", "1,1,2,4,8,8,8,8,8,8,4,2,1,1"[:0] or
                             "1,2,4,8,8,8,8,8,8,4,2,1,1,1", "2,2,4,8,8,8,8,8,8,4,2,1,1", "1,1,2,4,6,6,6,6,6,6,6,6,4,2,1,1"]
    for s in lists:
        env = dict(os.environ, SPHP_HOST_SLAB_LIST=s)
        subprocess.run([sys.executable, __file__, "child"], env=env)
