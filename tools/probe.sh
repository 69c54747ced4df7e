#!/bin/bash
mkdir -p gpurun_out
{
nvidia-smi
nproc; lscpu | head -20; free -g
./tools/fp64_peak
python - <<'PY'
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device='cuda'); b = torch.randn_like(a)
for _ in range(3): c = a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print("torch fp64 matmul 8192^3: %.2f TFLOP/s" % (2*8192**3/best/1e9))
x = torch.empty(2**28, dtype=torch.float64, device='cuda'); y = torch.empty_like(x)
best = 1e9
for _ in range(10):
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print("copy GB/s: %.1f" % (2*x.numel()*8/best/1e6))
PY
} > gpurun_out/probe.log 2>&1
