#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assembly.py -x -q -m gpu -k host > gpurun_out/pytest_asm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_asm.log
for d in 0 1; do for k in 4 8; do
  SPHP_HOST_DIRECT=$d SPHP_HOST_SLABS=$k timeout 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-extras --no-cpu > gpurun_out/bench_e2e_${d}_$k.log 2>&1
done; done
