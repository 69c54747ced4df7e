#!/bin/bash
# parity tests, smoke, then a short bench (no ncu in this call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --sweep --cpu-seconds 10 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
