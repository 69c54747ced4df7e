#!/bin/bash
# round-2 baseline: GPU tests + bench on a fresh box
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 900 python bench.py > gpurun_out/r2b_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2b_bench.log
