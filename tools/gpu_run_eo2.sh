#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/time_helm.py --P 2,3,4,5,6,7,8 > gpurun_out/tune_eo.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.log 2>&1
