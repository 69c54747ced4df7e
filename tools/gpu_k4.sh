#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_assembly.py tests/test_gpu_golden.py tests/test_hex_pin.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/time_helm.py --P 2,3,4,5,6,7,8 > gpurun_out/time_helm.log 2>&1
