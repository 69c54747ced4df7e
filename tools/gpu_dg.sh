#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dg.py -x -q -m gpu > gpurun_out/pytest_dg.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_dg.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
