#!/bin/bash
# full-size parity tests (BASELINE sizes) + hexpin P=7,8
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baseline.py tests/test_hex_pin.py -x -q -m gpu --durations=30 > gpurun_out/r2p_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
nproc >> gpurun_out/r2p_pytest.log
