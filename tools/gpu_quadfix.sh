#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_assembly.py tests/test_gpu_golden.py tests/test_gpu_solver.py tests/test_gpu_dg.py -x -q -m gpu > gpurun_out/pytest_q.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_q.log
timeout 300 python tools/time_quad.py > gpurun_out/quad_new.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 1 -c 1 -o gpurun_out/prof_quad2 python tools/prof_quad.py > gpurun_out/ncu_quad2.log 2>&1
