#!/bin/bash
# assembled-path check: GPU tests, algorithm timings, ncu launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_asm_variants.py > gpurun_out/asm_variants.log 2>&1
timeout 300 python tools/prof_split.py > gpurun_out/prof_split.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_split.csv python tools/prof_split.py > gpurun_out/ncu_split.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_split.log
