#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tune_periodic.log
: > $out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for L in 0; do
  SPHP_PERIODIC_L=$L timeout 120 python tools/time_periodic.py 2,3,4,5,6,7,8 >> $out 2>&1
done
timeout 300 python tools/time_asm_variants.py > gpurun_out/asm_variants.log 2>&1
