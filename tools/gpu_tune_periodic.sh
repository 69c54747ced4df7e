#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tune_periodic.log
: > $out
timeout 900 python -m pytest tests/test_gpu_assembly.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for dyn in 1; do for L in 0 8 16 32; do
  SPHP_PERIODIC_DYNAMIC=$dyn SPHP_PERIODIC_L=$L timeout 120 python tools/time_periodic.py 2,3,4,5,6,7,8 | sed "s/^/dyn=$dyn /" >> $out 2>&1
done; done
timeout 300 python tools/prof_split.py > gpurun_out/prof_split.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_split.csv python tools/prof_split.py > gpurun_out/ncu_split.log 2>&1
