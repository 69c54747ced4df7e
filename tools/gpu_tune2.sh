#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/tune.log
for v in 0 1 2 3 4; do
  SPHP_HELM_VARIANT=$v timeout 300 python tools/time_helm.py --P 2,3,4,5,6,7,8 >> gpurun_out/tune.log 2>&1
done
python tools/prof_helm.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_p4.csv python tools/prof_helm.py --reps 2 > gpurun_out/ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launch.log
