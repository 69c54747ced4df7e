#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/time_class.py 4 8 > gpurun_out/class_small.log 2>&1
echo "rc=$?" >> gpurun_out/class_small.log
timeout 900 python tools/time_class.py ${CLASS_PS:-2,3,4,5,6,7,8} 64 > gpurun_out/class_time.log 2>&1
echo "rc=$?" >> gpurun_out/class_time.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/class_launches.csv python tools/prof_helm.py --reps 2 --P ${CLASS_PP:-4} --mode assembled --alg class > /dev/null 2>&1
