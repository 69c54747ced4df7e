#!/bin/bash
mkdir -p gpurun_out
P=${CLASS_PP:-4}
python tools/prof_helm.py --reps 2 --P $P --mode assembled --alg class > gpurun_out/cp_run.log 2>&1
echo "rc=$?" >> gpurun_out/cp_run.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel|class_owner" -s 2 -c 2 \
    -o gpurun_out/cp_full python tools/prof_helm.py --reps 2 --P $P --mode assembled --alg class > gpurun_out/cp_ncu2.log 2>&1
echo "rc=$?" >> gpurun_out/cp_ncu2.log
