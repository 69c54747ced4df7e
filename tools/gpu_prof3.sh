#!/bin/bash
mkdir -p gpurun_out
python tools/prof_helm.py --reps 2 --mode assembled > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_p4_gather python tools/prof_helm.py --reps 2 --mode assembled > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
