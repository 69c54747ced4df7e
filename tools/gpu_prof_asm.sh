#!/bin/bash
mkdir -p gpurun_out
python tools/prof_helm.py --reps 2 --mode assembled > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_asm.csv \
    python tools/prof_helm.py --reps 2 --mode assembled > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel|owner" -s 2 -c 2 \
    -o gpurun_out/prof_asm python tools/prof_helm.py --reps 2 --mode assembled > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
