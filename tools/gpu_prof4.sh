#!/bin/bash
# ncu evidence for round 1: launch list (P=4, local + assembled) and one full
# capture each of the fused local kernel and the owner-computes sum
mkdir -p gpurun_out
python tools/prof_helm.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_p4.csv python tools/prof_helm.py --reps 2 > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_p4_local python tools/prof_helm.py --reps 2 --mode local > gpurun_out/ncu_full.log 2>&1 && \
ncu --set full --clock-control none -k regex:"owner" -s 1 -c 1 \
    -o gpurun_out/prof_p4_owner python tools/prof_helm.py --reps 2 --mode assembled >> gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
