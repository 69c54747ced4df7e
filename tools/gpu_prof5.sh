#!/bin/bash
mkdir -p gpurun_out
python tools/time_asm_variants.py > gpurun_out/asm_variants.log 2>&1
python tools/prof_helm.py --reps 2 --P 8 --mode local > gpurun_out/prof_plain8.log 2>&1 && \
ncu --set full --clock-control none -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_p8_local python tools/prof_helm.py --reps 2 --P 8 --mode local > gpurun_out/ncu_full8.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full8.log
