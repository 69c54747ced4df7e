#!/bin/bash
# phases at every P, then one ncu --set full of the class operator + owner at P=$CLASS_PP
mkdir -p gpurun_out
python tools/time_phases.py > gpurun_out/phases.log 2>&1
P=${CLASS_PP:-3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel|class_owner" -s 2 -c 2 \
    -o gpurun_out/cp_full_p$P python tools/prof_helm.py --reps 2 --P $P --mode assembled --alg class > gpurun_out/cp_ncu_p$P.log 2>&1
