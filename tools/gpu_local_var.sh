#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/local_var.log
for v in "" ${VARIANTS}; do
  echo "== variant '$v'" >> gpurun_out/local_var.log
  SPHP_LIBRARY_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"pipe_kernel" \
    python tools/prof_helm.py --reps 3 --P ${CLASS_PP:-4} --mode local 2>/dev/null | grep -E "pipe_kernel" | tail -2 | cut -c1-30,150- >> gpurun_out/local_var.log
done
