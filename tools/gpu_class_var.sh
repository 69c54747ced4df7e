#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/class_var.log
for v in "" ${VARIANTS}; do
  echo "== variant '$v'" >> gpurun_out/class_var.log
  SPHP_LIBRARY_VARIANT=$v timeout 300 python tools/time_class.py ${CLASS_PS:-4} 64 >> gpurun_out/class_var.log 2>&1
  SPHP_LIBRARY_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"class_owner|pipe_kernel" \
    python tools/prof_helm.py --reps 2 --P ${CLASS_PP:-4} --mode assembled --alg class 2>/dev/null | grep -E "class_owner|pipe_kernel" | tail -2 | cut -c1-40,200- >> gpurun_out/class_var.log
done
