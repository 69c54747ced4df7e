#!/bin/bash
# ncu --set full of the fused local Helmholtz at P=2 and P=5 (the orders
# furthest from the HBM roofline)
mkdir -p gpurun_out
for P in 2 5; do
  python tools/prof_helm.py --reps 2 --P $P --mode local > gpurun_out/prof_plain$P.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
      -o gpurun_out/prof_p${P}_local python tools/prof_helm.py --reps 2 --P $P --mode local > gpurun_out/ncu_full$P.log 2>&1
  echo "rc=$?" >> gpurun_out/ncu_full$P.log
done
