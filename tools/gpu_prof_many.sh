#!/bin/bash
# ncu --set full of two kernels per call (gpurun_out is capped at 64 MiB):
#   $1 = "helm68": Helmholtz P=6 and P=8 (local);  "ipdquad": hex
#   IProductWRTDerivBase P=4 and quad Helmholtz cfg2
mkdir -p gpurun_out
if [ "$1" = helm68 ]; then
for P in 6 8; do
  python tools/prof_helm.py --reps 2 --P $P --mode local > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
      -o gpurun_out/prof_p${P}_local python tools/prof_helm.py --reps 2 --P $P --mode local > gpurun_out/pm_$P.log 2>&1
done
else
python tools/prof_hexop.py iproductwrtderivbase 4 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_ipd_p4 python tools/prof_hexop.py iproductwrtderivbase 4 > gpurun_out/pm_ipd.log 2>&1
python tools/prof_quad.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_quad_helm python tools/prof_quad.py > gpurun_out/pm_quad.log 2>&1
fi
echo done
