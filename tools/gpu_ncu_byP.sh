#!/bin/bash
# one ncu --set full capture of the shipped fused local Helmholtz and of the
# class-range operator at every order P=2..8 (cfg4 64^3); text summaries only
mkdir -p gpurun_out/byP /tmp/byP
for P in ${PS:-2 3 4 5 6 7 8}; do
  if [ "${WHICH:-both}" != "class" ]; then
  python tools/prof_helm.py --reps 2 --P $P --mode local > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 1 -c 1 \
      -o /tmp/byP/local_p$P python tools/prof_helm.py --reps 2 --P $P --mode local > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/byP/local_p$P.ncu-rep > gpurun_out/byP/local_p$P.txt 2>&1
  fi
  if [ "${WHICH:-both}" != "local" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 1 -c 1 \
      -o /tmp/byP/class_p$P python tools/prof_helm.py --reps 2 --P $P --mode assembled --alg class > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/byP/class_p$P.ncu-rep > gpurun_out/byP/class_p$P.txt 2>&1
  fi
done
