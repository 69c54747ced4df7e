#!/bin/bash
# ncu --set full of the i-column plan: CASES="P:NE ..." MODE=local|assembled
mkdir -p gpurun_out/colncu /tmp/colncu
export SPHP_LIBRARY_VARIANT=${V-col}
MODE=${MODE:-local}
for c in ${CASES:-3:4 5:2 7:1 8:1}; do
  P=${c%%:*}; ne=${c#*:}
  export SPHP_HELM_VARIANT=1$ne SPHP_CLASS_NE_ENV=$ne
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 1 -c 1 \
      -o /tmp/colncu/${MODE}_p${P}_ne$ne python tools/prof_helm.py --reps 2 --P $P --mode $MODE --alg class > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/colncu/${MODE}_p${P}_ne$ne.ncu-rep > gpurun_out/colncu/${MODE}_p${P}_ne$ne.txt 2>&1
done
