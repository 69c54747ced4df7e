#!/bin/bash
# segment length x CTAs/SM sweep of the periodic scatter / owner kernels, low orders
mkdir -p gpurun_out
out=gpurun_out/tune_periodic2.log
: > $out
for L in 0 4 8 16 32; do for C in 0 2 4 8; do
  SPHP_PERIODIC_L=$L SPHP_PERIODIC_CTAS=$C timeout 120 python tools/time_periodic.py 2,3 >> $out 2>&1
done; done
