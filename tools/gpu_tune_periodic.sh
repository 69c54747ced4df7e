#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tune_periodic.log
: > $out
for L in 0 8 16 32; do
  SPHP_PERIODIC_L=$L timeout 120 python tools/time_periodic.py 2,3,4,5,6 >> $out 2>&1
done
