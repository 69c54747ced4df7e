#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/hexops_variants.log
for v in "" hb30 hb40 hb56 hb100; do for P in 2 4 6; do
  SPHP_LIBRARY_VARIANT=$v timeout 300 python tools/time_hexops.py $P >> gpurun_out/hexops_variants.log 2>&1
done; done
