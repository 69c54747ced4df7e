#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/quad_variants.log
for v in "" b40 b56 b100 n2b40 n2b56 n2b74; do
  SPHP_LIBRARY_VARIANT=$v timeout 300 python tools/time_quad.py >> gpurun_out/quad_variants.log 2>&1
done
