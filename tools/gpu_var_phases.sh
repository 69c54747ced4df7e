#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/var_phases.log
for v in "" ${VARIANTS}; do
  echo "== variant '$v'" >> gpurun_out/var_phases.log
  SPHP_LIBRARY_VARIANT=$v timeout 600 python tools/time_phases.py ${PS:-2,3} >> gpurun_out/var_phases.log 2>&1
done
