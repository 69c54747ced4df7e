#!/bin/bash
# full ncu capture of the split-path scatter and the owner sum
mkdir -p gpurun_out
timeout 300 python tools/prof_split.py > gpurun_out/prof_split.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"periodic_scatter_v2|owner_periodic_v3" -c 2 \
  -o gpurun_out/asm_full python tools/prof_split.py > gpurun_out/ncu_asm_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_asm_full.log
