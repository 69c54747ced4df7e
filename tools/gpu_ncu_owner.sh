#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/time_periodic.py 4 > gpurun_out/tp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"owner_periodic_v3|periodic_scatter_v2" -s 4 -c 2 \
  -o gpurun_out/owner_full python tools/time_periodic.py 4 > gpurun_out/ncu_owner.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_owner.log
