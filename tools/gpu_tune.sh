#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3 4; do
  SPHP_HELM_VARIANT=$v timeout 300 python tools/time_helm.py --P 2,3,4,5,6,7,8 >> gpurun_out/tune.log 2>&1
done
