#!/bin/bash
# tile-variant sweep (SPHP_HELM_VARIANT 0..4) of the Helmholtz after the
# layout changes: P=3 (part 0), P=5 (part 1), P=7 (part 2) variant builds
mkdir -p gpurun_out
: > gpurun_out/tune3.log
for v in 0 1 2 3 4; do
  SPHP_LIBRARY_VARIANT=tun0 SPHP_HELM_VARIANT=$v timeout 120 python tools/time_helm.py --P 2,3 >> gpurun_out/tune3.log 2>&1
  SPHP_LIBRARY_VARIANT=tun1 SPHP_HELM_VARIANT=$v timeout 120 python tools/time_helm.py --P 4,5 >> gpurun_out/tune3.log 2>&1
  SPHP_LIBRARY_VARIANT=tun2 SPHP_HELM_VARIANT=$v timeout 200 python tools/time_helm.py --P 6,7 >> gpurun_out/tune3.log 2>&1
done
