#!/bin/bash
# Q = 4 skewed-layout Helmholtz: parity, then P=2 timing per tile variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_hex_pin.py tests/test_gpu_assembly.py -x -q -k "helm or Helm or assembled or periodic or pin" > gpurun_out/q4_tests.log 2>&1
echo "rc=$?" >> gpurun_out/q4_tests.log
timeout 120 python tools/time_helm.py --P 2,3 > gpurun_out/q4_time.log 2>&1
for v in 1 2 4; do
  SPHP_LIBRARY_VARIANT=nb55 SPHP_HELM_VARIANT=$v timeout 120 python tools/time_helm.py --P 2 >> gpurun_out/q4_time.log 2>&1
done
python tools/prof_helm.py --reps 2 --P 2 --mode local > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_p2q4_local python tools/prof_helm.py --reps 2 --P 2 --mode local > gpurun_out/ncu_q4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_q4.log
