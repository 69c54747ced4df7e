#!/bin/bash
# k-major metric / global-geometry variants: local + class-assembled times per P, parity under the variant
mkdir -p gpurun_out
out=gpurun_out/kmajor.log
: > $out
for v in "" ${VARIANTS:-km kms}; do
  echo "== variant '$v'" >> $out
  SPHP_LIBRARY_VARIANT=$v timeout 600 python tools/time_helm.py --P ${PP:-2,3,4,5,6,7,8} --reps 10 >> $out 2>&1
done
for v in ${TESTV:-km}; do
  echo "== tests under '$v'" >> $out
  SPHP_LIBRARY_VARIANT=$v timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_assembly.py tests/test_gpu_solver.py tests/test_hex_pin.py 2>&1 | tail -3 >> $out
done
python tools/pcie_bw.py >> $out 2>&1
