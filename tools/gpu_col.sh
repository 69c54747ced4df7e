#!/bin/bash
# i-column plan (HexHelmCol): parity under the variant build, then local +
# class-assembled times per order for each tile size NE
mkdir -p gpurun_out
out=gpurun_out/col.log
: > $out
V=${V:-col}
echo "== tests under '$V'" >> $out
SPHP_LIBRARY_VARIANT=$V timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_hex_pin.py tests/test_gpu_assembly.py 2>&1 | tail -5 >> $out
echo "== baseline" >> $out
timeout 600 python tools/time_helm.py --P ${PP:-3,4,5,6,7,8} --reps 10 >> $out 2>&1
for ne in ${NES:-1 2 4 8}; do
  echo "== variant '$V' NE=$ne" >> $out
  SPHP_LIBRARY_VARIANT=$V SPHP_HELM_VARIANT=1$ne SPHP_CLASS_NE_ENV=$ne timeout 600 python tools/time_helm.py --P ${PP:-3,4,5,6,7,8} --reps 10 >> $out 2>&1
done
