#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2f_smoke.log
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2f_bench.log
