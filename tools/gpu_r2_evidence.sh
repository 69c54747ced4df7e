#!/bin/bash
# round-2 evidence: GPU tests, smoke, bench, the bench's ncu launch list, and
# ncu --set full of the shipped P=4 K4 kernel and the split assembly kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2e_smoke.log
timeout 900 python bench.py > gpurun_out/r2e_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2e_bench.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/r2e_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2e_ncu_bench.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_ncu_bench.log
python tools/prof_helm.py --reps 2 --P 4 --mode assembled > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -s 3 -c 3 \
    -o gpurun_out/r2e_prof_p4_asm python tools/prof_helm.py --reps 2 --P 4 --mode assembled > gpurun_out/r2e_ncu_p4.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_ncu_p4.log
