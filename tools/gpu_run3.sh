#!/bin/bash
# parity tests, bench, launch list and one full ncu capture of the fused kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --sweep --cpu-seconds 10 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
python tools/prof_helm.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_helm.py --reps 2 > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 1 -c 2 \
    -o gpurun_out/prof_helm python tools/prof_helm.py --reps 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
