#!/bin/bash
# ncu launch list of the bench command itself (after it exits 0 without ncu)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_small.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_bench.log
