#!/bin/bash
# round-2 evidence on the current build: fp64 peak, GPU tests, bench, DRAM
# traffic of the dominant kernels, the bench's launch list, one full ncu
# capture of the class-range operator
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r2_fp64_peak.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  -k regex:pipe_kernel --log-file gpurun_out/r2_traffic.csv python tools/prof_helm.py --reps 2 --P 4 --mode both --alg class > /dev/null 2>&1
python tools/make_traffic_json.py gpurun_out/r2_traffic.csv gpurun_out/r02_ncu_traffic.json 4 64 > gpurun_out/r2_traffic.log 2>&1
mkdir -p profiles && cp gpurun_out/r02_ncu_traffic.json profiles/ 2>/dev/null
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-sweep --no-extras > gpurun_out/r2_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel|class_owner" -s 2 -c 2 \
    -o gpurun_out/r2_full_p4_class python tools/prof_helm.py --reps 2 --P 4 --mode assembled --alg class > gpurun_out/r2_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ncu_full.log
