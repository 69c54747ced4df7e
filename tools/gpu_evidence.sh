#!/bin/bash
# round evidence: GPU tests, smoke, bench line, the bench's own ncu launch
# list, and one ncu --set full capture of the P=4 fused local kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/ev_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/ev_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/ev_bench_ref.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/ev_bench_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ev_ncu_bench.log 2>&1
echo "rc=$?" >> gpurun_out/ev_ncu_bench.log
python tools/prof_helm.py --reps 2 --P 4 --mode local > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_p4_local python tools/prof_helm.py --reps 2 --P 4 --mode local > gpurun_out/ev_ncu_p4.log 2>&1
echo "rc=$?" >> gpurun_out/ev_ncu_p4.log
