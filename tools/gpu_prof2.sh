#!/bin/bash
# launch list (P=4, both modes) + full capture of the fused local kernel (P=4)
mkdir -p gpurun_out
python tools/prof_helm.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_p4.csv python tools/prof_helm.py --reps 2 > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_p4_local python tools/prof_helm.py --reps 2 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
ls -la gpurun_out >> gpurun_out/ncu_full.log
