#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 5 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemv_tma -s 2 -c 2 -o gpurun_out/prof_gemv3 $CMD > gpurun_out/ncu_full.log 2>&1
CMD2="python bench.py --steps 5 --warmup 3 --no-extra --no-cpu --config qwen15 --batch 1"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qwen1.csv $CMD2 > gpurun_out/ncu_l2.log 2>&1
echo done
