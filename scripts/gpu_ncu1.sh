#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 5 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_w13_gemv -s 3 -c 1 -o gpurun_out/prof_w13 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
