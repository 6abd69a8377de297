#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 5 --warmup 3 --no-extra --no-cpu --no-graph --batch 1"
$CMD > gpurun_out/plain_b1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemv_tma -s 2 -c 2 -o gpurun_out/prof_b1 $CMD > gpurun_out/ncu_b1.log 2>&1
echo done
