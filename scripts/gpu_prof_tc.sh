#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-graph --batch 4096"
$CMD > gpurun_out/plain_tc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_experts -s 2 -c 1 -o gpurun_out/prof_tc1 $CMD > gpurun_out/ncu_tc.log 2>&1
echo done
