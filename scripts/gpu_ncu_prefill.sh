#!/bin/bash
# ncu --set full of the prefill tcgen05 kernels (one launch each) at Mixtral T = 4096
cd $GRAFT_REPO_ROOT
CMD="python bench.py --batch 4096 --steps 3 --warmup 3 --no-extra --no-cpu --no-graph"
$CMD > gpurun_out/np_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:k_tc_experts --launch-skip 6 --launch-count 2 -o gpurun_out/full_tc -f $CMD > gpurun_out/np_ncu.log 2>&1
echo rc=$? >> gpurun_out/np_ncu.log
