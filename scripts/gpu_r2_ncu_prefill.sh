#!/bin/bash
# round 2: what bounds the prefill tcgen05 kernels? ncu --set full of one w13 + one w2 launch at
# Mixtral and Qwen T = 4096 (plain runs first, must exit 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for cfg in mixtral qwen15; do
  CMD="python bench.py --config $cfg --batch 4096 --steps 3 --warmup 3 --no-extra --no-cpu --no-graph"
  $CMD > gpurun_out/r2/np_${cfg}_plain.log 2>&1 || { echo "plain failed $cfg"; continue; }
  timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:k_tc_experts --launch-skip 6 --launch-count 2 -o gpurun_out/r2/full_tc_${cfg} -f $CMD > gpurun_out/r2/np_${cfg}_ncu.log 2>&1
  echo rc=$? >> gpurun_out/r2/np_${cfg}_ncu.log
done
