#!/bin/bash
# per-CTA timeline of the decode step (PZ_TRACE build of route.cu + gemv_tc.cu); args: configs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for m in ${@:-mixtral qwen15 deepseek}; do
  for rep in 1 2; do
  TIMELINE_DUMP=gpurun_out/r2/timeline_${m}_64_$rep.npz PUZZLE_LIB=${TRACE_LIB:-build/variants/trace/libpuzzlemoe.so} timeout 300 python scripts/step_timeline.py $m 64 x > gpurun_out/r2/timeline_${m}_64_$rep.txt 2>&1
  done
done
