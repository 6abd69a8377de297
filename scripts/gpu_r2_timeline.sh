#!/bin/bash
# per-CTA timeline of the decode step (PZ_TRACE build of route.cu + gemv_tc.cu); args: config or config:T
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for arg in ${@:-mixtral qwen15 deepseek}; do
  m=${arg%%:*}; T=64; [ "$arg" != "$m" ] && T=${arg##*:}
  for rep in 1 2; do
  TIMELINE_DUMP=gpurun_out/r2/timeline_${m}_${T}_$rep.npz PUZZLE_LIB=${TRACE_LIB:-build/variants/trace/libpuzzlemoe.so} timeout 300 python scripts/step_timeline.py $m $T x > gpurun_out/r2/timeline_${m}_${T}_$rep.txt 2>&1
  done
done
