#!/bin/bash
# step timelines of graph-replayed forwards (PZ_TRACE build)
cd $GRAFT_REPO_ROOT
for c in "mixtral 64" "mixtral 1" "qwen15 64" "qwen15 1" "deepseek 64"; do
  PUZZLE_LIB=build/variants/trace/libpuzzlemoe.so timeout 300 python scripts/step_timeline.py $c >> gpurun_out/timeline.log 2>&1
done
