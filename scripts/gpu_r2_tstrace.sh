#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for v in ${TVARS:-tstrace}; do
PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 300 python scripts/trace_ts.py qwen15 4096 > gpurun_out/r2/tstrace_${v}_qwen15.txt 2>&1
done
if [ -n "$VARIANTS" ]; then bash scripts/gpu_ts_variants.sh; fi
