#!/bin/bash
# A/B of TS prefill build variants (build/variants/<name>) on the fine-grained and Mixtral layers
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for v in ${VARIANTS}; do
  AB_PATHS=ts PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 300 python scripts/prefill_ab.py ${CASES:-qwen15:4096 deepseek:4096 mixtral:4096} > gpurun_out/r2/var_$v.log 2>&1
done
