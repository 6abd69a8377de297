#!/bin/bash
# A/B of decode build variants (build/variants/<name>)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for rep in 1 2; do
for v in ${VARIANTS}; do
  PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 300 python scripts/decode_ab.py ${CASES:-mixtral:64 qwen15:64 deepseek:64} > gpurun_out/r2/dvar_${v}_$rep.log 2>&1
done
done
