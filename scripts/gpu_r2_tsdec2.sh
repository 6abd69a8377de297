#!/bin/bash
# TS with 8 decoder warps in the PAIRED-item regime (buckets <= 160 tokens on average).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for rep in 1 2; do for v in cur d8e16; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L AB_PATHS=ts timeout 600 python scripts/prefill_ab.py mixtral:512 mixtral:576 qwen15:1536 qwen15:2048 deepseek:1024 deepseek:1536 > gpurun_out/r2/tsdec2_${v}_$rep.log 2>&1
done; done
