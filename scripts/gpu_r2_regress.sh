#!/bin/bash
# Same-box A/B of the decode step (T 64) before the NX 64 / NX 128 changes (variant "old") and now.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for rep in 1 2; do for v in old cur; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L timeout 600 python scripts/decode_ab.py mixtral:64 qwen15:64 deepseek:64 qwen15:16 > gpurun_out/r2/regress_${v}_$rep.log 2>&1
done; done
