#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for v in cur n64x6w7 n64x4w8 n96x4w6; do
  AB_PATHS=ts PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 600 python scripts/prefill_ab.py mixtral:256 mixtral:512 mixtral:1024 qwen15:1024 qwen15:2048 deepseek:1024 deepseek:2048 > gpurun_out/r2/tss_$v.log 2>&1
done
