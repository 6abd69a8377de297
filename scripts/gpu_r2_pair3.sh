#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for rep in 1 2; do for v in head cur; do
  AB_PATHS=ts PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 600 python scripts/prefill_ab.py mixtral:256 mixtral:512 qwen15:512 qwen15:1024 qwen15:2048 deepseek:512 deepseek:1024 > gpurun_out/r2/pair3_${v}_$rep.log 2>&1
done; done
