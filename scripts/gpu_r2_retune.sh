#!/bin/bash
# Thresholds after the staged wide reducer: GEMV (NX 128 above 56, or above 44: variant) vs TS.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
CASES="mixtral:192 mixtral:448 mixtral:512 qwen15:768 qwen15:1280 qwen15:1536 deepseek:512 deepseek:768 deepseek:1024"
for rep in 1 2; do
  AB_PATHS=gemv,ts timeout 900 python scripts/prefill_ab.py $CASES > gpurun_out/r2/retune_cur_$rep.log 2>&1
  AB_PATHS=gemv PUZZLE_LIB=build/variants/nx128at44/libpuzzlemoe.so timeout 900 python scripts/prefill_ab.py mixtral:192 qwen15:768 deepseek:512 > gpurun_out/r2/retune_44_$rep.log 2>&1
done
