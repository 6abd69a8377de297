#!/bin/bash
# NX = 128 ring depths (W / X slots): the X ring's turnaround paced the 3-slot form (trace)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
CASES="mixtral:256 mixtral:384 qwen15:1024 deepseek:768"
for rep in 1 2; do for v in cur w5x4 w3x5 w4x4; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L AB_PATHS=gemv timeout 600 python scripts/prefill_ab.py $CASES > gpurun_out/r2/rings_${v}_$rep.log 2>&1
done; done
