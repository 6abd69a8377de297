#!/bin/bash
# Staged reducer for the wide decode configurations when two slots of the item's rows fit: parity, A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_nx64.py tests/test_gpu_moe.py tests/test_gpu_ep.py -x -q -m gpu > gpurun_out/r2/sred_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/sred_tests.log
for rep in 1 2; do for v in head2 cur; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L timeout 600 python scripts/decode_ab.py mixtral:128 mixtral:256 mixtral:384 qwen15:512 qwen15:1024 deepseek:512 deepseek:768 > gpurun_out/r2/sred_${v}_$rep.log 2>&1
done; done
