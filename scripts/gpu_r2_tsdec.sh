#!/bin/bash
# TS prefill with 8 decoder warps (K halves) instead of 4: parity of the variant, then A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
PUZZLE_LIB=build/variants/d8e16/libpuzzlemoe.so timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_moe.py -x -q -m gpu -k "tc or ts or prefill or mixed" > gpurun_out/r2/tsdec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/tsdec_tests.log
for rep in 1 2; do for v in cur d8e16 d8e8; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L AB_PATHS=ts timeout 600 python scripts/prefill_ab.py mixtral:4096 qwen15:4096 deepseek:4096 mixtral:1024 qwen15:2048 deepseek:1024 > gpurun_out/r2/tsdec_${v}_$rep.log 2>&1
done; done
