#!/bin/bash
# One-block stage MMA issue (4 MMAs + merged commits from one elected lane): parity, then A/B vs HEAD.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_moe.py tests/test_gpu_prefill.py tests/test_gpu_nx64.py tests/test_gpu_quant_forward.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/r2/mma4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/mma4_tests.log
for rep in 1 2; do for v in head cur; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L timeout 600 python scripts/decode_ab.py mixtral:64 qwen15:64 deepseek:64 > gpurun_out/r2/mma4_dec_${v}_$rep.log 2>&1
  env $L AB_PATHS=ts timeout 600 python scripts/prefill_ab.py mixtral:4096 qwen15:4096 deepseek:4096 mixtral:1024 qwen15:2048 > gpurun_out/r2/mma4_ts_${v}_$rep.log 2>&1
  env $L AB_PATHS=gemv timeout 600 python scripts/prefill_ab.py mixtral:128 mixtral:256 mixtral:384 qwen15:1024 deepseek:768 > gpurun_out/r2/mma4_gemv_${v}_$rep.log 2>&1
done; done
