#!/bin/bash
# Suspend-hint mbarrier waits in the decode kernels: A/B (cur = spinning waits).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
PUZZLE_LIB=build/variants/sall/libpuzzlemoe.so timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_nx64.py tests/test_gpu_quant_forward.py -x -q -m gpu > gpurun_out/r2/sleep_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/sleep_tests.log
for rep in 1 2; do for v in cur sroles sall; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L timeout 600 python scripts/decode_ab.py mixtral:64 qwen15:64 deepseek:64 qwen15:16 > gpurun_out/r2/sleep_dec_${v}_$rep.log 2>&1
  env $L timeout 600 python scripts/quant_rate.py > gpurun_out/r2/sleep_q_${v}_$rep.log 2>&1
  env $L AB_PATHS=gemv timeout 600 python scripts/prefill_ab.py mixtral:256 mixtral:384 qwen15:1024 > gpurun_out/r2/sleep_g_${v}_$rep.log 2>&1
done; done
