#!/bin/bash
# NX = 128 one-CTA-per-SM decode configuration: parity, then A/B vs NX 64 only (variant) vs TS.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_nx64.py tests/test_gpu_moe.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/r2/nx128_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2/nx128_tests.log
CASES="mixtral:192 mixtral:256 mixtral:320 mixtral:384 mixtral:512 mixtral:768 mixtral:1024 qwen15:768 qwen15:1024 qwen15:1536 qwen15:2048 deepseek:512 deepseek:768 deepseek:1024 deepseek:1536"
AB_PATHS=gemv,ts timeout 900 python scripts/prefill_ab.py $CASES > gpurun_out/r2/nx128_cur.log 2>&1
AB_PATHS=gemv PUZZLE_LIB=build/variants/nx64only/libpuzzlemoe.so timeout 900 python scripts/prefill_ab.py $CASES > gpurun_out/r2/nx128_nx64only.log 2>&1
