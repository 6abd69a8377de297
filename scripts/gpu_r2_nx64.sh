#!/bin/bash
# NX = 64 decode configuration: parity (new + existing GEMV tests), then the intermediate-batch
# A/B: NX 64 (in-tree) vs NX 32 only (variant) vs the TS prefill kernel.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_nx64.py tests/test_gpu_moe.py -x -q -m gpu > gpurun_out/r2/nx64_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2/nx64_tests.log
CASES="mixtral:64 mixtral:96 mixtral:128 mixtral:192 mixtral:256 mixtral:384 mixtral:512 qwen15:128 qwen15:256 qwen15:384 qwen15:512 qwen15:768 qwen15:1024 deepseek:256 deepseek:384 deepseek:512 deepseek:768"
AB_PATHS=gemv,ts timeout 900 python scripts/prefill_ab.py $CASES > gpurun_out/r2/nx64_cur.log 2>&1
AB_PATHS=gemv PUZZLE_LIB=build/variants/nx32/libpuzzlemoe.so timeout 900 python scripts/prefill_ab.py $CASES > gpurun_out/r2/nx64_nx32.log 2>&1
