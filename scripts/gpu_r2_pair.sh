#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1200 python -m pytest -q -x tests/test_gpu_prefill.py tests/test_gpu_moe.py tests/test_gpu_edge.py > gpurun_out/r2/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pair_tests.log
for v in head cur; do
  AB_PATHS=ts PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 600 python scripts/prefill_ab.py mixtral:256 mixtral:512 mixtral:1024 mixtral:4096 qwen15:1024 qwen15:2048 qwen15:4096 deepseek:1024 deepseek:2048 deepseek:4096 > gpurun_out/r2/pair_$v.log 2>&1
done
