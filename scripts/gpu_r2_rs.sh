#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
PUZZLE_LIB=build/variants/rs128/libpuzzlemoe.so timeout 1500 python -m pytest -q -x tests -m gpu > gpurun_out/r2/rs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/rs_tests.log
for v in rs4096 rs512 rs128; do
  AB_PATHS=ts,gemv PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 600 python scripts/prefill_ab.py mixtral:128 mixtral:256 mixtral:512 mixtral:1024 qwen15:128 qwen15:256 qwen15:512 qwen15:1024 deepseek:256 deepseek:1024 > gpurun_out/r2/rs_$v.log 2>&1
done
