#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1500 python -m pytest -q -x tests -m gpu > gpurun_out/r2/rs2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/rs2_tests.log
AB_PATHS=ts,gemv timeout 600 python scripts/prefill_ab.py mixtral:128 mixtral:256 mixtral:512 mixtral:1024 qwen15:128 qwen15:256 qwen15:512 qwen15:1024 deepseek:256 deepseek:1024 > gpurun_out/r2/rs_rnew.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/r2/rs2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2/rs2_bench.log
