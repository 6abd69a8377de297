#!/bin/bash
# TS prefill: parity, trace, A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 900 python -X faulthandler -m pytest tests/test_gpu_prefill.py -x -q -p no:cacheprovider -k "not mixtral" > gpurun_out/r2/ts_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/ts_tests.log
PUZZLE_LIB=build/variants/tstrace/libpuzzlemoe.so timeout 300 python scripts/trace_ts.py qwen15 4096 > gpurun_out/r2/trace_ts_qwen.txt 2>&1
timeout 600 python scripts/prefill_ab.py mixtral:4096 qwen15:4096 deepseek:4096 mixtral:1024 qwen15:512 > gpurun_out/r2/ts_ab.log 2>&1; echo "rc=$?" >> gpurun_out/r2/ts_ab.log
