#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1500 python -m pytest -q -x tests -m gpu > gpurun_out/r2/rdec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/rdec_tests.log
for rep in 1 2; do for v in rnew rdec; do
  AB_PATHS=gemv,ts PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 600 python scripts/prefill_ab.py mixtral:128 mixtral:256 mixtral:512 qwen15:128 qwen15:256 qwen15:512 deepseek:128 deepseek:256 deepseek:512 > gpurun_out/r2/rdec_${v}_$rep.log 2>&1
done; done
