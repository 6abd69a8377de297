#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 900 python -m pytest -q -x tests/test_gpu_prefill.py > gpurun_out/r2/seq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/seq_tests.log
TVARS="tstrace" bash scripts/gpu_r2_tstrace.sh
for rep in 1 2; do for v in seq0 seq1; do
  AB_PATHS=ts PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 300 python scripts/prefill_ab.py qwen15:4096 deepseek:4096 mixtral:4096 > gpurun_out/r2/var_${v}_$rep.log 2>&1
done; done
