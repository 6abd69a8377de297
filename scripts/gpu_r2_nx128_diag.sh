#!/bin/bash
# NX = 128 diagnosis: per-stage timeline of one CTA (trace build) at Mixtral T 256 (NX 128) and
# T 128 (NX 64); A/B of the deferred epilogue (PZ_TC_DEFER=1) on the wide configurations.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
PUZZLE_LIB=build/variants/trace/libpuzzlemoe.so timeout 300 python scripts/trace_gemv.py mixtral 256 > gpurun_out/r2/trace_nx128_m256.log 2>&1
PUZZLE_LIB=build/variants/trace/libpuzzlemoe.so timeout 300 python scripts/trace_gemv.py mixtral 128 > gpurun_out/r2/trace_nx64_m128.log 2>&1
CASES="mixtral:128 mixtral:256 mixtral:384 qwen15:1024 deepseek:768"
for rep in 1 2; do for v in cur defer; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L AB_PATHS=gemv timeout 600 python scripts/prefill_ab.py $CASES > gpurun_out/r2/diag_${v}_$rep.log 2>&1
done; done
