#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1500 python -m pytest -q -x tests -m gpu > gpurun_out/r2/id_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/id_tests.log
VARIANTS="id0 id1" bash scripts/gpu_decode_variants.sh
CASES="mixtral:1 qwen15:1 qwen15:16" VARIANTS="id0 id1" bash -c 'for rep in 1; do for v in $VARIANTS; do PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 300 python scripts/decode_ab.py $CASES > gpurun_out/r2/dvar_small_${v}.log 2>&1; done; done'
bash scripts/gpu_r2_timeline.sh mixtral qwen15
