#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1500 python -m pytest -q -x tests -m gpu > gpurun_out/r2/pd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pd_tests.log
VARIANTS="pd0 pd1" bash scripts/gpu_decode_variants.sh
bash scripts/gpu_r2_timeline.sh mixtral qwen15
