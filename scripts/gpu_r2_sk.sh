#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 600 python -m pytest -q -x tests/test_gpu_moe.py > gpurun_out/r2/sk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/sk_tests.log
VARIANTS="sk11 sk_a sk_b sk_c" bash scripts/gpu_decode_variants.sh
bash scripts/gpu_r2_timeline.sh mixtral qwen15
