#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 900 python -m pytest -q -x tests/test_gpu_moe.py tests/test_gpu_edge.py tests/test_gpu_quant_forward.py > gpurun_out/r2/setup_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/setup_tests.log
VARIANTS="head setup" bash scripts/gpu_decode_variants.sh
bash scripts/gpu_r2_timeline.sh qwen15
