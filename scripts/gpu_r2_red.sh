#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 600 python -m pytest -q -x tests/test_gpu_moe.py tests/test_gpu_quant_forward.py > gpurun_out/r2/red_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/red_tests.log
bash scripts/gpu_r2_timeline.sh mixtral
VARIANTS="base cpasync new" bash scripts/gpu_decode_variants.sh
