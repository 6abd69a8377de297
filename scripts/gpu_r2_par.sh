#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1200 python -m pytest -q -x tests/test_gpu_moe.py tests/test_gpu_quant_forward.py tests/test_gpu_ep.py tests/test_gpu_edge.py > gpurun_out/r2/par_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/par_tests.log
VARIANTS="cur own" bash scripts/gpu_decode_variants.sh
bash scripts/gpu_r2_timeline.sh mixtral
