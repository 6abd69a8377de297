#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2/early_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/early_tests.log
