#!/bin/bash
# round-2 baseline: smoke, GPU tests, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2/base_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2/base_smoke.log
timeout 1200 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/base_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/base_tests.log
timeout 1200 python bench.py > gpurun_out/r2/base_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2/base_bench.log
