#!/bin/bash
# quick re-check of a restored tree: smoke, GPU tests, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c_smoke.log
timeout 1200 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c_tests.log
timeout 1200 python bench.py > gpurun_out/c_bench.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench.log
