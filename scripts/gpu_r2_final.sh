#!/bin/bash
# final verification: smoke, whole GPU suite, default bench (twice), reference arm, EP 1-rank aux
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2/f_smoke.log
timeout 1800 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/f_tests.log
timeout 1200 python bench.py > gpurun_out/r2/f_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2/f_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2/f_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2/f_ref.log
timeout 600 python bench.py --steps 200 --warmup 20 --no-extra --no-cpu > gpurun_out/r2/f_bench200.log 2>&1; echo "rc=$?" >> gpurun_out/r2/f_bench200.log
