#!/bin/bash
# full GPU suite + smoke + a short bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2/suite.log 2>&1; echo "rc=$?" >> gpurun_out/r2/suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/r2/bench_quick.json 2> gpurun_out/r2/bench_quick.err; echo "rc=$?" >> gpurun_out/r2/bench_quick.err
