#!/bin/bash
# Final verification after the late round-2 changes: smoke, whole GPU suite, default bench,
# reference arm, a 200-step headline rerun.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2/z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2/z_smoke.log
timeout 1800 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/z_tests.log
timeout 1200 python bench.py > gpurun_out/r2/z_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2/z_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2/z_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2/z_ref.log
timeout 600 python bench.py --steps 200 --warmup 20 --no-extra --no-cpu > gpurun_out/r2/z_bench200.log 2>&1; echo "rc=$?" >> gpurun_out/r2/z_bench200.log
