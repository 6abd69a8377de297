#!/bin/bash
# end-of-round evidence: smoke, full GPU test suite, default bench, launch lists, ncu captures
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
timeout 1200 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f_tests.log
timeout 1200 python bench.py > gpurun_out/f_bench.log 2>&1; echo "rc=$?" >> gpurun_out/f_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref.log 2>&1; echo "rc=$?" >> gpurun_out/f_ref.log
bash scripts/gpu_profile_next.sh
bash scripts/gpu_profile.sh
bash scripts/gpu_ncu_prefill.sh
