#!/bin/bash
# tcgen05 decode-GEMV bring-up: parity tests, then headline bench for both implementations
cd $GRAFT_REPO_ROOT
timeout 600 python -X faulthandler -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t_tc.log 2>&1; echo "rc=$?" >> gpurun_out/t_tc.log
timeout 300 python bench.py --steps 100 --warmup 5 --no-extra --no-cpu > gpurun_out/b_tc.log 2>&1; echo "rc=$?" >> gpurun_out/b_tc.log

