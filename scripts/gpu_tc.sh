#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 240 python -X faulthandler -m pytest -x -q "tests/test_gpu_moe.py::test_forward_tc_small[1-tc_small]" > gpurun_out/tc1.log 2>&1; echo "rc=$?" >> gpurun_out/tc1.log
if grep -q "1 passed\|2 passed" gpurun_out/tc1.log; then
  timeout 400 python -X faulthandler -m pytest tests/test_gpu_moe.py -x -q -k "tc" > gpurun_out/tc2.log 2>&1; echo "rc=$?" >> gpurun_out/tc2.log
fi
timeout 600 python -X faulthandler bench.py --steps 100 --warmup 5 > gpurun_out/bench2.log 2>&1; echo "rc=$?" >> gpurun_out/bench2.log
