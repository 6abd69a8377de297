#!/bin/bash
# iteration: gpu tests (fast subset first), then bench
cd $GRAFT_REPO_ROOT
[ -x scripts/micro/hmma_rate ] && ./scripts/micro/hmma_rate > gpurun_out/hmma_rate.txt 2>&1
timeout 300 python -X faulthandler -m pytest tests/test_gpu_moe.py -x -q -k "gemv_small or tiny or skew or building" > gpurun_out/t1.log 2>&1; echo "rc=$?" >> gpurun_out/t1.log
if tail -1 gpurun_out/t1.log | grep -q "rc=0"; then
  timeout 900 python -X faulthandler bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
  if [ "$FULL" = "1" ]; then
    timeout 900 python -X faulthandler -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/t2.log 2>&1; echo "rc=$?" >> gpurun_out/t2.log
  fi
fi
