#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -k "tc" > gpurun_out/tc.log 2>&1; echo "rc=$?" >> gpurun_out/tc.log
if tail -1 gpurun_out/tc.log | grep -q "rc=0"; then
for c in "mixtral 4096" "qwen15 4096" "deepseek 4096"; do
  set -- $c
  timeout 300 python bench.py --config $1 --batch $2 --steps 20 --warmup 3 --no-cpu --no-extra > gpurun_out/tcb_$1.log 2>&1
done
fi
