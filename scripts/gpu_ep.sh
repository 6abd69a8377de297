#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -X faulthandler -m pytest tests/test_gpu_ep.py -x -q > gpurun_out/ep_test.log 2>&1; echo "rc=$?" >> gpurun_out/ep_test.log
# 1-rank torchrun smoke of the EP bench path is not possible (world>1 only); run the world-1 bench quickly
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-extra > gpurun_out/bench_q.log 2>&1; echo "rc=$?" >> gpurun_out/bench_q.log
