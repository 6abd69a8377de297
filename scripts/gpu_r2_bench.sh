#!/bin/bash
# default bench + the 1-rank EP path (C-ABI transport, self-check, strong-scaling aux)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 1500 python bench.py > gpurun_out/r2/b_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2/b_full.log
timeout 600 python bench.py --ep1 --steps 50 --warmup 5 --no-cpu > gpurun_out/r2/b_ep1.log 2>&1; echo "rc=$?" >> gpurun_out/r2/b_ep1.log
