#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -X faulthandler -m pytest tests -m "gpu" -x -q > gpurun_out/t_all.log 2>&1; echo "rc=$?" >> gpurun_out/t_all.log
timeout 1200 python -X faulthandler bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
