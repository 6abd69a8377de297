#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -X faulthandler bench.py --steps 100 --warmup 5 > gpurun_out/bench2.log 2>&1; echo "rc=$?" >> gpurun_out/bench2.log
