#!/bin/bash
cd $GRAFT_REPO_ROOT
python scripts/tune_gemv.py mixtral 64 1,2,4 4,7,14 3,4 > gpurun_out/tune_mix64.txt 2>&1
python scripts/tune_gemv.py qwen15 64 1,2,4 1,2,4 1,2 > gpurun_out/tune_qwen64.txt 2>&1
python scripts/tune_gemv.py qwen15 1 4,8,16 4,8,11 1 > gpurun_out/tune_qwen1.txt 2>&1
