#!/bin/bash
# NX 128: half-height activation boxes for positions with <= 64 tokens: parity (bounded), A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_nx64.py -x -q -m gpu > gpurun_out/r2/xhalf_tests.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/r2/xhalf_tests.log
if [ $rc -ne 0 ]; then exit 0; fi
for rep in 1 2; do for v in noxhalf cur; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L timeout 600 python scripts/decode_ab.py mixtral:256 mixtral:384 qwen15:1024 deepseek:768 qwen15:1280 deepseek:1024 > gpurun_out/r2/xhalf_${v}_$rep.log 2>&1
done; done
