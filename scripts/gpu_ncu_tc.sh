#!/bin/bash
# ncu --set full of the tcgen05 decode kernels (w13 + w2) at the headline config
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc --launch-skip 6 --launch-count 2 \
  -o gpurun_out/tcgemv -f python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-graph > gpurun_out/ncu_tc.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_tc.log
