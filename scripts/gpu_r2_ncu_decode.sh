#!/bin/bash
# ncu --set full of the decode kernels (one w13 + one w2 launch) at Qwen / DeepSeek B = 64
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for cfg in ${CFGS:-qwen15}; do
  timeout 300 python scripts/decode_ab.py $cfg:64 > gpurun_out/r2/nd_${cfg}_plain.log 2>&1 || { echo "plain failed $cfg"; continue; }
  timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:k_gemv_tc --launch-skip 20 --launch-count 2 -o gpurun_out/r2/full_gemv_${cfg} -f python scripts/decode_ab.py $cfg:64 > gpurun_out/r2/nd_${cfg}_ncu.log 2>&1
  echo rc=$? >> gpurun_out/r2/nd_${cfg}_ncu.log
done
