#!/bin/bash
# ncu --set full of the TS prefill kernels (one w13 + one w2 launch) at Qwen / DeepSeek T = 4096
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for cfg in ${CFGS:-qwen15 deepseek}; do
  AB_PATHS=ts python scripts/prefill_ab.py $cfg:4096 > gpurun_out/r2/nts_${cfg}_plain.log 2>&1 || { echo "plain failed $cfg"; continue; }
  AB_PATHS=ts timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:k_ts_experts --launch-skip 6 --launch-count 2 -o gpurun_out/r2/full_ts_${cfg} -f python scripts/prefill_ab.py $cfg:4096 > gpurun_out/r2/nts_${cfg}_ncu.log 2>&1
  echo rc=$? >> gpurun_out/r2/nts_${cfg}_ncu.log
done
