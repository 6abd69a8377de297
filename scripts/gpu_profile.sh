#!/bin/bash
# Profiling evidence (profiles/): each command first runs to exit 0 without ncu, then
#  1. launch lists (gpu__time_duration + dram bytes per launch, cold-cache, serialised) of the
#     headline decode step and a prefill step;
#  2. one ncu --set full capture of each decode kernel (w13, w2) at the headline config.
cd $GRAFT_REPO_ROOT
DEC="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-graph"
PRE="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-graph --batch 4096"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
$DEC > gpurun_out/p_dec.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_mixtral_decode64.csv $DEC > gpurun_out/p_dec_ncu.log 2>&1
$PRE > gpurun_out/p_pre.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_mixtral_prefill4096.csv $PRE > gpurun_out/p_pre_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc --launch-skip 6 --launch-count 2 \
  -o gpurun_out/full_gemv_tc -f $DEC > gpurun_out/p_full.log 2>&1
echo done >> gpurun_out/p_full.log
