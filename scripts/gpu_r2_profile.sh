#!/bin/bash
# Round-2 profiling evidence: launch lists of the headline decode step (the bench command the
# driver times) and the Mixtral / Qwen1.5 prefill steps; ncu --set full of the top decode kernel
# and of the TS prefill kernels (tensor-pipe counters); each command first exits 0 without ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
DEC="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-graph"
$DEC > gpurun_out/r2/p_dec.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
  --log-file gpurun_out/r2/launches_mixtral_decode64.csv $DEC > gpurun_out/r2/p_dec_ncu.log 2>&1
for cfg in mixtral qwen15 deepseek; do
  PRE="python bench.py --config $cfg --steps 3 --warmup 3 --no-extra --no-cpu --no-graph --batch 4096"
  $PRE > gpurun_out/r2/p_pre_$cfg.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
    --log-file gpurun_out/r2/launches_${cfg}_prefill4096.csv $PRE > gpurun_out/r2/p_pre_ncu_$cfg.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc --launch-skip 6 --launch-count 2 \
  -o gpurun_out/r2/full_gemv_mixtral64 -f $DEC > gpurun_out/r2/p_full_dec.log 2>&1
for cfg in mixtral qwen15; do
  PRE="python bench.py --config $cfg --steps 3 --warmup 3 --no-extra --no-cpu --no-graph --batch 4096"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ts_experts --launch-skip 6 --launch-count 2 \
    -o gpurun_out/r2/full_ts_${cfg}4096 -f $PRE > gpurun_out/r2/p_full_ts_$cfg.log 2>&1
done
echo done > gpurun_out/r2/p_done.txt
