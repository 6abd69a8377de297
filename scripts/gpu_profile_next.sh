#!/bin/bash
# Profiling evidence for the NEXT rows: each command first runs to exit 0 without ncu, then
#  1. launch list (time + DRAM bytes per launch) of one calibration step (NEXT-4, unmerged
#     Mixtral layer, 4096 tokens) -> the statistics kernel's DRAM traffic;
#  2. ncu --set full of the statistics kernel (h launch);
#  3. launch list of the 25%-ratio Mixtral decode step (NEXT-2, batch 64).
cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
CAL="python scripts/calib_bench.py"
$CAL > gpurun_out/n_cal.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
  -k regex:"k_group_colsumsq|k_tc_experts|k_route|k_combine" --log-file gpurun_out/launches_calib_mixtral4096.csv $CAL > gpurun_out/n_cal_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_group_colsumsq_part --launch-skip 1 --launch-count 1 \
  -o gpurun_out/full_calib -f $CAL > gpurun_out/n_full.log 2>&1
D25="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-graph --ratio 0.25"
$D25 > gpurun_out/n_d25.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_mixtral25_decode64.csv $D25 > gpurun_out/n_d25_ncu.log 2>&1
echo done >> gpurun_out/n_full.log
