#!/bin/bash
# Launch list of the expert-parallel decode step (fixed-capacity dispatch) in a 1-rank NCCL
# group: every kernel of one EP layer forward (route, ep_dispatch, NCCL all-to-alls,
# ep_recv_plan, gathers, decode experts, ep_home_index, combine), cold-cache and serialised.
cd $GRAFT_REPO_ROOT
EP="python bench.py --ep1 --steps 3 --warmup 3 --no-extra --no-cpu --no-graph"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
$EP > gpurun_out/p_ep.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_ep1_fixed_decode64.csv $EP > gpurun_out/p_ep_ncu.log 2>&1
echo rc=$? >> gpurun_out/p_ep_ncu.log
