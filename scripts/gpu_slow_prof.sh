#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/slow.log 2>&1; echo "rc=$?" >> gpurun_out/slow.log
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-graph"
$CMD > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_mixtral64.csv $CMD > gpurun_out/ncu_l.log 2>&1
CMD2="python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-graph --batch 4096"
$CMD2 > gpurun_out/plain_p.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_mixtral4096.csv $CMD2 > gpurun_out/ncu_p.log 2>&1
echo done
