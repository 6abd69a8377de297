#!/bin/bash
# NEXT-4 calibration statistics: parity tests + timing of the default build and every variant;
# route tests (scatter) and a prefill bench line
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_calib.py tests/test_gpu_moe.py -q -x -k "calib or route or tc_small or mixed" > gpurun_out/t_calib.log 2>&1; echo rc=$? >> gpurun_out/t_calib.log
timeout 300 python scripts/calib_bench.py > gpurun_out/cb_default.log 2>&1
for d in build/variants/*/; do [ -d "$d" ] || continue; n=$(basename $d)
  PUZZLE_LIB=$d/libpuzzlemoe.so timeout 300 python scripts/calib_bench.py > gpurun_out/cb_$n.log 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --no-cpu --batch 4096 > gpurun_out/b_pre.log 2>&1
