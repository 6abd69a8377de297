#!/bin/bash
# A/B of tuning variants (build/variants/*/libpuzzlemoe.so) on the headline bench; default first
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_moe.py -m gpu -x -q -p no:cacheprovider -k "gemv or decode or skew" > gpurun_out/t_var.log 2>&1; echo "rc=$?" >> gpurun_out/t_var.log
timeout 200 python bench.py --steps 100 --warmup 5 --no-extra --no-cpu > gpurun_out/v_default.log 2>&1
for d in build/variants/*/; do n=$(basename $d)
  PUZZLE_LIB=$d/libpuzzlemoe.so timeout 200 python bench.py --steps 100 --warmup 5 --no-extra --no-cpu > gpurun_out/v_$n.log 2>&1
done
