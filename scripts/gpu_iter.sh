#!/bin/bash
# one iteration: GPU parity tests, headline bench (+ variants), pipeline traces (trace* variants)
cd $GRAFT_REPO_ROOT
if [ "${SKIP_TESTS:-0}" = 0 ]; then
timeout 600 python -X faulthandler -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t_it.log 2>&1; echo "rc=$?" >> gpurun_out/t_it.log
fi
timeout 200 python bench.py --steps 100 --warmup 5 --no-extra --no-cpu > gpurun_out/v_default.log 2>&1
for d in build/variants/*/; do [ -d "$d" ] || continue; n=$(basename $d)
  case $n in
    trace*) PUZZLE_LIB=$d/libpuzzlemoe.so timeout 300 python scripts/trace_gemv.py mixtral 64 > gpurun_out/$n.log 2>&1 ;;
    *) PUZZLE_LIB=$d/libpuzzlemoe.so timeout 200 python bench.py --steps 100 --warmup 5 --no-extra --no-cpu > gpurun_out/v_$n.log 2>&1 ;;
  esac
done
