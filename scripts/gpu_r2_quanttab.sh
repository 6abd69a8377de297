#!/bin/bash
# NEXT-3 byte-table decode: quantised-class parity, then rate A/B vs the library before it (old).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_quant_forward.py tests/test_gpu_quant.py -x -q -m gpu > gpurun_out/r2/qtab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/qtab_tests.log
for rep in 1 2; do for v in old cur; do
  if [ $v = cur ]; then L=""; else L="PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so"; fi
  env $L timeout 600 python scripts/quant_rate.py > gpurun_out/r2/qtab_${v}_$rep.log 2>&1
done; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc --launch-skip 6 --launch-count 2 \
  -o gpurun_out/r2/full_gemv_quant_tab -f python scripts/quant_rate.py > gpurun_out/r2/qtab_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2/qtab_ncu.log
