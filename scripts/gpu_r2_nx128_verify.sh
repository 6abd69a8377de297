#!/bin/bash
# After the NX = 128 configuration and the new AUTO thresholds: smoke, whole GPU suite, default
# bench, AUTO intermediate sweep (back-to-back replays), launch list + ncu --set full of NX 128.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2/w_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2/w_smoke.log
timeout 1800 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/w_tests.log
timeout 1200 python bench.py > gpurun_out/r2/w_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2/w_bench.log
timeout 600 python scripts/decode_ab.py mixtral:64 mixtral:128 mixtral:256 mixtral:384 qwen15:64 qwen15:512 qwen15:1024 deepseek:64 deepseek:512 deepseek:768 > gpurun_out/r2/w_decode_ab.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2/w_launches_mixtral256.csv python scripts/decode_ab.py mixtral:256 > gpurun_out/r2/w_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc --launch-skip 20 --launch-count 2 \
  -o gpurun_out/r2/full_gemv_nx128_mixtral256 -f python scripts/decode_ab.py mixtral:256 > gpurun_out/r2/w_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2/w_ncu.log
