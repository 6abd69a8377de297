#!/bin/bash
# After the NX = 64 configuration: smoke, whole GPU suite, default bench, back-to-back decode
# replays at intermediate batches, launch list + one ncu --set full capture of the NX = 64 kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2/v_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2/v_smoke.log
timeout 1800 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/v_tests.log
timeout 1200 python bench.py > gpurun_out/r2/v_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2/v_bench.log
timeout 600 python scripts/decode_ab.py mixtral:64 mixtral:128 mixtral:192 qwen15:64 qwen15:512 qwen15:768 deepseek:64 deepseek:512 > gpurun_out/r2/v_decode_ab.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2/v_launches_mixtral128.csv python scripts/decode_ab.py mixtral:128 > gpurun_out/r2/v_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc --launch-skip 20 --launch-count 2 \
  -o gpurun_out/r2/full_gemv_nx64_mixtral128 -f python scripts/decode_ab.py mixtral:128 > gpurun_out/r2/v_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2/v_ncu.log
