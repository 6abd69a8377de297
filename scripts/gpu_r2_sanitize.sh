#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over small forwards of every
# kernel family (decode GEMV, TS and TC prefill, routing both forms, combine, EP index kernels,
# pack / unpack / merge, calibration statistics): scripts/sanitize_cases.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
python scripts/sanitize_cases.py > gpurun_out/r2/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/r2/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py \
    > gpurun_out/r2/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2/san_$tool.log
done
