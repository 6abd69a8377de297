#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2
for v in head headE8 nolamE8 nopairE8; do
  AB_PATHS=ts PUZZLE_LIB=build/variants/$v/libpuzzlemoe.so timeout 600 python scripts/prefill_ab.py mixtral:256 mixtral:4096 qwen15:4096 > gpurun_out/r2/pair2_$v.log 2>&1
done
