#!/bin/bash
cd $GRAFT_REPO_ROOT
PUZZLE_LIB=build/variants/trace/libpuzzlemoe.so timeout 300 python scripts/trace_gemv.py ${1:-mixtral} ${2:-64} ${3:-} > gpurun_out/trace.log 2>&1; echo "rc=$?" >> gpurun_out/trace.log
