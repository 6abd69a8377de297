#!/bin/bash
# the compute-sanitizer substitute: the sanitizer cases and the whole GPU test suite against the
# checked build (-DPZ_CHECKED: device invariant checks that trap)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
export PUZZLE_LIB=build/variants/checked/libpuzzlemoe.so
timeout 900 python scripts/sanitize_cases.py > gpurun_out/r2/checked_cases.log 2>&1; echo "rc=$?" >> gpurun_out/r2/checked_cases.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/checked_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2/checked_tests.log
