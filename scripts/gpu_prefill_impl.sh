#!/bin/bash
# prefill: tcgen05 grouped GEMM (default) vs PUZZLE_PREFILL_IMPL alternatives ($@, e.g. pair tmem)
cd $GRAFT_REPO_ROOT
for c in mixtral qwen15 deepseek; do
  timeout 200 python bench.py --config $c --batch 4096 --steps 20 --warmup 3 --no-extra --no-cpu > gpurun_out/pi_gemm_$c.log 2>&1
  for impl in "$@"; do
    PUZZLE_PREFILL_IMPL=$impl timeout 200 python bench.py --config $c --batch 4096 --steps 20 --warmup 3 --no-extra --no-cpu > gpurun_out/pi_${impl}_$c.log 2>&1
  done
done
