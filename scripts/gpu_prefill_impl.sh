#!/bin/bash
# prefill: tcgen05 grouped GEMM (default) vs the decode-into-TMEM kernels' prefill configuration
cd $GRAFT_REPO_ROOT
for c in mixtral qwen15 deepseek; do
  timeout 200 python bench.py --config $c --batch 4096 --steps 20 --warmup 3 --no-extra --no-cpu > gpurun_out/pi_gemm_$c.log 2>&1
  PUZZLE_PREFILL_IMPL=tmem timeout 200 python bench.py --config $c --batch 4096 --steps 20 --warmup 3 --no-extra --no-cpu > gpurun_out/pi_tmem_$c.log 2>&1
done
