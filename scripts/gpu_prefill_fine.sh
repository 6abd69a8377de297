cd $GRAFT_REPO_ROOT
for c in qwen15 deepseek; do
 for impl in "" tmem; do
  PUZZLE_PREFILL_IMPL=$impl timeout 300 python bench.py --config $c --batch 4096 --no-extra --no-cpu --steps 30 --warmup 3 > gpurun_out/pf_${c}_${impl:-tc}.log 2>&1
 done
done
