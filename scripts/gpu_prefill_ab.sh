#!/bin/bash
# prefill A/B: default build vs each build/variants/* on the three prefill configs
cd $GRAFT_REPO_ROOT
for c in mixtral qwen15 deepseek; do
  timeout 200 python bench.py --config $c --batch 4096 --steps 20 --warmup 3 --no-extra --no-cpu > gpurun_out/pf_default_$c.log 2>&1
  for d in build/variants/*/; do [ -d "$d" ] || continue; n=$(basename $d); case $n in trace*|tctrace) continue;; esac
    PUZZLE_LIB=$d/libpuzzlemoe.so timeout 200 python bench.py --config $c --batch 4096 --steps 20 --warmup 3 --no-extra --no-cpu > gpurun_out/pf_${n}_$c.log 2>&1
  done
done
