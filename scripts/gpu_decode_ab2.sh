#!/bin/bash
# decode A/B, two rounds (suffix r1/r2) of default vs build/variants/* on three decode configs
cd $GRAFT_REPO_ROOT
for r in r1 r2; do
for cb in ${AB_CONFIGS:-"mixtral 64" "qwen15 64" "deepseek 64"}; do set -- $cb
  timeout 200 python bench.py --config $1 --batch $2 --steps 100 --warmup 5 --no-extra --no-cpu > gpurun_out/da_default_$1_$2_$r.log 2>&1
  for d in build/variants/*/; do [ -d "$d" ] || continue; n=$(basename $d); case $n in trace*|tctrace) continue;; esac
    PUZZLE_LIB=$d/libpuzzlemoe.so timeout 200 python bench.py --config $1 --batch $2 --steps 100 --warmup 5 --no-extra --no-cpu > gpurun_out/da_${n}_$1_$2_$r.log 2>&1
  done
done
done
