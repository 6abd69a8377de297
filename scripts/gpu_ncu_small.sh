#!/bin/bash
# ncu --set full of the small kernels around the decode GEMVs (route / gather / combine) at a
# fine-grained decode config
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config ${1:-qwen15} --batch ${2:-64} --steps 3 --warmup 3 --no-extra --no-cpu --no-graph"
$CMD > gpurun_out/s_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"k_route_small|k_gather_rows|k_combine" --launch-skip 9 --launch-count 3 -o gpurun_out/small -f $CMD > gpurun_out/s_ncu.log 2>&1
echo rc=$? >> gpurun_out/s_ncu.log
