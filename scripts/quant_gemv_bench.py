"""Standalone timing of puzzle_quant_gemv (NEXT-3) through bench.quant_gemv_rates; prints one
JSON line. Used for the ncu captures under profiles/r01 (quant_gemv_*)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402

dev = torch.device("cuda:0")
m = 1 << 28
g = torch.Generator(device=dev).manual_seed(5)
w = torch.rand(m, device=dev, generator=g)
planes = [torch.randint(0, 2, (m,), dtype=torch.uint8, device=dev, generator=g) for _ in range(4)]
print(json.dumps(bench.quant_gemv_rates(pz, w, planes, dev)))
