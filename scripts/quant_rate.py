"""NEXT-3 quantised forward rates (bench.quant_forward_rates) next to the packed forward."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402

pz.load_library()
for r in bench.quant_forward_rates(pz, torch.device("cuda", 0), bench.peaks()):
    print(json.dumps(r))
