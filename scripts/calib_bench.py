"""Run bench.calib_run alone (NEXT-4 calibration statistics on the unmerged Mixtral layer)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402

pz.load_library()
dev = torch.device("cuda:0")
print(json.dumps(bench.calib_run(pz, None, dev, bench.peaks())))
