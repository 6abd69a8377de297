"""NEXT-1 fused merge + pack (puzzle_merge_experts_pack) rate on a Mixtral w1 slot: 4 pairs x
[14336, 4096] bf16 experts; algorithmic bytes 6 per element (W_i, W_j in, packed word out)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402

pz.load_library()
dev = torch.device("cuda", 0)
wi = (torch.randn(4, 14336, 4096, device=dev) * 0.0156).to(torch.bfloat16)
wj = (torch.randn(4, 14336, 4096, device=dev) * 0.0156).to(torch.bfloat16)
ni = 1 + torch.randn(4, 4096, device=dev).abs()
nj = 1 + torch.randn(4, 4096, device=dev).abs()
st = pz.new_stats(dev)
mo = pz.merge_experts_pack(wi, wj, ni, nj, 0.4, stats=st)
torch.cuda.synchronize()
ms = bench.timed_steps(lambda: pz.merge_experts_pack(wi, wj, ni, nj, 0.4, out=mo, stats=st), 10) / 10
gbs = wi.numel() * 6 / (ms / 1e3) / 1e9
print(f"merge+pack {wi.numel()} elems: {ms:.3f} ms, {gbs:.0f} GB/s = {gbs / bench.peaks()['hbm_gbs']:.3f} of measured HBM; stats {st.cpu().tolist()}")
