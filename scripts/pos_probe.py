"""Decode-kernel probe: w13/w2 GEMV times on the Mixtral layer at batch 64 when the tokens use
both positions of every pair (normal routing), only position 0 or only position 1 (logits of
the other position's experts pushed down) -- separates the per-position cost (MMA + TMEM store
+ epilogue) from the streaming cost."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402
import synth  # noqa: E402

pz.load_library()
dev = torch.device("cuda:0")
cfg = synth.CONFIGS["mixtral"]
layer, _ = bench.build_layer_gpu(pz, cfg, synth.seeds(cfg)["weights"], dev)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
hidden, logits = bench.make_inputs(cfg, T, synth.seeds(cfg)["activations"], dev)
slot = layer.expert_slot.cpu()
res = {}
for name, keep in (("both", None), ("pos0", 0), ("pos1", 1)):
    lg = logits.clone()
    if keep is not None:
        for e in range(cfg.n_experts):
            if int(slot[e]) % 2 != keep:
                lg[:, e] -= 100.0
    out = torch.empty_like(hidden)
    ws = layer.workspace(T, cfg.top_k)
    step = lambda: layer.forward(hidden, lg, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    with pz.profile_window() as prof:
        bench.timed_steps(step, 50)
    k = {n: round(t / c * 1000, 1) for n, (c, t) in prof.kernels.items()}
    res[name] = {"touched_pairs": bench.touched_pairs(layer, lg, cfg), "kernel_us": k}
print(json.dumps(res))
