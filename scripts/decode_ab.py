"""Decode-shape step timing (CUDA-graph replays back to back, as the headline bench) of the
configs given as config:T, plus per-kernel averages from an eager profile window; packed-
weight GB/s over the step and fraction of the measured HBM peak.

    python scripts/decode_ab.py [config:T ...]   (default mixtral:64 qwen15:64 deepseek:64)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402
import synth  # noqa: E402


def main():
    pz.load_library()
    dev = torch.device("cuda", 0)
    pk = bench.peaks()
    cases = sys.argv[1:] or ["mixtral:64", "qwen15:64", "deepseek:64"]
    for case in cases:
        name, T = case.split(":")
        T = int(T)
        cfg = synth.CONFIGS[name]
        layer, _ = bench.build_layer_gpu(pz, cfg, synth.seeds(cfg)["weights"], dev)
        hidden, logits = bench.make_inputs(cfg, T, synth.seeds(cfg)["activations"], dev)
        out = torch.empty_like(hidden)
        ws = layer.workspace(T, cfg.top_k)
        eager = lambda: layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
        eager()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            eager()
        for _ in range(10):
            g.replay()
        torch.cuda.synchronize()
        K = 100
        ms = bench.timed_steps(g.replay, K) / K
        with pz.profile_window() as prof:
            bench.timed_steps(eager, 30)
        kern = {k: round(t / n * 1e3, 2) for k, (n, t) in prof.kernels.items()}
        nt = bench.touched_pairs(layer, logits, cfg)
        ab = bench.algorithmic_bytes(cfg, nt, T)
        gbs = (ab["w13"] + ab["w2"]) / (ms / 1e3) / 1e9
        if "experts_gemv" in kern:  # one fused launch for both projections
            w13 = w2 = (ab["w13"] + ab["w2"]) / (kern["experts_gemv"] / 1e6) / 1e9
        else:
            w13 = ab["w13"] / (kern.get("w13_gemv", 1e9) / 1e6) / 1e9
            w2 = ab["w2"] / (kern.get("w2_gemv", 1e9) / 1e6) / 1e9
        print(json.dumps({"config": name, "T": T, "ms_step": round(ms, 4), "step_gbs": round(gbs), "frac_step": round(gbs / pk["hbm_gbs"], 3),
                          "w13_frac": round(w13 / pk["hbm_gbs"], 3), "w2_frac": round(w2 / pk["hbm_gbs"], 3), "kernel_us": kern}),
              flush=True)
        del layer, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
