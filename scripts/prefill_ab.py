"""A/B of the prefill kernel paths (PUZZLE_PATH_TC vs PUZZLE_PATH_TS) on full-size layers
built on the GPU (bench.build_layer_gpu), L2 flushed between steps; prints per-kernel times
and TFLOP/s of the projection kernels (dense-equivalent 2*3*d*f*T*k).

    python scripts/prefill_ab.py [config:T ...]   (default mixtral:4096 qwen15:4096 deepseek:4096)
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
    cases = sys.argv[1:] or ["mixtral:4096", "qwen15:4096", "deepseek:4096"]
    paths = [p for p in os.environ.get("AB_PATHS", "tc,ts").split(",")]
    for case in cases:
        name, T = case.split(":")
        T = int(T)
        cfg = synth.CONFIGS[name]
        layer, _ = bench.build_layer_gpu(pz, cfg, synth.seeds(cfg)["weights"], dev)
        hidden, logits = bench.make_inputs(cfg, T, synth.seeds(cfg)["activations"], dev)
        flush = torch.empty(2 * bench.l2_bytes(dev), dtype=torch.uint8, device=dev)
        outs = {}
        for p in paths:
            path = {"tc": pz.PATH_TC, "ts": pz.PATH_TS, "gemv": pz.PATH_GEMV}[p]
            out = torch.empty_like(hidden)
            ws = layer.workspace(T, cfg.top_k)
            step = lambda: layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out, workspace=ws, path=path)
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            K = 20
            ms = bench.timed_steps(step, K, lambda: flush.zero_()) / K
            with pz.profile_window() as prof:
                bench.timed_steps(step, K, lambda: flush.zero_())
            kern = {k: round(t / n * 1e3, 2) for k, (n, t) in prof.kernels.items()}
            proj_us = sum(v for k, v in kern.items() if k.startswith("w13") or k.startswith("w2"))
            flops = 2 * 3 * cfg.d_model * cfg.d_ff * T * cfg.top_k
            tf = flops / (proj_us / 1e6) / 1e12
            outs[p] = out.float()
            print(json.dumps({"config": name, "T": T, "path": p, "ms_step": round(ms, 4), "kernel_us": kern,
                              "tflops_proj": round(tf, 1), "frac_bf16_peak": round(tf / pk["bf16_tflops"], 3)}),
                  flush=True)
        if len(outs) > 1:
            ks = list(outs)
            print(json.dumps({"config": name, "T": T, "max_abs_diff": (outs[ks[0]] - outs[ks[1]]).abs().max().item()}))
        del layer
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
