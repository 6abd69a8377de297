"""Small invocations of every kernel family of libpuzzlemoe for compute-sanitizer
(scripts/gpu_r2_sanitize.sh): decode GEMV (single + multi pass, dense slots), TS and TC prefill,
both routing forms, combine, the fixed-capacity EP index kernels and the peer-memory EP kernels
(simulated 2-rank world in one process, buffers in one allocation), pack / unpack / fused merge,
calibration statistics. Each forward is checked against the oracle (north-star tolerance) so
the sanitizer run is also a correctness run; exit code 0 = every check passed."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402
import synth  # noqa: E402
from helpers import assert_close, oracle_mixed_layer, oracle_packed_layer  # noqa: E402


def layer_of(cfg):
    w13, w2, slot, _ = oracle_packed_layer(cfg)
    return pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(), torch.from_numpy(w2.view(np.int16)).cuda(),
                             torch.from_numpy(slot).cuda()), (w13, w2, slot)


def forward_case(cfg, T, path, residual=True):
    layer, (w13, w2, slot) = layer_of(cfg)
    hb = synth.hidden_bits(cfg, T)
    lg = synth.router_logits(cfg, T)
    rb = synth.hidden_bits(cfg, T, seed=99) if residual else None
    h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    r = torch.from_numpy(rb.view(np.int16)).cuda().view(torch.bfloat16) if residual else None
    out = layer.forward(h, torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize, residual=r, path=path)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, rb)
    assert_close(out.float().cpu().numpy(), ref, f"{cfg.name} T={T} path={path}")
    print("ok forward", cfg.name, T, path, flush=True)


def main():
    pz.load_library()
    small = synth.MoEConfig("san_small", 5, 256, 512, 8, 2, True)
    fine = synth.MoEConfig("san_fine", 6, 128, 192, 16, 4, False)
    forward_case(synth.CONFIGS["tiny"], 8, pz.PATH_AUTO)
    forward_case(small, 1, pz.PATH_GEMV)
    forward_case(small, 64, pz.PATH_GEMV)                 # decode routing, stream-K splits
    forward_case(small, 150, pz.PATH_GEMV)                # multi-pass, large-batch routing
    forward_case(fine, 33, pz.PATH_GEMV)
    forward_case(small, 300, pz.PATH_TS)                  # TS prefill, 2-CTA clusters
    forward_case(small, 300, pz.PATH_TC)                  # shared-memory-operand prefill
    forward_case(synth.MoEConfig("san_ts", 7, 384, 192, 12, 3, False), 200, pz.PATH_TS)
    # 25 % layout: dense bf16 slots
    cfg = synth.MoEConfig("san_mix", 12, 256, 512, 8, 2, True)
    w13, w2, slot, dense = oracle_mixed_layer(cfg, 2)
    lay = pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(), torch.from_numpy(w2.view(np.int16)).cuda(),
                            torch.from_numpy(slot).cuda(), torch.from_numpy(dense).cuda())
    for T, path in ((7, pz.PATH_GEMV), (200, pz.PATH_TS)):
        hb, lg = synth.hidden_bits(cfg, T), synth.router_logits(cfg, T)
        out = lay.forward(torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16), torch.from_numpy(lg).cuda(),
                          cfg.top_k, cfg.renormalize, path=path)
        torch.cuda.synchronize()
        assert_close(out.float().cpu().numpy(), oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize,
                                                                   pair_dense=dense), "dense slots")
        print("ok dense slots", T, path, flush=True)
    # calibration statistics (NEXT-4)
    layer, (w13, w2, slot) = layer_of(small)
    T = 40
    hb, lg = synth.hidden_bits(small, T), synth.router_logits(small, T)
    sx = torch.zeros((2 * small.n_pairs, small.d_model), dtype=torch.float64, device="cuda")
    sh = torch.zeros((2 * small.n_pairs, small.d_ff), dtype=torch.float64, device="cuda")
    layer.forward_calib(torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16), torch.from_numpy(lg).cuda(),
                        small.top_k, small.renormalize, sx, sh)
    torch.cuda.synchronize()
    ref_x, _ = oracle.calib_sumsq(w13, slot, hb, lg, small.top_k, small.renormalize)
    assert np.allclose(sx.cpu().numpy(), ref_x, rtol=1e-9, atol=1e-9)
    print("ok calib", flush=True)
    # pack / unpack / fused merge (bit-exact)
    w_i, w_j, n_i, n_j = synth.expert_pair_slot(small, 0, "w1")
    art = oracle.merge(w_i, w_j, n_i, n_j, 0.4)
    want, _ = oracle.pack_artifacts(art)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    got = pz.merge_pack(t(art["w_merged"]), t(art["m_i"]), t(art["m_j"]), t(art["s_i"]), t(art["s_j"]))
    assert np.array_equal(got.cpu().numpy().view(np.uint16), want)
    for pos in (0, 1):
        dec = pz.unpack(got, pos).view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(dec, oracle.unpack(want, pos))
    got2 = pz.merge_experts_pack(t(w_i).to(torch.bfloat16), t(w_j).to(torch.bfloat16), t(n_i), t(n_j), 0.4)
    assert np.array_equal(got2.cpu().numpy().view(np.uint16).reshape(want.shape), want)
    print("ok pack/unpack/merge", flush=True)
    # fixed-capacity EP index kernels + peer-memory kernels: simulated 2-rank world in one
    # process (tests/test_gpu_ep.py drives the same; here only to exercise the kernels)
    import subprocess
    rc = subprocess.call([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          os.path.join(ROOT, "tests", "test_gpu_ep.py"), "-k",
                          "simulated_world"])
    assert rc == 0, "EP simulated-world cases"
    print("ok ep", flush=True)
    print("all sanitizer cases passed")


if __name__ == "__main__":
    main()
