"""GPU edge cases of the forward against the oracle (through the C ABI): empty batches, every
expert selected, exact logit ties, repeated calls on one workspace (stream-K counters and the
route scratch are reset by the kernels themselves), a 512-expert router."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_close, oracle_packed_layer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    import paper_2511_04805_b200 as pz
    pz.load_library()
    return pz


def _layer(pz, cfg):
    w13, w2, slot, _ = oracle_packed_layer(cfg)
    layer = pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(), torch.from_numpy(w2.view(np.int16)).cuda(),
                              torch.from_numpy(slot).cuda())
    return layer, w13, w2, slot


def _dev_bits(bits):
    return torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)


def test_empty_batch_is_a_noop(pz):
    cfg = synth.MoEConfig("edge0", 40, 256, 256, 8, 2, True)
    layer, *_ = _layer(pz, cfg)
    hidden = torch.empty((0, cfg.d_model), dtype=torch.bfloat16, device="cuda")
    logits = torch.empty((0, cfg.n_experts), dtype=torch.float32, device="cuda")
    for path in (pz.PATH_GEMV, pz.PATH_TC):
        out = layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, path=path)
        assert out.shape == (0, cfg.d_model)


@pytest.mark.parametrize("path", ["gemv", "tc"])
@pytest.mark.parametrize("T", [3, 64, 150])
def test_every_expert_selected(pz, path, T):
    cfg = synth.MoEConfig("edge_all", 41, 256, 256, 6, 6, False)  # top_k == n_experts
    layer, w13, w2, slot = _layer(pz, cfg)
    hb = synth.hidden_bits(cfg, T, seed=410)
    lg = synth.router_logits(cfg, T, seed=411)
    out = layer.forward(_dev_bits(hb), torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize,
                        path=pz.PATH_GEMV if path == "gemv" else pz.PATH_TC)
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize)
    assert_close(out.float().cpu().numpy(), ref, f"all experts {path} T={T}")


@pytest.mark.parametrize("T", [5, 64, 200])
def test_exact_logit_ties(pz, T):
    """All logits equal: the lowest expert ids win (R13) and the gates are uniform."""
    cfg = synth.MoEConfig("edge_tie", 42, 256, 256, 8, 2, True)
    layer, w13, w2, slot = _layer(pz, cfg)
    hb = synth.hidden_bits(cfg, T, seed=420)
    lg = np.zeros((T, cfg.n_experts), np.float32)
    lg[T // 2:, 3:] = 0.5  # second half: a tie among experts 3..7
    idx, gate, *_ = layer.route(torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize)
    want_idx, want_gate = oracle.route(lg, cfg.top_k, cfg.renormalize)
    assert np.array_equal(idx.cpu().numpy(), want_idx)
    np.testing.assert_allclose(gate.cpu().numpy(), want_gate, rtol=1e-6)
    out = layer.forward(_dev_bits(hb), torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize)
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize)
    assert_close(out.float().cpu().numpy(), ref, f"ties T={T}")


def test_repeated_calls_share_one_workspace(pz):
    """Decode batches of different sizes through one workspace: each call resets its own
    counters, so every result equals a fresh call bit for bit (the decode path is
    deterministic: fixed stream-K cuts and summation order)."""
    cfg = synth.MoEConfig("edge_rep", 43, 256, 512, 8, 2, True)
    layer, w13, w2, slot = _layer(pz, cfg)
    ws = layer.workspace(64, cfg.top_k)
    seq = [64, 3, 64, 1, 17, 64, 64]
    outs = []
    for i, T in enumerate(seq):
        hb = synth.hidden_bits(cfg, T, seed=430 + T)
        lg = synth.router_logits(cfg, T, seed=440 + T)
        outs.append(layer.forward(_dev_bits(hb), torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize,
                                  workspace=ws).clone())
    torch.cuda.synchronize()
    for T, o in zip(seq, outs):
        hb = synth.hidden_bits(cfg, T, seed=430 + T)
        lg = synth.router_logits(cfg, T, seed=440 + T)
        fresh_ws = torch.zeros_like(ws)
        fresh = layer.forward(_dev_bits(hb), torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize,
                              workspace=fresh_ws)
        assert torch.equal(o.view(torch.int16), fresh.view(torch.int16)), T
    ref = oracle.moe_forward(w13, w2, slot, synth.hidden_bits(cfg, 17, seed=447),
                             synth.router_logits(cfg, 17, seed=457), cfg.top_k, cfg.renormalize)
    assert_close(outs[4].float().cpu().numpy(), ref, "repeat T=17")


@pytest.mark.parametrize("T", [1, 40, 700])
def test_router_512_experts(pz, T):
    """The largest supported router (E = 512, 256 pairs; k = 8): indices bit-exact, gates."""
    cfg = synth.MoEConfig("edge512", 44, 64, 64, 512, 8, False)
    P = cfg.n_pairs
    slot = torch.from_numpy(synth.pairing(cfg)[1]).cuda()
    anchor = torch.zeros(64, dtype=torch.int16, device="cuda")
    rl = pz.RoutingLayer(P, cfg.d_model, cfg.d_ff, slot, anchor)
    lg = synth.router_logits(cfg, T, seed=450)
    idx, gate, off, tok, aof = rl.route(torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize)
    want_idx, want_gate = oracle.route(lg, cfg.top_k, cfg.renormalize)
    assert np.array_equal(idx.cpu().numpy(), want_idx)
    np.testing.assert_allclose(gate.cpu().numpy(), want_gate, rtol=2e-6, atol=1e-8)
    counts = np.bincount(synth.pairing(cfg)[1][want_idx.reshape(-1)], minlength=2 * P)
    assert np.array_equal(np.diff(off.cpu().numpy()), counts)


@pytest.mark.parametrize("name,T", [("mixtral", 64), ("mixtral", 4096), ("qwen15", 64)])
def test_graph_replay_matches_eager_full_size(pz, name, T):
    """bench.py times CUDA-graph replays of the whole forward at the BASELINE sizes: a replay
    must reproduce the eager call (bit for bit on the deterministic decode path), and sampled
    rows must match the oracle (oracle-packed weights, seeded inputs)."""
    cfg = synth.CONFIGS[name]
    layer, w13, w2, slot = _layer(pz, cfg)
    hb = synth.hidden_bits(cfg, T, seed=460)
    lg = synth.router_logits(cfg, T, seed=461)
    hidden, logits = _dev_bits(hb), torch.from_numpy(lg).cuda()
    ws = layer.workspace(T, cfg.top_k)
    eager = layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, workspace=ws).clone()
    out = torch.empty_like(hidden)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    if T <= 64:
        assert torch.equal(out.view(torch.int16), eager.view(torch.int16))
    else:  # prefill: the in-bucket order (R18) may move a row between tiles; same math
        assert (out.float() - eager.float()).abs().max().item() <= 2e-2
    rows = np.sort(np.random.default_rng(5).choice(T, 4, replace=False))
    ref = oracle.moe_forward(w13, w2, slot, hb[rows], lg[rows], cfg.top_k, cfg.renormalize)
    assert_close(out.float().cpu().numpy()[rows], ref, f"graph {name} T={T}")
