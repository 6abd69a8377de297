"""GPU parity for puzzle_moe_forward (route + gate/up/SwiGLU + down + combine) against the
f64 oracle FFN, through the C ABI, under the north-star tolerance (tests/helpers.py)."""
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
    return pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(),
                             torch.from_numpy(w2.view(np.int16)).cuda(),
                             torch.from_numpy(slot).cuda()), (w13, w2, slot)


def _run(pz, cfg, T, path, residual=True, skew=0.0, sample=None, seed_shift=0):
    layer, (w13, w2, slot) = _layer(pz, cfg)
    hb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + seed_shift)
    lg = synth.router_logits(cfg, T, seed=synth.seeds(cfg)["logits"] + seed_shift, skew=skew)
    rb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + 1000 + seed_shift) if residual else None
    h_dev = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    l_dev = torch.from_numpy(lg).cuda()
    r_dev = torch.from_numpy(rb.view(np.int16)).cuda().view(torch.bfloat16) if residual else None
    out = layer.forward(h_dev, l_dev, cfg.top_k, cfg.renormalize, residual=r_dev, path=path)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    rows = np.arange(T) if sample is None else np.sort(np.random.default_rng(7).choice(T, sample, replace=False))
    ref = oracle.moe_forward(w13, w2, slot, hb[rows], lg[rows], cfg.top_k, cfg.renormalize,
                             None if rb is None else rb[rows])
    return got[rows], ref


SMALL = [
    synth.CONFIGS["tiny"],
    synth.MoEConfig("small_mix", 5, 256, 512, 8, 2, True),       # several row blocks, split-K
    synth.MoEConfig("small_fine", 6, 128, 192, 16, 4, False),    # d_ff = 3 x 64 (ragged row blocks)
    synth.MoEConfig("small_k6", 7, 192, 320, 12, 6, False),
]


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: c.name)
@pytest.mark.parametrize("T", [1, 3, 8, 17, 64, 70])
def test_forward_gemv_small(pz, cfg, T):
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV)
    assert_close(got, ref, f"{cfg.name} T={T}")


def test_tiny_config_exact_shape(pz):
    cfg = synth.CONFIGS["tiny"]
    got, ref = _run(pz, cfg, 8, pz.PATH_AUTO, residual=False)
    assert_close(got, ref, "tiny")


@pytest.mark.parametrize("T", [48, 64])
def test_decode_split_item_many_pieces(pz, T):
    """Stream-K reduction with many pieces per item (gemv_tc.cu reducer): one pair and
    d_ff = 8192, so a w2 item (128 rows x 128 K-stages) spans ~16 CTAs of ~8 stages and the
    pieces' slots (up to 64 rows each) exceed the W / X rings -- staged in several rounds
    with the running sum carried in staged slot 0."""
    cfg = synth.MoEConfig("many_pieces", 23, 256, 8192, 2, 1, True)
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV)
    assert_close(got, ref, f"many pieces T={T}")


def test_skewed_routing_all_tokens_one_pair(pz):
    """Every token routed to the same pair (>64 tokens per position: multiple passes)."""
    cfg = synth.MoEConfig("skew", 8, 128, 256, 8, 2, True)
    got, ref = _run(pz, cfg, 150, pz.PATH_GEMV, skew=50.0)
    assert_close(got, ref, "skew")


@pytest.mark.parametrize("T", [7, 37, 64, 300, 1000])  # <= 64: two-grid decode routing; 1000 x 6 > 4096: multi-CTA
def test_route_outputs(pz, T):
    cfg = synth.MoEConfig("route", 9, 64, 64, 64, 6, False)
    layer, (w13, w2, slot) = _layer(pz, cfg)
    lg = synth.router_logits(cfg, T)
    lg[5, 10] = lg[5, 11] = lg[5].max() + 1.0  # an exact tie -> lower index first
    idx, gate, off, tok, aof = layer.route(torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize)
    want_idx, want_gate = oracle.route(lg, cfg.top_k, cfg.renormalize)
    assert np.array_equal(idx.cpu().numpy(), want_idx)
    np.testing.assert_allclose(gate.cpu().numpy(), want_gate, rtol=2e-6, atol=1e-7)
    off = off.cpu().numpy()
    tok = tok.cpu().numpy()
    aof = aof.cpu().numpy()
    buckets = slot[want_idx.reshape(-1)]
    counts = np.bincount(buckets, minlength=2 * cfg.n_pairs)
    assert np.array_equal(np.diff(off), counts) and off[0] == 0
    # assignment (t, j) lands inside its bucket and points back at its token
    for i, a in enumerate(aof):
        b = buckets[i]
        assert off[b] <= a < off[b + 1] and tok[a] == i // cfg.top_k
    assert len(set(aof.tolist())) == T * cfg.top_k


@pytest.mark.parametrize("name", ["qwen15", "deepseek"])
@pytest.mark.parametrize("T", [1, 16, 64])
def test_forward_full_size_fine_grained(pz, name, T):
    """BASELINE config 4 decode at full size: EVERY token of the batch against the oracle
    (all tokens for decode)."""
    cfg = synth.CONFIGS[name]
    got, ref = _run(pz, cfg, T, pz.PATH_AUTO)
    assert_close(got, ref, f"{name} T={T}")


@pytest.mark.slow
@pytest.mark.parametrize("T", [1, 16, 64])
def test_forward_full_size_mixtral(pz, T):
    """BASELINE config 2 (the headline workload at T = 64): every token against the oracle."""
    cfg = synth.CONFIGS["mixtral"]
    got, ref = _run(pz, cfg, T, pz.PATH_AUTO)
    assert_close(got, ref, f"mixtral T={T}")


def test_experts_and_combine_building_blocks(pz):
    """route -> gather -> experts -> combine reproduces forward (the EP decomposition)."""
    cfg = SMALL[1]
    layer, (w13, w2, slot) = _layer(pz, cfg)
    T = 40
    hb = torch.from_numpy(synth.hidden_bits(cfg, T).view(np.int16)).cuda().view(torch.bfloat16)
    lg = torch.from_numpy(synth.router_logits(cfg, T)).cuda()
    full = layer.forward(hb, lg, cfg.top_k, cfg.renormalize)
    idx, gate, off, tok, aof = layer.route(lg, cfg.top_k, cfg.renormalize)
    x_rows = pz.gather_rows(hb, tok)
    y = layer.experts(x_rows, off)
    out = pz.moe_combine(y, aof, gate)
    torch.cuda.synchronize()
    diff = (out.float() - full.float()).abs()
    # identical math; only the (unspecified) order of assignments inside a bucket may differ
    assert diff.max().item() <= 2e-2, (diff.max().item(), int((diff > 0).sum()))


TC_SMALL = [
    synth.MoEConfig("tc_small", 10, 256, 256, 8, 2, True),
    synth.MoEConfig("tc_fine", 11, 512, 384, 16, 4, False),   # d_ff = 3 x 128: ragged n-blocks
]


@pytest.mark.parametrize("cfg", TC_SMALL, ids=lambda c: c.name)
@pytest.mark.parametrize("T", [1, 5, 64, 130, 300])
def test_forward_tc_small(pz, cfg, T):
    got, ref = _run(pz, cfg, T, pz.PATH_TC)
    assert_close(got, ref, f"tc {cfg.name} T={T}")


def test_forward_tc_large_batch_routing(pz):
    """T*k > 4096: multi-CTA routing with the bucket-order row copy fused into the scatter."""
    cfg = TC_SMALL[1]
    got, ref = _run(pz, cfg, 1100, pz.PATH_TC, sample=48)
    assert_close(got, ref, "tc large-batch routing")


def test_forward_tc_skewed_multi_mtile(pz):
    """>256 tokens in one bucket: several 256-row M tiles, partial last tile with <=128 rows."""
    cfg = synth.MoEConfig("tc_skew", 12, 256, 256, 8, 2, True)
    got, ref = _run(pz, cfg, 700, pz.PATH_TC, skew=50.0, sample=64)
    assert_close(got, ref, "tc skew")


def test_tc_matches_gemv_path(pz):
    cfg = TC_SMALL[0]
    layer, _ = _layer(pz, cfg)
    T = 96
    hb = torch.from_numpy(synth.hidden_bits(cfg, T).view(np.int16)).cuda().view(torch.bfloat16)
    lg = torch.from_numpy(synth.router_logits(cfg, T)).cuda()
    a = layer.forward(hb, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_TC).float()
    b = layer.forward(hb, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV).float()
    torch.cuda.synchronize()
    assert (a - b).abs().max().item() <= 2e-2


@pytest.mark.parametrize("name,T", [("qwen15", 512), ("deepseek", 256)])
def test_forward_tc_full_size_fine_grained(pz, name, T):
    cfg = synth.CONFIGS[name]
    got, ref = _run(pz, cfg, T, pz.PATH_TC, sample=16)
    assert_close(got, ref, f"tc {name} T={T}")


@pytest.mark.slow
def test_forward_tc_full_size_mixtral_prefill(pz):
    cfg = synth.CONFIGS["mixtral"]
    got, ref = _run(pz, cfg, 4096, pz.PATH_AUTO, sample=4)
    assert_close(got, ref, "mixtral prefill T=4096")


def test_residual_stack_matches_chained_oracle(pz):
    """BASELINE.json config 5 in miniature: x_{l+1} = x_l + MoE_l(x_l) over 3 layers with
    per-layer logits; the oracle chain is independent (its own bf16-rounded outputs feed it)."""
    base = synth.MoEConfig("stack", 40, 128, 256, 8, 2, True)
    T, n_layers = 24, 3
    x_bits = synth.hidden_bits(base, T, seed=500)
    x_dev = torch.from_numpy(x_bits.view(np.int16)).cuda().view(torch.bfloat16)
    ref_bits = x_bits
    for l in range(n_layers):
        cfg = synth.MoEConfig(f"stack{l}", 41 + l, 128, 256, 8, 2, True)
        layer, (w13, w2, slot) = _layer(pz, cfg)
        lg = synth.router_logits(cfg, T, seed=600 + l)
        x_dev = layer.forward(x_dev, torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize, residual=x_dev)
        ref = oracle.moe_forward(w13, w2, slot, ref_bits, lg, cfg.top_k, cfg.renormalize, ref_bits)
        ref_bits = synth.to_bf16_bits(ref.astype(np.float32))
    torch.cuda.synchronize()
    got = x_dev.float().cpu().numpy().astype(np.float64)
    ref = oracle.bf16_bits_to_f32(ref_bits).astype(np.float64)
    # DESIGN.md R19: both chains round every layer's output to bf16 independently, so besides
    # the single-layer bound each layer may contribute one bf16 ulp of |x| (~2^-8 relative)
    ulp = np.abs(ref) * 2.0 ** -8
    assert np.all(np.abs(got - ref) <= 2e-2 + n_layers * ulp), np.max(np.abs(got - ref) - n_layers * ulp)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 5e-3


def _random_cases(n, tc, seed):
    """Seeded random layer shapes: GEMV path (d, d_ff multiples of 64, any T) or tcgen05 path
    (d % 256, d_ff % 128, T > 64)."""
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        E = int(rng.choice([2, 4, 6, 10, 24, 64]))
        k = int(rng.integers(1, min(8, E) + 1))
        if tc:
            d, f = 256 * int(rng.integers(1, 3)), 128 * int(rng.integers(1, 4))
            T = int(rng.choice([65, 200, 513]))
        else:
            d, f = 64 * int(rng.integers(1, 9)), 64 * int(rng.integers(1, 11))
            T = int(rng.choice([1, 2, 33, 64]))
        cases.append((synth.MoEConfig(f"rnd{'tc' if tc else 'gv'}{i}", 60 + i + (20 if tc else 0), d, f, E, k,
                                      bool(rng.integers(0, 2))), T))
    return cases


@pytest.mark.parametrize("cfg,T", _random_cases(10, False, 11) + _random_cases(6, True, 12),
                         ids=lambda x: x.name if hasattr(x, "name") else str(x))
def test_forward_random_shapes(pz, cfg, T):
    """Random shapes / expert counts / top-k / renormalisation through the path AUTO picks
    (decode GEMV for T <= 64, tcgen05 otherwise): stream-K splits, ragged row blocks, empty and
    single-position pairs, multi-pass buckets."""
    got, ref = _run(pz, cfg, T, pz.PATH_AUTO)
    assert_close(got, ref, f"{cfg.name} d={cfg.d_model} f={cfg.d_ff} E={cfg.n_experts} k={cfg.top_k} T={T}")


# ---- the 25% compression ratio: merged pairs + unmerged dense bf16 slots (reading R20) ----
MIXED = [
    (synth.MoEConfig("mix25_small", 12, 256, 512, 8, 2, True), 2),     # Mixtral-like: 2 pairs + 4 dense
    (synth.MoEConfig("mix25_fine", 13, 256, 384, 16, 4, False), 4),    # 4 pairs + 8 dense
    (synth.MoEConfig("mix25_alldense", 14, 256, 256, 6, 2, True), 0),  # every expert dense
]


def _run_mixed(pz, cfg, n_merged, T, path, seed_shift=0):
    from helpers import oracle_mixed_layer
    w13, w2, slot, dense = oracle_mixed_layer(cfg, n_merged)
    layer = pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(), torch.from_numpy(w2.view(np.int16)).cuda(),
                              torch.from_numpy(slot).cuda(), torch.from_numpy(dense).cuda())
    hb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + seed_shift)
    lg = synth.router_logits(cfg, T, seed=synth.seeds(cfg)["logits"] + seed_shift)
    rb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + 1000 + seed_shift)
    out = layer.forward(torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16), torch.from_numpy(lg).cuda(),
                        cfg.top_k, cfg.renormalize,
                        residual=torch.from_numpy(rb.view(np.int16)).cuda().view(torch.bfloat16), path=path)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, rb, pair_dense=dense)
    return out.float().cpu().numpy(), ref


@pytest.mark.parametrize("case", MIXED, ids=lambda c: c[0].name)
@pytest.mark.parametrize("T", [1, 7, 64, 200])
@pytest.mark.parametrize("path", ["gemv", "tc"])
def test_forward_mixed_dense_slots(pz, case, T, path):
    cfg, n_merged = case
    got, ref = _run_mixed(pz, cfg, n_merged, T, pz.PATH_GEMV if path == "gemv" else pz.PATH_TC)
    assert_close(got, ref, f"{cfg.name} merged={n_merged} T={T} {path}")
