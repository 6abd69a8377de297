"""NEXT-3 on the tensor cores: the MoE forward over the quantised weight class
(puzzle_moe_forward_quant: the decode-shape kernels decode the code bytes into the tcgen05 A
operand, both experts of a pair from one read) against the oracle: every expert's weights
dequantised by the pinned oracle.quant_unpack (R23) and run as dense bf16 slots through the
pinned oracle forward (R20 dense-slot form, f64 accumulation), under the north-star tolerance."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    import paper_2511_04805_b200 as pz
    pz.load_library()
    return pz


_cache = {}


def quant_layer(cfg):
    """Oracle merge + oracle quant_pack per projection; plus the dequantised dense reference."""
    if cfg in _cache:
        return _cache[cfg]
    _, slot = synth.pairing(cfg)
    P, d, f = cfg.n_pairs, cfg.d_model, cfg.d_ff
    c13 = np.empty((P, 2, f, d), np.uint8)
    s13 = np.empty((P, 2, f, d // 128), np.float32)
    c2 = np.empty((P, d, f), np.uint8)
    s2 = np.empty((P, d, f // 128), np.float32)
    for p in range(P):
        for name in synth.SLOTS:
            art = oracle.merge(*synth.expert_pair_slot(cfg, p, name), 0.4)
            codes, scales = oracle.quant_pack(art["w_merged"], art["m_i"], art["m_j"], art["s_i"], art["s_j"])
            if name == "w1":
                c13[p, 0], s13[p, 0] = codes, scales
            elif name == "w3":
                c13[p, 1], s13[p, 1] = codes, scales
            else:
                c2[p], s2[p] = codes, scales
    # reference layout: every (pair, pos) a dense slot 2 p + pos holding the dequantised expert
    w13_ref = np.empty((2 * P, 2, f, d), np.uint16)
    w2_ref = np.empty((2 * P, d, f), np.uint16)
    for p in range(P):
        for pos in (0, 1):
            for j in (0, 1):
                w13_ref[2 * p + pos, j] = oracle.quant_unpack(c13[p, j], s13[p, j], pos)
            w2_ref[2 * p + pos] = oracle.quant_unpack(c2[p], s2[p], pos)
    slot_ref = (2 * slot).astype(np.int32)  # expert at (p, pos) -> dense slot 2 p + pos, position 0
    dense = np.ones(2 * P, np.uint8)
    _cache[cfg] = (c13, s13, c2, s2, slot), (w13_ref, w2_ref, slot_ref, dense)
    return _cache[cfg]


def _run(pz, cfg, T, seed=0):
    (c13, s13, c2, s2, slot), (w13r, w2r, slotr, dense) = quant_layer(cfg)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    layer = pz.QuantMoELayer(t(c13), t(s13), t(c2), t(s2), t(slot))
    hb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + seed)
    lg = synth.router_logits(cfg, T, seed=synth.seeds(cfg)["logits"] + seed)
    rb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + 500 + seed)
    out = layer.forward(t(hb.view(np.int16)).view(torch.bfloat16), t(lg), cfg.top_k, cfg.renormalize,
                        residual=t(rb.view(np.int16)).view(torch.bfloat16))
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13r, w2r, slotr, hb, lg, cfg.top_k, cfg.renormalize, rb, pair_dense=dense)
    return out.float().cpu().numpy(), ref


CFGS = [synth.MoEConfig("q_small", 20, 256, 512, 8, 2, True),
        synth.MoEConfig("q_fine", 21, 128, 384, 16, 4, False),
        synth.MoEConfig("q_k6", 22, 384, 256, 12, 6, False)]


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("T", [1, 5, 16, 64, 100])
def test_quant_forward_matches_oracle(pz, cfg, T):
    got, ref = _run(pz, cfg, T)
    assert_close(got, ref, f"quant {cfg.name} T={T}")


def test_quant_forward_split_item_many_pieces(pz):
    """The reducer's multi-round staging with the quantised class's smaller rings (72 KB):
    one pair, d_ff = 8192 (w2 items of 128 K-stages over CTAs of ~8 stages)."""
    cfg = synth.MoEConfig("q_many_pieces", 24, 256, 8192, 2, 1, True)
    got, ref = _run(pz, cfg, 64)
    assert_close(got, ref, "quant many pieces")


def test_quant_forward_skewed_multi_pass(pz):
    """One pair takes most tokens: several passes of 32 per position, split work items."""
    cfg = CFGS[0]
    (c13, s13, c2, s2, slot), (w13r, w2r, slotr, dense) = quant_layer(cfg)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    layer = pz.QuantMoELayer(t(c13), t(s13), t(c2), t(s2), t(slot))
    T = 90
    hb = synth.hidden_bits(cfg, T)
    lg = synth.router_logits(cfg, T, skew=50.0)
    out = layer.forward(t(hb.view(np.int16)).view(torch.bfloat16), t(lg), cfg.top_k, cfg.renormalize)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13r, w2r, slotr, hb, lg, cfg.top_k, cfg.renormalize, pair_dense=dense)
    assert_close(out.float().cpu().numpy(), ref, "quant skewed")


@pytest.mark.parametrize("name,T", [("qwen15", 64), ("deepseek", 16)])
def test_quant_forward_full_size_fine_grained(pz, name, T):
    """BASELINE config 4 shapes, every token."""
    got, ref = _run(pz, synth.CONFIGS[name], T)
    assert_close(got, ref, f"quant {name} T={T}")


def test_quant_forward_rejects_bad_layers(pz):
    import ctypes
    d = pz.QuantLayerDesc(8, 4, 4096 + 64, 14336, 4096, 4096, 4096, 4096, 4096)  # d_model % 128
    assert pz.load_library().puzzle_moe_quant_workspace_size(ctypes.byref(d), 64, 2) == 0


def test_quant_forward_scale_range_paths(pz):
    """The decoder's two forms (gemv_tc.cu decode_pass_q): the byte-table decode with the exact
    +-2^-63 sign / mask product for group scales in [2^-126, 2^61], the integer form for any
    other finite scale. Groups of every projection are re-scaled by 2^-127 (codes kept: the
    dequantised values are bf16 subnormals) or 2^70 with their codes zeroed (flags kept), on
    rows spread over every tile quarter, so that both forms alternate inside one stage range;
    the reference dequantises the modified layer with the oracle."""
    cfg = CFGS[0]
    (c13, s13, c2, s2, slot), _ = quant_layer(cfg)
    c13, s13, c2, s2 = c13.copy(), s13.copy(), c2.copy(), s2.copy()
    rng = np.random.default_rng(31)
    for codes, scales in ((c13.reshape(-1, c13.shape[-1]), s13.reshape(-1, s13.shape[-1])),
                          (c2.reshape(-1, c2.shape[-1]), s2.reshape(-1, s2.shape[-1]))):
        rows = rng.choice(scales.shape[0], scales.shape[0] // 5, replace=False)
        for r in rows:
            g = int(rng.integers(scales.shape[1]))
            if r % 2:
                scales[r, g] = np.float32(scales[r, g] * np.float32(2.0 ** -127))
            else:
                scales[r, g] = np.float32(2.0 ** 70)
                codes[r, 128 * g:128 * (g + 1)] &= 0xF0  # flags kept, code 0
    P, d, f = cfg.n_pairs, cfg.d_model, cfg.d_ff
    w13r = np.empty((2 * P, 2, f, d), np.uint16)
    w2r = np.empty((2 * P, d, f), np.uint16)
    for p in range(P):
        for pos in (0, 1):
            for j in (0, 1):
                w13r[2 * p + pos, j] = oracle.quant_unpack(c13[p, j], s13[p, j], pos)
            w2r[2 * p + pos] = oracle.quant_unpack(c2[p], s2[p], pos)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    layer = pz.QuantMoELayer(t(c13), t(s13), t(c2), t(s2), t(slot))
    T = 64
    hb = synth.hidden_bits(cfg, T)
    lg = synth.router_logits(cfg, T)
    out = layer.forward(t(hb.view(np.int16)).view(torch.bfloat16), t(lg), cfg.top_k, cfg.renormalize)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13r, w2r, (2 * slot).astype(np.int32), hb, lg, cfg.top_k, cfg.renormalize,
                             pair_dense=np.ones(2 * P, np.uint8))
    assert_close(out.float().cpu().numpy(), ref, "quant scale-range paths")
