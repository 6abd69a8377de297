"""Pins for the oracle router and MoE FFN (O5; reading R13).

Pinned by library routines and special cases: torch.topk/torch.softmax for routing,
a dense torch f64 SwiGLU FFN for self-merged pairs (Eq. 8 reduces to the identity),
Eq. 8 reconstruction + torch f64 for general merged pairs (Table 1 echo),
top-1 renormalised gate == 1, and token-permutation equivariance."""
import numpy as np
import pytest
import torch

import oracle
import synth


def _dense_ffn_f64(x, w1, w3, w2):
    """torch f64 SwiGLU expert: W2 (silu(W1 x) * (W3 x)); x [T, d], W1/W3 [f, d], W2 [d, f]."""
    x = torch.as_tensor(x, dtype=torch.float64)
    g = x @ torch.as_tensor(w1, dtype=torch.float64).T
    u = x @ torch.as_tensor(w3, dtype=torch.float64).T
    return (torch.nn.functional.silu(g) * u) @ torch.as_tensor(w2, dtype=torch.float64).T


def test_route_matches_torch_topk_and_softmax():
    rng = np.random.default_rng(0)
    logits = rng.standard_normal((300, 64)).astype(np.float32)
    for k, renorm in ((1, True), (2, True), (4, False), (6, False)):
        idx, gate = oracle.route(logits, k, renorm)
        lt = torch.from_numpy(logits).double()
        tv, ti = torch.topk(lt, k, dim=-1)  # no ties among continuous draws
        assert np.array_equal(idx, ti.numpy())
        if renorm:
            want = torch.softmax(tv, dim=-1)
        else:
            want = torch.gather(torch.softmax(lt, dim=-1), 1, ti)
        np.testing.assert_allclose(gate, want.numpy(), rtol=1e-13, atol=1e-15)


def test_route_ties_go_to_lower_index_and_top1_gate_is_one():
    logits = np.array([[0.5, 0.5, 0.5, 0.1], [2.0, 3.0, 3.0, 3.0]], np.float32)
    idx, gate = oracle.route(logits, 2, True)
    assert idx.tolist() == [[0, 1], [1, 2]]
    idx, gate = oracle.route(logits, 1, True)
    assert gate.tolist() == [[1.0], [1.0]]


def _merged_pair(cfg, rng, self_merge=False):
    """Pack one pair per the oracle; returns packed w13 [1,2,f,d], w2 [1,d,f] and the
    dense bf16 source experts."""
    d, f = cfg.d_model, cfg.d_ff
    src = {}
    packed = {}
    for slot, shape in (("w1", (f, d)), ("w3", (f, d)), ("w2", (d, f))):
        w_i = synth.to_bf16_values(rng.standard_normal(shape).astype(np.float32) / np.sqrt(shape[1]))
        w_j = w_i.copy() if self_merge else synth.to_bf16_values(
            rng.standard_normal(shape).astype(np.float32) / np.sqrt(shape[1]))
        n_i = 1 + np.abs(rng.standard_normal(shape[1])).astype(np.float32)
        n_j = 1 + np.abs(rng.standard_normal(shape[1])).astype(np.float32)
        art = oracle.merge(w_i, w_j, n_i, n_j, 0.4)
        packed[slot], _ = oracle.pack_artifacts(art)
        src[slot] = (w_i, w_j)
    w13 = np.stack([packed["w1"], packed["w3"]])[None]
    w2 = packed["w2"][None]
    return w13, w2, src


def test_self_merged_pair_equals_dense_expert():
    cfg = synth.CONFIGS["tiny"]
    rng = np.random.default_rng(1)
    w13, w2, src = _merged_pair(cfg, rng, self_merge=True)
    T = 8
    hb = synth.hidden_bits(cfg, T)
    x = oracle.bf16_bits_to_f32(hb)
    logits = np.array([[0.3, -0.2]] * 4 + [[-1.0, 2.0]] * 4, np.float32)
    out = oracle.moe_forward(w13, w2, np.array([0, 1], np.int32), hb, logits, 1, True)
    # both experts of a self-merged pair equal the source expert (minus exponent clamp;
    # the 1/sqrt(in) draws all sit inside [112, 143] except a few flushed-up tiny ones)
    w1, w3, w2d = (oracle.bf16_bits_to_f32(oracle.unpack(w, 0)) for w in (w13[0, 0], w13[0, 1], w2[0]))
    for name, dec in (("w1", w1), ("w3", w3), ("w2", w2d)):
        src_w = src[name][0]
        ok = np.abs(src_w) >= 2.0 ** -15
        assert np.array_equal(dec[ok], src_w[ok]), name
    want = _dense_ffn_f64(x, w1, w3, w2d).numpy()
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-12)
    # and the unclamped source expert differs only by the tiny clamped entries
    want_src = _dense_ffn_f64(x, src["w1"][0], src["w3"][0], src["w2"][0]).numpy()
    np.testing.assert_allclose(out, want_src, rtol=0, atol=1e-3)


def test_general_pair_equals_eq8_reconstruction_and_residual():
    """Table 1 echo: FFN over packed words == FFN over the Eq. 8 reconstruction of the
    bf16-rounded merge artifacts, evaluated by torch f64 matmuls (library routine)."""
    cfg = synth.CONFIGS["tiny"]
    rng = np.random.default_rng(2)
    w13, w2, _ = _merged_pair(cfg, rng)
    T = 16
    hb = synth.hidden_bits(cfg, T, seed=11)
    rb = synth.hidden_bits(cfg, T, seed=12)
    x = oracle.bf16_bits_to_f32(hb)
    logits = synth.router_logits(cfg, T, seed=13)
    out = oracle.moe_forward(w13, w2, np.array([1, 0], np.int32), hb, logits, 1, True, rb)
    idx, _ = oracle.route(logits, 1, True)
    want = oracle.bf16_bits_to_f32(rb).astype(np.float64)
    for t in range(T):
        e = int(idx[t, 0])
        pos = [1, 0][e]  # expert_slot = [1, 0]: expert 0 is pos 1
        w1, w3, w2d = (oracle.bf16_bits_to_f32(oracle.unpack(w, pos)) for w in (w13[0, 0], w13[0, 1], w2[0]))
        want[t] += _dense_ffn_f64(x[t:t + 1], w1, w3, w2d).numpy()[0]
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-12)


def test_topk_combination_and_permutation_equivariance():
    cfg = synth.MoEConfig("t4", 0, 32, 64, 4, 2, False)
    rng = np.random.default_rng(3)
    w13_list, w2_list = [], []
    for _ in range(cfg.n_pairs):
        a, b, _ = _merged_pair(cfg, rng)
        w13_list.append(a[0])
        w2_list.append(b[0])
    w13 = np.stack(w13_list)
    w2 = np.stack(w2_list)
    slot = np.array([2, 0, 3, 1], np.int32)
    T = 12
    hb = synth.hidden_bits(cfg, T, seed=5)
    logits = synth.router_logits(cfg, T, seed=6)
    out = oracle.moe_forward(w13, w2, slot, hb, logits, 2, False)
    # explicit combination from per-expert top-1-style single evaluations
    idx, gate = oracle.route(logits, 2, False)
    x = oracle.bf16_bits_to_f32(hb)
    want = np.zeros((T, cfg.d_model))
    for t in range(T):
        for j in range(2):
            p, pos = divmod(int(slot[idx[t, j]]), 2)
            w1, w3, w2d = (oracle.bf16_bits_to_f32(oracle.unpack(w, pos))
                           for w in (w13[p, 0], w13[p, 1], w2[p]))
            want[t] += gate[t, j] * _dense_ffn_f64(x[t:t + 1], w1, w3, w2d).numpy()[0]
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-13)
    perm = rng.permutation(T)
    out_p = oracle.moe_forward(w13, w2, slot, hb[perm], logits[perm], 2, False)
    assert np.array_equal(out_p, out[perm])


def test_expert_ffn_matches_forward_and_dense():
    """oracle.expert_ffn on rows routed to one expert == the dense f64 FFN of the Eq. 8
    reconstruction, and == moe_forward for a top-1 renormalised route (gate 1)."""
    cfg = synth.CONFIGS["tiny"]
    rng = np.random.default_rng(9)
    w13, w2, _ = _merged_pair(cfg, rng)
    hb = synth.hidden_bits(cfg, 5, seed=21)
    x = oracle.bf16_bits_to_f32(hb)
    for pos in (0, 1):
        y = oracle.expert_ffn(w13, w2, 0, pos, hb)
        w1, w3, w2d = (oracle.bf16_bits_to_f32(oracle.unpack(w, pos)) for w in (w13[0, 0], w13[0, 1], w2[0]))
        np.testing.assert_allclose(y, _dense_ffn_f64(x, w1, w3, w2d).numpy(), rtol=1e-12, atol=1e-13)
        logits = np.zeros((5, 2), np.float32)
        logits[:, pos] = 1.0  # expert `pos` is at position pos with expert_slot = [0, 1]
        out = oracle.moe_forward(w13, w2, np.array([0, 1], np.int32), hb, logits, 1, True)
        np.testing.assert_allclose(out, y, rtol=1e-12, atol=1e-13)


def _mixed_layer(cfg, rng, n_merged, n_dense):
    """25% ratio layout (reading R20): n_merged packed pairs, then n_dense slots that each
    hold one unmerged expert's plain bf16 weights at position 0. Returns w13, w2,
    expert_slot, pair_dense and the dense experts' float weights."""
    d, f = cfg.d_model, cfg.d_ff
    w13, w2, dense_src = [], [], []
    for _ in range(n_merged):
        a, b, _ = _merged_pair(cfg, rng)
        w13.append(a[0])
        w2.append(b[0])
    for _ in range(n_dense):
        w1 = synth.to_bf16_values(rng.standard_normal((f, d)).astype(np.float32) / np.sqrt(d))
        w3 = synth.to_bf16_values(rng.standard_normal((f, d)).astype(np.float32) / np.sqrt(d))
        wd = synth.to_bf16_values(rng.standard_normal((d, f)).astype(np.float32) / np.sqrt(f))
        w13.append(np.stack([synth.to_bf16_bits(w1), synth.to_bf16_bits(w3)]))
        w2.append(synth.to_bf16_bits(wd))
        dense_src.append((w1, w3, wd))
    P = n_merged + n_dense
    slot = np.array([2 * p + q for p in range(n_merged) for q in (0, 1)] +
                    [2 * (n_merged + i) for i in range(n_dense)], np.int32)
    pair_dense = np.array([0] * n_merged + [1] * n_dense, np.uint8)
    return np.stack(w13), np.stack(w2), slot, pair_dense, dense_src


def test_dense_slots_equal_plain_bf16_ffn():
    """R20: a dense slot computes the FFN of its bf16 weights as stored (no Algorithm-1
    decode, no exponent clamp), pinned by torch f64 matmuls on the float weights; the
    merged pair next to it is unchanged (Eq. 8 reconstruction)."""
    cfg = synth.MoEConfig("t25", 0, 32, 64, 4, 2, True)
    rng = np.random.default_rng(31)
    w13, w2, slot, dense, dsrc = _mixed_layer(cfg, rng, 1, 2)
    # tiny magnitudes below 2^-15 would be clamped by a packed slot but not by a dense one
    w13[1, 0, 0, :4] = synth.to_bf16_bits(np.array([1e-6, -3e-7, 2e-8, 0.0], np.float32))
    dsrc[0] = (oracle.bf16_bits_to_f32(w13[1, 0]), dsrc[0][1], dsrc[0][2])
    T = 12
    hb = synth.hidden_bits(cfg, T, seed=32)
    x = oracle.bf16_bits_to_f32(hb)
    logits = synth.router_logits(cfg, T, seed=33)
    out = oracle.moe_forward(w13, w2, slot, hb, logits, 2, True, pair_dense=dense)
    idx, gate = oracle.route(logits, 2, True)
    want = np.zeros((T, cfg.d_model))
    for t in range(T):
        for j in range(2):
            e = int(idx[t, j])
            if e >= 2:
                w1, w3, wd = dsrc[e - 2]
            else:
                w1, w3, wd = (oracle.bf16_bits_to_f32(oracle.unpack(w, e)) for w in (w13[0, 0], w13[0, 1], w2[0]))
            want[t] += gate[t, j] * _dense_ffn_f64(x[t:t + 1], w1, w3, wd).numpy()[0]
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-13)
    assert set(idx.reshape(-1).tolist()) >= {0, 1, 2, 3}  # every slot kind exercised
    for e in (2, 3):
        y = oracle.expert_ffn(w13, w2, int(slot[e]) // 2, 0, hb, dense=True)
        np.testing.assert_allclose(y, _dense_ffn_f64(x, *dsrc[e - 2]).numpy(), rtol=1e-12, atol=1e-13)


def test_dense_slot_layout_errors():
    cfg = synth.MoEConfig("t25", 0, 32, 64, 4, 2, True)
    rng = np.random.default_rng(34)
    w13, w2, slot, dense, _ = _mixed_layer(cfg, rng, 1, 2)
    hb = synth.hidden_bits(cfg, 3, seed=35)
    logits = synth.router_logits(cfg, 3, seed=36)
    bad = slot.copy()
    bad[3] = 5  # position 1 of a dense slot
    with pytest.raises(ValueError):
        oracle.moe_forward(w13, w2, bad, hb, logits, 2, True, pair_dense=dense)
    bad = slot.copy()
    bad[3] = bad[2]  # two experts in one slot
    with pytest.raises(ValueError):
        oracle.moe_forward(w13, w2, bad, hb, logits, 2, True, pair_dense=dense)
    with pytest.raises(ValueError):
        oracle.expert_ffn(w13, w2, 1, 1, hb, dense=True)
