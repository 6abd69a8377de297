"""Pins for the oracle's calibration statistics (NEXT-4; Eq. 4 ||X||_2 per input column over
the activations routed to an expert, from a single forward pass).

Pinned by a hand-computed worked case, the duplicate-token scaling law, numpy column norms of
the routed rows (selection by the pinned router), and the SwiGLU intermediate evaluated with
torch f64 matmuls on the dense / Eq. 8-reconstructed weights."""
import numpy as np
import torch

import oracle
import synth
from test_oracle_ffn import _mixed_layer


def test_hand_worked_case():
    # d = 2, two experts in one merged pair (slots 0, 1), top-1: token 0 -> expert 1, token 1 -> expert 0,
    # token 2 -> expert 1. x values exact in bf16.
    x = np.array([[1.0, -2.0], [0.5, 3.0], [-4.0, 0.25]], np.float32)
    hb = synth.to_bf16_bits(x)
    logits = np.array([[0.0, 1.0], [1.0, 0.0], [-1.0, 2.0]], np.float32)
    w13 = np.zeros((1, 2, 64, 2), np.uint16)
    sx, _ = oracle.calib_sumsq(w13, np.array([0, 1], np.int32), hb, logits, 1, True, want_h=False)
    assert sx.tolist() == [[0.25, 9.0], [1.0 + 16.0, 4.0 + 0.0625]]
    # top-2: both slots see every token
    sx, _ = oracle.calib_sumsq(w13, np.array([0, 1], np.int32), hb, logits, 2, True, want_h=False)
    assert sx.tolist() == [[17.25, 13.0625], [17.25, 13.0625]]


def test_duplicated_tokens_scale_sums():
    cfg = synth.MoEConfig("c4", 0, 32, 64, 4, 2, False)
    rng = np.random.default_rng(41)
    w13, w2, slot, dense, _ = _mixed_layer(cfg, rng, 1, 2)
    hb = synth.hidden_bits(cfg, 5, seed=42)
    lg = synth.router_logits(cfg, 5, seed=43)
    sx1, sh1 = oracle.calib_sumsq(w13, slot, hb, lg, 2, False, pair_dense=dense)
    sx3, sh3 = oracle.calib_sumsq(w13, slot, np.tile(hb, (3, 1)), np.tile(lg, (3, 1)), 2, False, pair_dense=dense)
    np.testing.assert_allclose(sx3, 3 * sx1, rtol=1e-14)
    np.testing.assert_allclose(sh3, 3 * sh1, rtol=1e-12)


def test_matches_routed_rows_and_torch_swiglu():
    cfg = synth.MoEConfig("c6", 0, 32, 64, 6, 2, True)
    rng = np.random.default_rng(44)
    w13, w2, slot, dense, dsrc = _mixed_layer(cfg, rng, 1, 4)  # slots: 1 merged pair + 4 dense
    T = 20
    hb = synth.hidden_bits(cfg, T, seed=45)
    lg = synth.router_logits(cfg, T, seed=46)
    sx, sh = oracle.calib_sumsq(w13, slot, hb, lg, cfg.top_k, cfg.renormalize, pair_dense=dense)
    idx, _ = oracle.route(lg, cfg.top_k, cfg.renormalize)
    x = oracle.bf16_bits_to_f32(hb).astype(np.float64)
    P = w13.shape[0]
    for b in range(2 * P):
        experts = np.nonzero(slot == b)[0]
        rows = [t for t in range(T) for j in range(cfg.top_k) if idx[t, j] in experts]
        want_x = np.linalg.norm(x[rows], axis=0) ** 2 if rows else np.zeros(cfg.d_model)
        np.testing.assert_allclose(sx[b], want_x, rtol=1e-13, atol=0)
        if not rows:
            assert not sh[b].any()
            continue
        q, pos = divmod(b, 2)
        if dense[q]:
            w1, w3 = (oracle.bf16_bits_to_f32(w13[q, i]) for i in (0, 1))
        else:
            w1, w3 = (oracle.bf16_bits_to_f32(oracle.unpack(w13[q, i], pos)) for i in (0, 1))
        xt = torch.from_numpy(x[rows])
        h = torch.nn.functional.silu(xt @ torch.from_numpy(w1).double().T) * (xt @ torch.from_numpy(w3).double().T)
        np.testing.assert_allclose(sh[b], (h ** 2).sum(0).numpy(), rtol=1e-11, atol=1e-300)


def test_group_colsumsq_worked_case():
    rows = synth.to_bf16_bits(np.array([[1.0, 2.0], [3.0, -1.0], [0.5, 0.0], [-2.0, 4.0]], np.float32))
    out = oracle.group_colsumsq(rows, [0, 2, 2, 4])  # groups: rows 0-1, empty, rows 2-3
    assert out.tolist() == [[10.0, 5.0], [0.0, 0.0], [4.25, 16.0]]
