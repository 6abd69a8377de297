"""Pins for the oracle's quantised PuzzleMoE format (NEXT-3; Appendix A.3; SPEC
quantization module S:467-505; readings R21-R23): the SPEC worked example, the all-zero and
single-maximum groups, the round-trip error bound |dequant - w| <= scale / 2, masked entries
exactly zero, signs, and the byte layout."""
import numpy as np
import torch

import oracle


def _planes(shape, rng, p=0.5):
    return [(rng.random(shape) < p).astype(np.uint8) for _ in range(4)]


def _bf16_to_f32(bits):
    return oracle.bf16_bits_to_f32(bits).astype(np.float64)


def test_spec_worked_example():
    """values [1, 2, 0.5, 4], 3 bits -> scale 4/7, codes [2, 4, 1, 7], dequant
    [1.1429, 2.2857, 0.5714, 4.0] (here the rest of the 128-group is 0, so max stays 4)."""
    w = np.zeros((1, 128), np.float32)
    w[0, :4] = [1.0, 2.0, 0.5, 4.0]
    ones = np.ones((1, 128), np.uint8)
    zeros = np.zeros((1, 128), np.uint8)
    codes, scales = oracle.quant_pack(w, ones, ones, zeros, zeros)
    assert scales[0, 0] == np.float32(4.0) / np.float32(7.0)
    assert (codes[0, :4] & 7).tolist() == [2, 4, 1, 7]
    assert not (codes[0, 4:] & 7).any()
    deq = _bf16_to_f32(oracle.quant_unpack(codes, scales, 0))[0, :4]
    np.testing.assert_allclose(deq, [1.1429, 2.2857, 0.5714, 4.0], rtol=4e-3)  # bf16 operand
    # the byte carries M_i M_j in bits 5/4 (both set here), no signs
    assert ((codes[0, :4] >> 4) == 0b0011).all()


def test_zero_group_and_single_maximum():
    rng = np.random.default_rng(1)
    w = np.zeros((2, 256), np.float32)
    w[1, 128 + 17] = 3.25  # group 3: one nonzero value
    pl = _planes(w.shape, rng)
    codes, scales = oracle.quant_pack(w, *pl)
    assert scales[0].tolist() == [1.0, 1.0] and scales[1, 0] == 1.0  # all-zero groups: scale 1
    assert scales[1, 1] == np.float32(3.25) / np.float32(7.0)
    assert (codes[1, 128 + 17] & 7) == 7 and not (codes & 7).sum() - 7
    # the maximum of a group always round-trips to code 7 * scale = max (within f32 / bf16 rounding)
    deq = _bf16_to_f32(oracle.quant_unpack(codes, scales, 0))
    if pl[0][1, 128 + 17]:
        assert abs(abs(deq[1, 128 + 17]) - 3.25) <= 3.25 * 2 ** -8


def test_round_trip_bound_masks_and_signs():
    rng = np.random.default_rng(2)
    rows, cols = 16, 512
    w = np.abs(rng.standard_normal((rows, cols))).astype(np.float32) * rng.choice([1e-3, 1.0, 50.0], (rows, 1)).astype(np.float32)
    m0, m1, s0, s1 = _planes((rows, cols), rng)
    codes, scales = oracle.quant_pack(w, m0, m1, s0, s1)
    sc = np.repeat(scales, 128, axis=1).astype(np.float64)
    # codes: |code * scale - w| <= scale / 2 (+ one f32 ulp of the division)
    q = (codes & 7).astype(np.float64)
    assert np.all(np.abs(q * sc - w) <= sc * (0.5 + 1e-6))
    for pos, (m, s) in enumerate(((m0, s0), (m1, s1))):
        deq = oracle.quant_unpack(codes, scales, pos)
        v = _bf16_to_f32(deq)
        assert np.all(deq[m == 0] == 0)                          # masked entries exactly +0
        nz = (m == 1) & (q > 0)
        assert np.all(np.signbit(v[nz]) == (s[nz] == 1))          # the position's sign bit
        want = torch.tensor(q * sc, dtype=torch.float32).to(torch.bfloat16).double().numpy()  # library RNE
        np.testing.assert_array_equal(np.abs(v[m == 1]), want[m == 1])
    # byte layout: the flag nibble is exactly S_i S_j M_i M_j, bit 3 clear
    assert np.array_equal(codes >> 4, (s0 << 3) | (s1 << 2) | (m0 << 1) | m1)
    assert not (codes & 8).any()


def test_quantised_merge_pipeline_error():
    """Eq. 1-7 merge -> quantise -> dequantise: every kept entry of expert i is within
    scale/2 (+ bf16 rounding) of the bf16-rounded merged magnitude (Eq. 8 with W_merged
    replaced by its 3-bit level)."""
    rng = np.random.default_rng(3)
    w_i = (rng.standard_normal((8, 256)) / 16).astype(np.float32)
    w_j = (rng.standard_normal((8, 256)) / 16).astype(np.float32)
    art = oracle.merge(w_i, w_j, np.ones(256, np.float32), np.ones(256, np.float32), 0.4)
    codes, scales = oracle.quant_pack(art["w_merged"], art["m_i"], art["m_j"], art["s_i"], art["s_j"])
    deq = _bf16_to_f32(oracle.quant_unpack(codes, scales, 0))
    sc = np.repeat(scales, 128, axis=1).astype(np.float64)
    kept = art["m_i"] == 1
    ref = np.where(art["s_i"] == 1, -1.0, 1.0) * art["w_merged"]
    assert np.all(np.abs(deq[kept] - ref[kept]) <= sc[kept] * 0.5 + np.abs(ref[kept]) * 2 ** -8 + 1e-12)
    assert np.all(deq[~kept] == 0)


def test_quant_gemv_lossless_case_equals_plain_matmul():
    """quant_gemv pinned to the plain definition y = x ((-1)^S M w)^T, built from the original
    magnitudes and bit-planes (not from the codes): with every group's values on the grid
    k * 2^e (k in 0..7, the group maximum 7 * 2^e) the format is lossless (scale = 2^e exactly,
    codes = k, bf16(k * 2^e) exact), so the GEMV must equal the signed, masked dense matmul.
    Non-square shapes and unequal token counts catch a transposed operand or swapped
    positions; the sign / mask planes of i and j differ, so taking j's bits for i fails."""
    rng = np.random.default_rng(11)
    rows, cols, n_i, n_j = 5, 256, 3, 4
    k = rng.integers(0, 8, (rows, cols)).astype(np.float32)
    k[:, ::128] = 7.0
    e = rng.integers(-6, 4, (rows, cols // 128)).astype(np.float32)
    w = k * np.repeat(np.exp2(e), 128, axis=1)
    m0, m1, s0, s1 = _planes((rows, cols), rng)
    codes, scales = oracle.quant_pack(w, m0, m1, s0, s1)
    xs = [torch.randn(n, cols).to(torch.bfloat16) for n in (n_i, n_j)]
    xbits = [t.view(torch.int16).numpy().view(np.uint16) for t in xs]
    y_i, y_j = oracle.quant_gemv(codes, scales, *xbits)
    wd = w.astype(np.float64)
    want_i = xs[0].double().numpy() @ (np.where(s0 != 0, -1.0, 1.0) * (m0 != 0) * wd).T
    want_j = xs[1].double().numpy() @ (np.where(s1 != 0, -1.0, 1.0) * (m1 != 0) * wd).T
    assert y_i.shape == (n_i, rows) and y_j.shape == (n_j, rows)
    np.testing.assert_allclose(y_i, want_i, rtol=0, atol=1e-12)
    np.testing.assert_allclose(y_j, want_j, rtol=0, atol=1e-12)
    assert not np.allclose(y_i, xs[0].double().numpy() @ (np.where(s1 != 0, -1.0, 1.0) * (m1 != 0) * wd).T)
