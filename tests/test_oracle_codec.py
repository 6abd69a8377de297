"""Pins for the oracle's bit codec (O1 RNE, O3 pack, O4 Algorithm 1).

Each pin is fixed by something other than the oracle itself: SPEC/paper golden words,
a second byte-literal transcription of Algorithm 1 written independently
below, exhaustive bijection over all 2^16 words, and torch's CPU f32->bf16 cast
(a library RNE routine)."""
import os

import numpy as np
import pytest
import torch

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "codec_vectors.tsv")


def _golden_rows():
    rows = []
    with open(GOLDEN) as fh:
        for line in fh:
            if not line.strip() or line.startswith("#"):
                continue
            op, args, expected, cite = line.rstrip("\n").split("\t")
            rows.append((op, [int(a, 0) for a in args.split()], [int(e, 0) for e in expected.split()], cite))
    return rows


def _alg1_literal(word: int, expert_pos: int) -> int:
    """Algorithm 1, transcribed statement by statement from P:200-209 with Python ints
    (independent of oracle/puzzle_oracle.c)."""
    mask_bit = (word >> (13 - expert_pos)) & 1
    if mask_bit == 0:
        return 0x0000
    sign_bit = (word >> (15 - expert_pos)) & 1
    exp = (word & 0x0F80) + (112 << 7)
    return ((sign_bit << 15) | exp | (word & 0x007F)) & 0xFFFF


@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: f"{r[0]}-{r[3].split()[0]}")
def test_golden_vectors(row):
    op, args, expected, cite = row
    if op == "shift":
        # shift_exponent is pack's payload: pack with all-zero header bits.
        mag = oracle.bf16_bits_to_f32(np.array([args[0]], np.uint16))
        z = np.zeros(1, np.uint8)
        word, _ = oracle.pack(mag, z, z, z, z)
        payload = int(word[0]) & 0x0FFF
        e_prime = payload >> 7
        shifted = ((e_prime + 112) << 7) | (payload & 0x7F)
        assert (shifted, e_prime) == (expected[0], expected[1]), cite
    elif op == "pack":
        mag = oracle.bf16_bits_to_f32(np.array([args[0]], np.uint16))
        s0, s1, m0, m1 = (np.array([v], np.uint8) for v in args[1:])
        word, _ = oracle.pack(mag, m0, m1, s0, s1)
        assert int(word[0]) == expected[0], cite
    elif op == "decode":
        got = oracle.unpack(np.array([args[0]], np.uint16), args[1])
        assert int(got[0]) == expected[0], cite
        assert _alg1_literal(args[0], args[1]) == expected[0], cite
    else:
        raise AssertionError(op)


ALL_WORDS = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)


@pytest.mark.parametrize("pos", [0, 1])
def test_unpack_exhaustive_vs_literal_alg1(pos):
    got = oracle.unpack(ALL_WORDS, pos)
    want = np.array([_alg1_literal(int(w), pos) for w in ALL_WORDS], np.uint16)
    assert np.array_equal(got, want)


def test_swar_two_lane_decode_matches_alg1():
    """The two-words-per-u32 SWAR form used by the GPU register path,
    checked here against Alg. 1 for all 2^16 words in both lanes and both positions."""
    lo = ALL_WORDS.astype(np.uint32)
    hi = np.roll(lo, 12345)
    W = lo | (hi << 16)
    for pos in (0, 1):
        m = ((W >> np.uint32(13 - pos)) & np.uint32(0x00010001)) * np.uint32(0xFFFF)
        dec = (((W & np.uint32(0x0FFF0FFF)) + np.uint32(0x38003800)) |
               ((W << np.uint32(pos)) & np.uint32(0x80008000))) & m
        want_lo = oracle.unpack(lo.astype(np.uint16), pos)
        want_hi = oracle.unpack(hi.astype(np.uint16), pos)
        assert np.array_equal((dec & 0xFFFF).astype(np.uint16), want_lo)
        assert np.array_equal((dec >> 16).astype(np.uint16), want_hi)


def test_pack_is_bijection_onto_all_words():
    """Every word is (4 header bits, 5-bit e', 7-bit mantissa); packing the magnitude
    (e'+112, mantissa) with those header bits must reproduce the word exactly."""
    w = ALL_WORDS.astype(np.uint32)
    s0 = ((w >> 15) & 1).astype(np.uint8)
    s1 = ((w >> 14) & 1).astype(np.uint8)
    m0 = ((w >> 13) & 1).astype(np.uint8)
    m1 = ((w >> 12) & 1).astype(np.uint8)
    mag_bits = ((((w >> 7) & 0x1F) + 112) << 7 | (w & 0x7F)).astype(np.uint16)
    mag = oracle.bf16_bits_to_f32(mag_bits)
    packed, stats = oracle.pack(mag, m0, m1, s0, s1)
    assert np.array_equal(packed, ALL_WORDS)
    assert stats.tolist() == [0, 0, 0, 0]


def test_round_trip_reproduces_signed_masked_value():
    """decode(pack(|w|, S, M), pos) == (-1)^S * M * |w| for in-range magnitudes (Eq. 8)."""
    rng = np.random.default_rng(0)
    n = 200_000
    e = rng.integers(112, 144, n)
    mant = rng.integers(0, 128, n)
    mag = oracle.bf16_bits_to_f32(((e << 7) | mant).astype(np.uint16))
    s0, s1, m0, m1 = (rng.integers(0, 2, n).astype(np.uint8) for _ in range(4))
    packed, _ = oracle.pack(mag, m0, m1, s0, s1)
    for pos, s, m in ((0, s0, m0), (1, s1, m1)):
        got = oracle.bf16_bits_to_f32(oracle.unpack(packed, pos)).astype(np.float64)
        want = np.where(m == 1, np.where(s == 1, -1.0, 1.0) * mag.astype(np.float64), 0.0)
        assert np.array_equal(got, want)
        # masked-out entries decode to +0.0 exactly (bits 0x0000)
        assert np.all(oracle.unpack(packed, pos)[m == 0] == 0)


def test_header_payload_independence():
    rng = np.random.default_rng(1)
    words = rng.integers(0, 1 << 16, 50_000).astype(np.uint16)
    for pos in (0, 1):
        base = oracle.unpack(words, pos)
        for bit in (15, 14, 13, 12):
            flipped = oracle.unpack(words ^ np.uint16(1 << bit), pos)
            both = (base != 0) & (flipped != 0)
            assert np.array_equal(base[both] & 0x7FFF, flipped[both] & 0x7FFF)


def test_exponent_clamp_and_counters():
    vals = np.array([2.0 ** -20, 0.0, 1e-30, 2.0 ** 17, 3.0e38, 1.0], np.float32)
    z = np.zeros(vals.size, np.uint8)
    packed, stats = oracle.pack(vals, z, z, z, z)
    e_prime = (packed.astype(np.int64) >> 7) & 0x1F
    assert e_prime.tolist() == [0, 0, 0, 31, 31, 15]
    # rounded up: 2^-20, 0.0, 1e-30; saturated: 2^17 (exp 144), 3e38 (exp 254)
    assert stats.tolist() == [3, 2, 0, 0]
    # saturation monotonicity: clamping never moves a magnitude the wrong way
    dec = oracle.bf16_bits_to_f32(oracle.unpack(packed | np.uint16(0x3000), 0))
    assert np.all(dec[:3] >= vals[:3]) and np.all(dec[3:5] <= vals[3:5])
    _, stats = oracle.pack(np.array([np.inf, -1.0], np.float32), z[:2], z[:2], z[:2], z[:2])
    assert stats[2] == 1 and stats[3] == 1


def test_rne_matches_torch_cast_on_sweep():
    """O1 bf16_rne against torch's CPU f32->bf16 cast (library RNE) over a strided sweep
    of all non-negative finite f32 bit patterns plus every exact halfway case."""
    u = np.arange(0, 0x7F800000, 97, dtype=np.uint64).astype(np.uint32)
    hi = np.arange(0, 0x7F80, dtype=np.uint32) << 16
    halfway = np.concatenate([hi | 0x8000, hi | 0x7FFF, hi | 0x8001, hi | 0xFFFF])
    u = np.concatenate([u, halfway[halfway < 0x7F800000]])
    x = u.view(np.float32)
    got = oracle.bf16_round(x)
    want = torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, want)


def test_rne_nan_and_inf_match_torch_cast():
    """O1 bf16_rne on the non-finite patterns: +-Inf stay Inf, every NaN stays a (quiet) NaN
    with its sign and top payload bits, as torch's CPU cast does (a NaN rounded
    by the plain RNE formula became -0)."""
    rng = np.random.default_rng(7)
    payload = rng.integers(1, 1 << 23, 4000, dtype=np.uint64).astype(np.uint32)
    nans = np.concatenate([0x7F800000 | payload, 0xFF800000 | payload,
                           np.array([0x7FC00000, 0x7FFFFFFF, 0xFFFFFFFF, 0x7F800001, 0x7F810000], np.uint32)])
    infs = np.array([0x7F800000, 0xFF800000], np.uint32)
    u = np.concatenate([nans.astype(np.uint32), infs])
    x = u.view(np.float32)
    got = oracle.bf16_round(x)
    want = torch.from_numpy(x.copy()).to(torch.bfloat16)
    # torch returns one canonical NaN: compare NaN-ness, then the kept sign / quiet bit
    assert np.array_equal(np.isnan(want.float().numpy()), (got & 0x7FFF) > 0x7F80)
    assert np.array_equal(got[-2:], want[-2:].view(torch.int16).numpy().view(np.uint16))
    assert np.array_equal(got[:-2] >> 15, u[:-2] >> 31) and np.all(got[:-2] & 0x0040)
