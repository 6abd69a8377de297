"""Pins for the oracle's merge (Eq. 1-7) and reconstruction (Eq. 8).

Pinned by: SPEC's 2x2 worked example (golden file), identity merges, the Appendix B
closed form against the oracle's similarity-mask frequency on i.i.d.
Gaussians, the similar-entry error bound and salient-entry exactness,
tie and scale properties, and 50% byte accounting."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.analysis import similarity_fraction_closed

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "merge_2x2.json")


def _reconstruct(packed, pos):
    return oracle.bf16_bits_to_f32(oracle.unpack(packed, pos))


def test_worked_2x2_example():
    g = json.load(open(GOLDEN))
    art = oracle.merge(g["w_i"], g["w_j"], g["norms_i"], g["norms_j"], g["tau_sim"])
    for key in ("m_sim", "m_sal_i", "m_i", "m_j"):
        assert art[key].tolist() == g[key], key
    np.testing.assert_allclose(art["w_merged"], g["w_merged"], rtol=0, atol=1e-7)
    packed, stats = oracle.pack_artifacts(art)
    assert packed.tolist() == g["packed"]
    assert stats.tolist() == [0, 0, 0, 0]
    assert oracle.unpack(packed, 0).tolist() == g["decode_pos0_bits"]
    assert oracle.unpack(packed, 1).tolist() == g["decode_pos1_bits"]
    # reconstructions equal SPEC's up to the bf16 rounding of 0.55
    np.testing.assert_allclose(_reconstruct(packed, 0), g["reconstruct_pos0"], atol=2e-3)
    np.testing.assert_allclose(_reconstruct(packed, 1), g["reconstruct_pos1"], atol=2e-3)
    # GEMV of S:310 on the decoded pos-0 weights (f64 dot products by numpy)
    y = _reconstruct(packed, 0).astype(np.float64) @ np.array(g["gemv_x"])
    assert y.tolist() == g["gemv_pos0"]


def _bf16_in_range_weights(rng, shape, scale=0.05):
    w = oracle.bf16_bits_to_f32(oracle.bf16_round(rng.standard_normal(shape).astype(np.float32) * scale))
    mag_bits = oracle.bf16_round(np.abs(w))
    e = (mag_bits.astype(np.int64) >> 7) & 0xFF
    w[(e < 112) | (e > 143)] = np.float32(0.25)  # keep exponents inside [112, 143]
    return w


@pytest.mark.parametrize("seed", range(10))
def test_identity_merges_bit_exact(seed):
    """Self-merge and negated-pair merge reconstruct the source bit-exactly (S:80,
    S:157)."""
    rng = np.random.default_rng(seed)
    rows, cols = rng.integers(1, 129, 2)
    w = _bf16_in_range_weights(rng, (rows, cols))
    n1 = 1 + np.abs(rng.standard_normal(cols)).astype(np.float32)
    n2 = 1 + np.abs(rng.standard_normal(cols)).astype(np.float32)
    art = oracle.merge(w, w, n1, n2)
    assert art["m_sim"].all() and art["m_i"].all() and art["m_j"].all()
    packed, _ = oracle.pack_artifacts(art)
    assert np.array_equal(_reconstruct(packed, 0), w)
    assert np.array_equal(_reconstruct(packed, 1), w)
    art = oracle.merge(w, -w, n1, n2)
    packed, _ = oracle.pack_artifacts(art)
    assert np.array_equal(_reconstruct(packed, 0), w)
    assert np.array_equal(_reconstruct(packed, 1), -w + 0.0)  # -0.0 -> +0.0 (masked / zero)


def test_appendix_b_closed_form_value():
    # P:596-610 with rho=1, tau=0.4: (2/pi)[atan(7/3) - atan(3/7)] = (4/pi) atan(7/3) - 1
    want = 4.0 / math.pi * math.atan(7.0 / 3.0) - 1.0
    assert abs(similarity_fraction_closed(1.0, 0.4) - want) < 1e-15
    assert abs(want - 0.4844758) < 1e-7
    assert similarity_fraction_closed(1.0, 0.0) == 0.0
    # symmetry rho <-> 1/rho
    for tau in (0.1, 0.4, 0.7):
        assert abs(similarity_fraction_closed(2.0, tau) - similarity_fraction_closed(0.5, tau)) < 1e-12


@pytest.mark.parametrize("rho,tau", [(1.0, 0.4), (2.0, 0.4), (1.0, 0.1), (0.5, 0.7)])
def test_similarity_fraction_matches_appendix_b(rho, tau):
    """Fraction of M^sim = 1 entries the oracle produces on i.i.d. N(0,1) vs N(0,rho^2)
    experts equals the closed form within a 4-sigma binomial band."""
    rng = np.random.default_rng(42)
    n_rows, n_cols = 500, 2000
    w_i = rng.standard_normal((n_rows, n_cols)).astype(np.float32)
    w_j = (rho * rng.standard_normal((n_rows, n_cols))).astype(np.float32)
    ones = np.ones(n_cols, np.float32)
    art = oracle.merge(w_i, w_j, ones, ones, tau)
    n = w_i.size
    p = similarity_fraction_closed(rho, tau)
    frac = art["m_sim"].mean()
    assert abs(frac - p) < 4 * math.sqrt(p * (1 - p) / n), (frac, p)
    # with equal norms the exclusive masks split the rest evenly (rho = 1)
    if rho == 1.0:
        excl_i = (art["m_i"] & (1 - art["m_j"])).mean()
        assert abs(excl_i - (1 - p) / 2) < 4 * math.sqrt(0.25 / n) * 2


def test_masks_invariants_and_error_bounds():
    rng = np.random.default_rng(3)
    rows, cols = 256, 384
    w_i = _bf16_in_range_weights(rng, (rows, cols))
    w_j = _bf16_in_range_weights(rng, (rows, cols))
    n_i = 1 + np.abs(rng.standard_normal(cols)).astype(np.float32)
    n_j = 1 + np.abs(rng.standard_normal(cols)).astype(np.float32)
    tau = 0.4
    art = oracle.merge(w_i, w_j, n_i, n_j, tau)
    assert np.all(art["m_i"] | art["m_j"])                          # completeness (Eq. 6)
    assert np.all(art["m_sal_i"] ^ art["m_sal_j"])                  # complementary (Eq. 5)
    assert np.array_equal(art["s_i"], (w_i < 0).astype(np.uint8))  # Eq. 3
    assert np.all(art["w_merged"] >= 0)
    packed, _ = oracle.pack_artifacts(art)
    ulp = lambda x: np.spacing(np.abs(x).astype(np.float32)) * 2 ** 16  # one bf16 ulp
    for pos, w, own_sal in ((0, w_i, art["m_sal_i"]), (1, w_j, art["m_sal_j"])):
        rec = _reconstruct(packed, pos).astype(np.float64)
        sim = art["m_sim"] == 1
        bound = tau * art["w_merged"].astype(np.float64) + ulp(art["w_merged"])
        assert np.all(np.abs(rec - w)[sim] <= bound[sim])
        sal = (~sim) & (own_sal == 1)
        assert np.array_equal(rec[sal], w[sal].astype(np.float64))  # S:181 (bf16 inputs)
        pruned = (~sim) & (own_sal == 0)
        assert np.all(rec[pruned] == 0.0)


def test_tie_goes_to_expert_i_and_zero_rules():
    # equal saliency, dissimilar magnitudes cannot tie; use norms to tie A_i == A_j
    art = oracle.merge([[1.0]], [[-0.25]], [1.0], [4.0], 0.4)
    assert art["m_sim"][0, 0] == 0 and art["m_sal_i"][0, 0] == 1 and art["m_i"][0, 0] == 1
    assert art["w_merged"][0, 0] == 1.0
    # 0/0 -> Delta = 0 -> similar, merged exactly to 0 (reading R4)
    art = oracle.merge([[0.0]], [[-0.0]], [1.0], [1.0], 0.0)
    assert art["m_sim"][0, 0] == 1 and art["w_merged"][0, 0] == 0.0
    assert art["s_j"][0, 0] == 0  # -0.0 is not < 0 (reading R6)
    # (x, 0) -> Delta = 1 -> dissimilar for tau < 1, similar for tau = 1
    assert oracle.merge([[0.5]], [[0.0]], [1.0], [1.0], 0.99)["m_sim"][0, 0] == 0
    assert oracle.merge([[0.5]], [[0.0]], [1.0], [1.0], 1.0)["m_sim"][0, 0] == 1
    with pytest.raises(ValueError):
        oracle.merge([[0.5]], [[0.0]], [1.0], [1.0], 1.5)


def test_scale_equivariance_and_tau_monotonicity():
    rng = np.random.default_rng(5)
    w_i = rng.standard_normal((64, 96)).astype(np.float32)
    w_j = rng.standard_normal((64, 96)).astype(np.float32)
    n_i = 1 + np.abs(rng.standard_normal(96)).astype(np.float32)
    n_j = 1 + np.abs(rng.standard_normal(96)).astype(np.float32)
    a = oracle.merge(w_i, w_j, n_i, n_j, 0.4)
    b = oracle.merge(4 * w_i, 4 * w_j, n_i, n_j, 0.4)  # power of two: exact in f32
    for key in ("m_sim", "m_sal_i", "m_i", "m_j", "s_i", "s_j"):
        assert np.array_equal(a[key], b[key])
    assert np.array_equal(4 * a["w_merged"], b["w_merged"])
    prev = None
    for tau in (0.0, 0.1, 0.3, 0.4, 0.6, 1.0):
        cur = oracle.merge(w_i, w_j, n_i, n_j, tau)["m_sim"]
        if prev is not None:
            assert np.all(prev <= cur)
        prev = cur
    assert prev.all()


def test_packed_bytes_are_half_of_two_bf16_experts():
    """50% compression accounting: one uint16 word per entry replaces
    two bf16 entries."""
    rng = np.random.default_rng(6)
    w_i = rng.standard_normal((32, 48)).astype(np.float32)
    w_j = rng.standard_normal((32, 48)).astype(np.float32)
    ones = np.ones(48, np.float32)
    packed, _ = oracle.pack_artifacts(oracle.merge(w_i, w_j, ones, ones))
    assert packed.nbytes * 2 == 2 * w_i.size * 2
