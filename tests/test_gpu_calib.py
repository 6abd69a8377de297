"""GPU parity for the NEXT-4 calibration statistics (Eq. 4 ||X||_2 inputs)
against the oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import oracle_mixed_layer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    import paper_2511_04805_b200 as pz
    pz.load_library()
    return pz


@pytest.mark.parametrize("cols,counts", [(8, [3, 0, 5]), (512, [1, 1000, 0, 77]), (1416, [4096, 3, 0, 2000, 9])])
def test_group_colsumsq_matches_oracle(pz, cols, counts):
    rng = np.random.default_rng(cols)
    n = sum(counts)
    rows = synth.to_bf16_bits(rng.standard_normal((n, cols)).astype(np.float32) * 3)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    want = oracle.group_colsumsq(rows, off)
    dev_rows = torch.from_numpy(rows.view(np.int16)).cuda()
    got = torch.full((len(counts), cols), 0.5, dtype=torch.float64, device="cuda")  # accumulates
    pz.group_colsumsq(dev_rows, torch.from_numpy(off).cuda(), got)
    # f32 sums of 8 exact squares per thread, then f64: relative error <= ~2^-21
    np.testing.assert_allclose(got.cpu().numpy() - 0.5, want, rtol=1e-6, atol=1e-9)
    a = torch.zeros_like(got)
    b = torch.zeros_like(got)
    pz.group_colsumsq(dev_rows, torch.from_numpy(off).cuda(), a)
    pz.group_colsumsq(dev_rows, torch.from_numpy(off).cuda(), b)
    assert torch.equal(a, b)  # no atomics: bit-reproducible


CASES = [
    (synth.MoEConfig("cal_dense", 21, 256, 512, 8, 2, True), 0),   # an unmerged model: all slots dense
    (synth.MoEConfig("cal_mix", 22, 256, 384, 12, 4, False), 3),   # merged pairs + dense slots
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0].name)
@pytest.mark.parametrize("T", [5, 64, 300])
@pytest.mark.parametrize("path", ["gemv", "tc"])
def test_forward_calib_matches_oracle(pz, case, T, path):
    cfg, n_merged = case
    w13, w2, slot, dense = oracle_mixed_layer(cfg, n_merged)
    layer = pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(), torch.from_numpy(w2.view(np.int16)).cuda(),
                              torch.from_numpy(slot).cuda(), torch.from_numpy(dense).cuda())
    hb = synth.hidden_bits(cfg, T, seed=50 + T)
    lg = synth.router_logits(cfg, T, seed=60 + T)
    h_dev = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    l_dev = torch.from_numpy(lg).cuda()
    P = layer.n_pairs
    sx = torch.zeros((2 * P, cfg.d_model), dtype=torch.float64, device="cuda")
    sh = torch.zeros((2 * P, cfg.d_ff), dtype=torch.float64, device="cuda")
    p = pz.PATH_GEMV if path == "gemv" else pz.PATH_TC
    out = layer.forward_calib(h_dev, l_dev, cfg.top_k, cfg.renormalize, sx, sh, path=p)
    ref_out = layer.forward(h_dev, l_dev, cfg.top_k, cfg.renormalize, path=p)
    torch.cuda.synchronize()
    # the forward is unchanged (bitwise only up to the unspecified in-bucket order, R18: with
    # T > 64 a token's pass may or may not straddle a stream-K cut)
    assert (out.float() - ref_out.float()).abs().max().item() <= 2e-2
    want_x, want_h = oracle.calib_sumsq(w13, slot, hb, lg, cfg.top_k, cfg.renormalize, pair_dense=dense)
    # x rows are copied exactly: only the summation (f32 over 8 rows, then f64) differs
    np.testing.assert_allclose(sx.cpu().numpy(), want_x, rtol=1e-6, atol=0)
    # h is the forward's bf16 SwiGLU row (R16): |h_gpu^2 - h^2| <= ~2 * 2^-8 h^2 + accumulation error
    got_h = sh.cpu().numpy()
    assert np.all(np.abs(got_h - want_h) <= 1.6e-2 * want_h + 1e-6), np.abs(got_h - want_h).max()
    # a second batch accumulates
    layer.forward_calib(h_dev, l_dev, cfg.top_k, cfg.renormalize, sx, None, path=p)
    np.testing.assert_allclose(sx.cpu().numpy(), 2 * want_x, rtol=1e-6, atol=0)
