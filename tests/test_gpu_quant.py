"""GPU parity for the NEXT-3 quantised packer pair (puzzle_quant_pack / puzzle_quant_unpack)
against the oracle, bit for bit (codes, scales, dequantised bf16), through the C ABI."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    import paper_2511_04805_b200 as pz
    pz.load_library()
    return pz


def _case(rows, cols, seed, kind="gauss"):
    rng = np.random.default_rng(seed)
    if kind == "gauss":
        w = np.abs(rng.standard_normal((rows, cols))).astype(np.float32) * rng.choice(
            [1e-4, 1.0, 300.0], (rows, 1)).astype(np.float32)
    elif kind == "ties":  # 7 w / max lands exactly on k + 1/2 for many entries
        mx = np.float32(4.0)
        w = (rng.integers(0, 7, (rows, cols)).astype(np.float32) + np.float32(0.5)) * (mx / np.float32(7.0))
        w[:, ::128] = mx
    else:  # zeros, single values, subnormals, negatives clamp to 0
        w = np.zeros((rows, cols), np.float32)
        w[::3, 5] = 1e-40
        w[1::3, 7] = 2.5
        w[2::3, 9] = -1.0
    planes = [(rng.random((rows, cols)) < 0.5).astype(np.uint8) for _ in range(4)]
    return w, planes


@pytest.mark.parametrize("rows,cols,kind", [(1, 128, "gauss"), (7, 384, "gauss"), (256, 1408, "gauss"),
                                            (64, 4096, "ties"), (9, 256, "edge")])
def test_quant_pack_unpack_bit_exact(pz, rows, cols, kind):
    w, (m0, m1, s0, s1) = _case(rows, cols, rows * 7 + cols, kind)
    want_codes, want_scales = oracle.quant_pack(w, m0, m1, s0, s1)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    codes, scales = pz.quant_pack(dev(w), dev(m0), dev(m1), dev(s0), dev(s1))
    torch.cuda.synchronize()
    assert np.array_equal(codes.cpu().numpy(), want_codes)
    assert np.array_equal(scales.cpu().numpy().view(np.uint32), want_scales.view(np.uint32))
    for pos in (0, 1):
        got = pz.quant_unpack(codes, scales, pos).view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, oracle.quant_unpack(want_codes, want_scales, pos)), pos


def test_quant_argument_errors(pz):
    x = torch.zeros((2, 100), dtype=torch.float32, device="cuda")
    u = torch.zeros((2, 100), dtype=torch.uint8, device="cuda")
    with pytest.raises(pz.PuzzleError):
        pz.quant_pack(x, u, u, u, u)  # cols % 128 != 0


def _bf16_tokens(n, cols, seed):
    return torch.randn(n, cols, generator=torch.Generator().manual_seed(seed)).to(torch.bfloat16)


@pytest.mark.parametrize("rows,cols,n_i,n_j", [(1, 128, 1, 0), (3, 128, 0, 2), (1023, 4096, 1, 1), (513, 1408, 2, 1), (65, 512, 3, 7),
                                               (37, 384, 5, 9), (256, 1408, 8, 17),
                                               (1023, 4096, 23, 3), (4096, 14336, 12, 20)])
def test_quant_gemv_matches_oracle(pz, rows, cols, n_i, n_j):
    """puzzle_quant_gemv vs oracle.quant_gemv (f64): ragged row pairs (odd rows), token chunks of
    1 / 2 / 4 tokens per position (all three kernel instances) with ragged tails, an empty side, and the Mixtral w2 shape (4096 x 14336) of one merged
    pair. Tolerance derived from the kernel's summation: each lane sums cols/32 products in order
    and a 5-level tree follows, so |err| <= (cols/32 + 5) * 2^-24 * sum|w x| (plus one rounding
    of the sum), here with a factor 2 margin."""
    w, planes = _case(rows, cols, rows + cols)
    codes_np, scales_np = oracle.quant_pack(w, *planes)
    xi, xj = _bf16_tokens(n_i, cols, 1), _bf16_tokens(n_j, cols, 2)
    bits = [t.view(torch.int16).numpy().view(np.uint16) for t in (xi, xj)]
    want_i, want_j = oracle.quant_gemv(codes_np, scales_np, *bits)
    codes, scales = torch.from_numpy(codes_np).cuda(), torch.from_numpy(scales_np).cuda()
    y_i, y_j = pz.quant_gemv(codes, scales, xi.cuda(), xj.cuda())
    torch.cuda.synchronize()
    for pos, (x, got, want) in enumerate(((xi, y_i, want_i), (xj, y_j, want_j))):
        assert got.shape == (x.shape[0], rows)
        if x.shape[0] == 0:
            continue
        wabs = np.abs(oracle.bf16_bits_to_f32(oracle.quant_unpack(codes_np, scales_np, pos)).astype(np.float64))
        bound = np.abs(x.double().numpy()) @ wabs.T
        tol = 2 * ((cols / 32 + 6) * 2.0 ** -24) * bound + 1e-30
        err = np.abs(got.cpu().double().numpy() - want)
        assert (err <= tol).all(), (pos, float(err.max()), float((err / np.maximum(bound, 1e-30)).max()))


def test_quant_gemv_argument_errors(pz):
    codes = torch.zeros((4, 100), dtype=torch.uint8, device="cuda")
    with pytest.raises(pz.PuzzleError):
        pz.quant_gemv(codes, torch.ones((4, 1), device="cuda"), torch.zeros((1, 100), dtype=torch.bfloat16,
                      device="cuda"), torch.zeros((0, 100), dtype=torch.bfloat16, device="cuda"))
