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
