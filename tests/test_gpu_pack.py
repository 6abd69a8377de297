"""GPU parity for the packer pair (a1)/(a2) and the fused merge+pack (NEXT-1): bit-exact
against the oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    import paper_2511_04805_b200 as pz
    pz.load_library()
    return pz


def _u16(t: torch.Tensor) -> np.ndarray:
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("pos", [0, 1])
def test_unpack_all_words(pz, pos):
    words = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    got = pz.unpack(torch.from_numpy(words.view(np.int16)).cuda(), pos)
    assert np.array_equal(_u16(got.view(torch.int16)), oracle.unpack(words, pos))


@pytest.mark.parametrize("n,offset", [(1, 0), (7, 1), (4099, 3), (1 << 20, 0), (1 << 20, 5)])
def test_unpack_ragged_and_misaligned(pz, n, offset):
    rng = np.random.default_rng(n + offset)
    words = rng.integers(0, 1 << 16, n + offset, dtype=np.uint32).astype(np.uint16)
    dev = torch.from_numpy(words.view(np.int16)).cuda()[offset:]
    for pos in (0, 1):
        got = pz.unpack(dev, pos)
        assert np.array_equal(_u16(got.view(torch.int16)), oracle.unpack(words[offset:], pos))


@pytest.mark.parametrize("n,offset", [(1, 0), (5, 1), (1023, 0), (1 << 20, 0), (1 << 20 | 3, 2)])
def test_pack_bit_exact_random(pz, n, offset):
    rng = np.random.default_rng(n)
    mags = np.abs(rng.standard_normal(n + offset).astype(np.float32)) * np.float32(0.05)
    mags[:: 97] = 0.0
    mags[1:: 101] = np.float32(2.0 ** -30)   # clamped up
    mags[2:: 103] = np.float32(70000.0)      # saturated (exp 143+)
    planes = [rng.integers(0, 2, n + offset, dtype=np.uint8) for _ in range(4)]
    planes[0][:: 5] = 7  # nonzero = 1
    want, want_stats = oracle.pack(mags[offset:], planes[0][offset:], planes[1][offset:],
                                   planes[2][offset:], planes[3][offset:])
    stats = pz.new_stats()
    dev = [torch.from_numpy(a).cuda()[offset:] for a in (mags, *planes)]
    got = pz.merge_pack(dev[0], dev[1], dev[2], dev[3], dev[4], stats=stats)
    assert np.array_equal(_u16(got), want)
    assert stats.cpu().numpy().astype(np.uint64).tolist() == want_stats.tolist()


def test_pack_rne_sweep_over_all_nonnegative_finite_f32(pz):
    """Every non-negative finite f32 bit pattern, in chunks, GPU vs oracle (R3)."""
    chunk = 1 << 26
    z = torch.zeros(chunk, dtype=torch.uint8, device="cuda")
    z_np = np.zeros(chunk, np.uint8)
    for start in range(0, 0x7F800000, chunk):
        n = min(chunk, 0x7F800000 - start)
        u = np.arange(start, start + n, dtype=np.uint32)
        x = u.view(np.float32)
        want, _ = oracle.pack(x, z_np[:n], z_np[:n], z_np[:n], z_np[:n])
        got = pz.merge_pack(torch.from_numpy(x).cuda(), z[:n], z[:n], z[:n], z[:n])
        assert np.array_equal(_u16(got), want), hex(start)


@pytest.mark.parametrize("cfg_name,slot", [("tiny", "w1"), ("tiny", "w2"), ("qwen15", "w1"), ("qwen15", "w2")])
def test_merge_experts_pack_bit_exact(pz, cfg_name, slot):
    cfg = synth.CONFIGS[cfg_name]
    mats = []
    for p in range(min(cfg.n_pairs, 2)):
        mats.append(synth.expert_pair_slot(cfg, p, slot))
    want = []
    st_want = np.zeros(4, np.uint64)
    for w_i, w_j, n_i, n_j in mats:
        packed, st = oracle.pack_artifacts(oracle.merge(w_i, w_j, n_i, n_j, 0.4))
        want.append(packed)
        st_want += st
    to_dev = lambda a: torch.from_numpy(np.stack(a)).cuda()
    wi = to_dev([m[0] for m in mats]).to(torch.bfloat16)
    wj = to_dev([m[1] for m in mats]).to(torch.bfloat16)
    ni = to_dev([m[2] for m in mats])
    nj = to_dev([m[3] for m in mats])
    stats = pz.new_stats()
    got = pz.merge_experts_pack(wi, wj, ni, nj, 0.4, stats=stats)
    assert np.array_equal(_u16(got), np.stack(want))
    assert stats.cpu().numpy().astype(np.uint64).tolist() == st_want.tolist()


def test_merge_experts_pack_edge_values(pz):
    """Zeros, negative zeros, ties, exact-threshold ratios and tiny magnitudes."""
    rng = np.random.default_rng(9)
    rows, cols = 64, 256
    vals = np.array([0.0, -0.0, 1.0, -1.0, 0.25, 3.0 / 7.0, 1e-30, -2.0 ** -20, 0.6, 0.4], np.float32)
    w_i = synth.to_bf16_values(rng.choice(vals, (rows, cols)) * rng.choice([1, 2, 0.5], (rows, cols)).astype(np.float32))
    w_j = synth.to_bf16_values(rng.choice(vals, (rows, cols)))
    n_i = rng.choice(np.array([1.0, 2.0, 4.0, 0.0], np.float32), cols)
    n_j = rng.choice(np.array([1.0, 2.0, 4.0], np.float32), cols)
    for tau in (0.0, 0.4, 1.0, 0.6):
        want, st = oracle.pack_artifacts(oracle.merge(w_i, w_j, n_i, n_j, tau))
        got = pz.merge_experts_pack(torch.from_numpy(w_i).cuda().to(torch.bfloat16),
                                    torch.from_numpy(w_j).cuda().to(torch.bfloat16),
                                    torch.from_numpy(n_i).cuda(), torch.from_numpy(n_j).cuda(), tau)
        assert np.array_equal(_u16(got), want), tau


def test_merge_similarity_decision_near_tau(pz):
    """Eq. 1-2 at the threshold (reading R17): for every bf16 b within a few percent of the
    value that puts |a - b| / (a + b) exactly at tau, over many a, the GPU's similarity decision
    (an approximate quotient with an exact fallback near tau) equals the oracle's correctly
    rounded f32 division -- the packed words must be bit-identical. Also huge, subnormal-sum
    and non-finite cases, where the fallback decides."""
    a_bits = np.arange(0x3C00, 0x4400, 7, dtype=np.uint16)                 # a in ~[2^-7, 2^9)
    a = (a_bits.astype(np.uint32) << 16).view(np.float32)
    rows = []
    for tau in (0.4, 0.6, 0.1, 1.0 / 3.0):
        tau32 = np.float32(tau)
        for av in a[:: max(1, len(a) // 96)]:
            b0 = np.float32(av * (1 - tau32) / (1 + tau32))
            b_bits = (b0.view(np.uint32) >> 16).astype(np.int64) + np.arange(-24, 24)
            b = (b_bits.astype(np.uint32) << 16).view(np.float32)
            rows.append((np.full_like(b, av), b, tau32))
    extra_i = np.array([3.0e38, 1e-39, -1e-39, np.inf, 2.0 ** -126, 1.0], np.float32)
    extra_j = np.array([3.0e38, 1e-39, 1e-39, 1.0, 2.0 ** -126, np.nan], np.float32)
    for tau in (0.4, 0.6, 0.1, 1.0 / 3.0):
        w_i = np.concatenate([r[0] for r in rows if r[2] == np.float32(tau)] + [extra_i])
        w_j = np.concatenate([r[1] for r in rows if r[2] == np.float32(tau)] + [extra_j])
        pad = (-len(w_i)) % 8
        w_i = np.concatenate([w_i, np.ones(pad, np.float32)])[None, :]
        w_j = np.concatenate([w_j, np.ones(pad, np.float32)])[None, :]
        w_i, w_j = synth.to_bf16_values(w_i), synth.to_bf16_values(w_j)
        n = np.ones(w_i.shape[1], np.float32)
        want, _ = oracle.pack_artifacts(oracle.merge(w_i, w_j, n, n, float(np.float32(tau))))
        got = pz.merge_experts_pack(torch.from_numpy(w_i).cuda().to(torch.bfloat16),
                                    torch.from_numpy(w_j).cuda().to(torch.bfloat16),
                                    torch.from_numpy(n).cuda(), torch.from_numpy(n).cuda(), float(np.float32(tau)))
        assert np.array_equal(_u16(got), want), tau
