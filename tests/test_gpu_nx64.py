"""GPU parity of the decode-shape kernels' wide configurations against the f64 oracle FFN under
the north-star tolerance (gemv_tc.cu): NX = 64 (one pass of up to 64 tokens per position, two
TMEM A buffers, partial slots summed from L2 by the stream-K reducer) once experts average more
than 20 tokens (n_assign > 40 * n_pairs), and NX = 128 (one CTA per SM, 512 TMEM columns, 16
decoder warps on K quarters) above 56 tokens per expert (n_assign > 112 * n_pairs)."""
import pytest

import synth
from helpers import assert_close
from test_gpu_moe import _run, pz  # noqa: F401  (module fixture)

pytestmark = pytest.mark.gpu

CASES = [
    # (config, T): average tokens per expert = T k / E
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 100),      # 25 / expert: one pass
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 200),      # 50: NX 64, some buckets two passes
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 250),      # 62.5: NX 128, one pass
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 400),      # 100: NX 128, one pass
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 600),      # 150: NX 128, two passes
    (synth.MoEConfig("nx128_fine", 9, 128, 192, 16, 4, False), 240),  # 60: NX 128, ragged row blocks
    (synth.MoEConfig("nx64_fine", 6, 128, 192, 16, 4, False), 90),    # ragged row blocks (d_ff 3 x 64)
    (synth.MoEConfig("nx64_k6", 7, 192, 320, 12, 6, False), 61),      # 30.5 / expert, top-6
]


@pytest.mark.parametrize("cfg,T", CASES, ids=lambda v: getattr(v, "name", str(v)))
def test_nx64_small(pz, cfg, T):
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV)
    assert_close(got, ref, f"{cfg.name} T={T}")


@pytest.mark.parametrize("T", [41, 64, 100, 200])
def test_nx64_split_items_many_pieces(pz, T):
    """One pair, d_ff 8192: each w2 item (128 K-stages) is split across many CTAs; the reducer
    sums the pieces' fp32 partial slots (up to 128 (position, token) rows) from L2 in CTA order."""
    cfg = synth.MoEConfig("many_pieces", 23, 256, 8192, 2, 1, True)
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV)
    assert_close(got, ref, f"many pieces T={T}")


@pytest.mark.parametrize("T", [150, 300])
def test_nx128_skewed_one_pair(pz, T):
    """Every token on one pair: 150 tokens per position = three passes of 64 (37.5 tokens per
    expert on average: NX 64), 300 = three passes of 128 (75 on average: NX 128); the last
    pass ragged."""
    cfg = synth.MoEConfig("skew", 8, 128, 256, 8, 2, True)
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV, skew=50.0)
    assert_close(got, ref, f"skew T={T}")


@pytest.mark.parametrize("name,T,sample", [("qwen15", 512, 48), ("deepseek", 384, 48), ("qwen15", 1024, 48),
                                           ("deepseek", 768, 48)])
def test_nx64_full_size_fine_grained(pz, name, T, sample):
    """Config 4 layers at intermediate batches (34 / 36 tokens per expert: NX = 64; 68 / 72:
    NX = 128), a seeded token sample against the oracle."""
    cfg = synth.CONFIGS[name]
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV, sample=sample)
    assert_close(got, ref, f"{name} T={T}")


@pytest.mark.slow
@pytest.mark.parametrize("T", [128, 256, 512])
def test_nx64_full_size_mixtral(pz, T):
    """Mixtral layer at 32 / 64 / 128 tokens per expert (the serving regime between decode and
    prefill) through the NX = 64 / 128 configurations (T 512: two passes of 128 for the larger
    buckets); 24 seeded tokens against the oracle."""
    cfg = synth.CONFIGS["mixtral"]
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV, sample=24)
    assert_close(got, ref, f"mixtral T={T}")
