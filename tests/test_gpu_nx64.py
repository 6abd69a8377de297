"""GPU parity of the decode-shape kernels' NX = 64 configuration (gemv_tc.cu: one pass of up to
64 tokens per position, two TMEM A buffers, partial slots summed from L2 by the stream-K
reducer), which runs once experts average more than 20 tokens (n_assign > 40 * n_pairs),
against the f64 oracle FFN under the north-star tolerance."""
import pytest

import synth
from helpers import assert_close
from test_gpu_moe import _run, pz  # noqa: F401  (module fixture)

pytestmark = pytest.mark.gpu

CASES = [
    # (config, T): average tokens per expert = T k / E
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 100),      # 25 / expert: one pass
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 250),      # 62.5: one pass, some buckets two
    (synth.MoEConfig("nx64_mix", 5, 256, 512, 8, 2, True), 400),      # 100: two passes of 64
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


def test_nx64_skewed_one_pair(pz):
    """Every token on one pair: 150 tokens per position = three passes of 64 (the last ragged)."""
    cfg = synth.MoEConfig("skew", 8, 128, 256, 8, 2, True)
    got, ref = _run(pz, cfg, 150, pz.PATH_GEMV, skew=50.0)
    assert_close(got, ref, "skew nx64")


@pytest.mark.parametrize("name,T,sample", [("qwen15", 512, 48), ("deepseek", 384, 48)])
def test_nx64_full_size_fine_grained(pz, name, T, sample):
    """Config 4 layers at intermediate batches (34 / 36 tokens per expert) through the NX = 64
    decode configuration, a seeded token sample against the oracle."""
    cfg = synth.CONFIGS[name]
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV, sample=sample)
    assert_close(got, ref, f"{name} T={T}")


@pytest.mark.slow
@pytest.mark.parametrize("T", [128, 256])
def test_nx64_full_size_mixtral(pz, T):
    """Mixtral layer at 32 / 64 tokens per expert (the paper's serving regime between decode and
    prefill) through the NX = 64 configuration; 24 seeded tokens against the oracle."""
    cfg = synth.CONFIGS["mixtral"]
    got, ref = _run(pz, cfg, T, pz.PATH_GEMV, sample=24)
    assert_close(got, ref, f"mixtral T={T}")
