"""GPU parity of the prefill-shape paths (PUZZLE_PATH_TS: decoded weights as the TMEM A
operand with up to 384 tokens of a bucket on N; PUZZLE_PATH_TC: shared-memory-operand grouped
GEMM) against the f64 oracle FFN (Eq. 8 / Alg. 1), under the north-star
tolerance; plus the full-size configs at the token counts the bench times (BASELINE.json
configs 3 and 4, T = 4096) on seeded token samples that include the heaviest buckets."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_close, oracle_mixed_layer, oracle_packed_layer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pz():
    import paper_2511_04805_b200 as pz
    pz.load_library()
    return pz


def _layer(pz, cfg):
    w13, w2, slot, _ = oracle_packed_layer(cfg)
    return pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(),
                             torch.from_numpy(w2.view(np.int16)).cuda(),
                             torch.from_numpy(slot).cuda()), (w13, w2, slot)


def _heavy_sample(cfg, lg, slot, n, seed=7):
    """n seeded token rows: half uniformly at random, half among the tokens routed to the
    fullest buckets (the multi-chunk / second-tile cases)."""
    T = lg.shape[0]
    top = np.argsort(-lg, axis=1, kind="stable")[:, :cfg.top_k]
    buckets = slot[top]                                           # [T, k] bucket of each assignment
    counts = np.bincount(buckets.ravel(), minlength=2 * cfg.n_pairs)
    heavy = np.argsort(-counts, kind="stable")[:4]
    in_heavy = np.flatnonzero(np.isin(buckets, heavy).any(axis=1))
    rng = np.random.default_rng(seed)
    a = rng.choice(in_heavy, min(n // 2, len(in_heavy)), replace=False)
    rest = np.setdiff1d(np.arange(T), a)
    b = rng.choice(rest, n - len(a), replace=False)
    return np.sort(np.concatenate([a, b])), int(counts.max())


def _run(pz, cfg, T, path, sample=None, skew=0.0, seed_shift=0):
    layer, (w13, w2, slot) = _layer(pz, cfg)
    hb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + seed_shift)
    lg = synth.router_logits(cfg, T, seed=synth.seeds(cfg)["logits"] + seed_shift, skew=skew)
    rb = synth.hidden_bits(cfg, T, seed=synth.seeds(cfg)["activations"] + 1000 + seed_shift)
    out = layer.forward(torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16), torch.from_numpy(lg).cuda(),
                        cfg.top_k, cfg.renormalize,
                        residual=torch.from_numpy(rb.view(np.int16)).cuda().view(torch.bfloat16), path=path)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    max_bucket = None
    if sample is None:
        rows = np.arange(T)
    else:
        rows, max_bucket = _heavy_sample(cfg, lg, slot, sample)
    ref = oracle.moe_forward(w13, w2, slot, hb[rows], lg[rows], cfg.top_k, cfg.renormalize, rb[rows])
    return got[rows], ref, max_bucket


PATHS = {"ts": 3, "tc": 2}
SMALL = [
    synth.MoEConfig("pf_small", 10, 256, 256, 8, 2, True),
    synth.MoEConfig("pf_fine", 11, 512, 384, 16, 4, False),   # d_ff = 3 x 128
    synth.MoEConfig("pf_odd", 15, 384, 192, 12, 3, False),    # d_model = 3 x 128, d_ff = 3 x 64 (TS only)
]


@pytest.mark.parametrize("path", ["ts", "tc"])
@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: c.name)
@pytest.mark.parametrize("T", [1, 5, 65, 130, 300, 777])
def test_prefill_small(pz, path, cfg, T):
    if path == "tc" and (cfg.d_model % 256 or cfg.d_ff % 128):
        pytest.skip("the shared-memory-operand kernel needs d_model % 256 and d_ff % 128")
    got, ref, _ = _run(pz, cfg, T, PATHS[path])
    assert_close(got, ref, f"{path} {cfg.name} T={T}")


@pytest.mark.parametrize("path", ["ts", "tc"])
def test_prefill_skewed_multi_chunk(pz, path):
    """Buckets of > 384 (and > 768) tokens: several token chunks of one bucket (TS), several
    256-row M tiles with a partial last one (TC)."""
    cfg = synth.MoEConfig("pf_skew", 12, 256, 256, 8, 2, True)
    got, ref, mb = _run(pz, cfg, 1500, PATHS[path], skew=50.0, sample=96)
    assert mb > 768
    assert_close(got, ref, f"{path} skew")


@pytest.mark.parametrize("T", [65, 128, 256, 512, 1024])
def test_prefill_ts_intermediate_batches(pz, T):
    """The 65-1024 token regime (the paper's own workload uses 1024-token prefills)."""
    cfg = synth.MoEConfig("pf_mid", 16, 512, 512, 16, 2, True)
    got, ref, _ = _run(pz, cfg, T, PATHS["ts"])
    assert_close(got, ref, f"ts mid T={T}")


@pytest.mark.parametrize("case", [(synth.MoEConfig("pfmix", 12, 256, 512, 8, 2, True), 2),
                                  (synth.MoEConfig("pfmix_all", 14, 256, 256, 6, 2, True), 0)],
                         ids=["two_merged", "all_dense"])
@pytest.mark.parametrize("T", [65, 400])
def test_prefill_ts_dense_slots(pz, case, T):
    """25 % ratio layout (reading R20): dense bf16 slots skip Algorithm 1 in the TS kernel."""
    cfg, n_merged = case
    w13, w2, slot, dense = oracle_mixed_layer(cfg, n_merged)
    layer = pz.PackedMoELayer(torch.from_numpy(w13.view(np.int16)).cuda(), torch.from_numpy(w2.view(np.int16)).cuda(),
                              torch.from_numpy(slot).cuda(), torch.from_numpy(dense).cuda())
    hb = synth.hidden_bits(cfg, T)
    lg = synth.router_logits(cfg, T)
    out = layer.forward(torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16), torch.from_numpy(lg).cuda(),
                        cfg.top_k, cfg.renormalize, path=PATHS["ts"])
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, None, pair_dense=dense)
    assert_close(out.float().cpu().numpy(), ref, f"ts dense {cfg.name} T={T}")


@pytest.mark.parametrize("path", ["ts", "tc"])
@pytest.mark.parametrize("name", ["qwen15", "deepseek"])
def test_prefill_full_size_fine_grained_4096(pz, path, name):
    """BASELINE config 4 prefill at the benchmarked T = 4096: 64 seeded tokens, half of them
    from the four fullest buckets (> 256 tokens each: second M tile / multi-chunk paths)."""
    cfg = synth.CONFIGS[name]
    got, ref, mb = _run(pz, cfg, 4096, PATHS[path], sample=64)
    assert mb > 256
    assert_close(got, ref, f"{path} {name} T=4096")


@pytest.mark.slow
@pytest.mark.parametrize("path", ["ts", "tc"])
def test_prefill_full_size_mixtral_4096(pz, path):
    """BASELINE config 3 (Mixtral layer, T = 4096): a seeded 256-token sample (BASELINE.md
    section 4.2), half of it from the fullest buckets."""
    cfg = synth.CONFIGS["mixtral"]
    got, ref, _ = _run(pz, cfg, 4096, PATHS[path], sample=256)
    assert_close(got, ref, f"{path} mixtral T=4096")


def test_prefill_ts_matches_tc(pz):
    """Both prefill kernels on one layer and batch: same values up to accumulation order."""
    cfg = SMALL[1]
    layer, _ = _layer(pz, cfg)
    T = 900
    hb = torch.from_numpy(synth.hidden_bits(cfg, T).view(np.int16)).cuda().view(torch.bfloat16)
    lg = torch.from_numpy(synth.router_logits(cfg, T)).cuda()
    a = layer.forward(hb, lg, cfg.top_k, cfg.renormalize, path=PATHS["ts"]).float()
    b = layer.forward(hb, lg, cfg.top_k, cfg.renormalize, path=PATHS["tc"]).float()
    torch.cuda.synchronize()
    assert (a - b).abs().max().item() <= 2e-2
