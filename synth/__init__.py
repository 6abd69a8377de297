"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no merge, pack, decode, routing or
FFN): it only draws random numbers with the shapes and distributions of the paper's
workloads and rounds them to bf16 with torch's CPU cast.

Configs follow BASELINE.json ``configs``; seeds follow SURVEY.md §8(d): base 2511,
weights = base + 10*cfg + 1, activations + 2, logits + 3.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

SEED_BASE = 2511


@dataclasses.dataclass(frozen=True)
class MoEConfig:
    name: str
    index: int          # position in BASELINE.json configs (seed derivation)
    d_model: int
    d_ff: int
    n_experts: int
    top_k: int
    renormalize: bool   # Mixtral: softmax over the k selected; Qwen/DeepSeek: full softmax (R13)

    @property
    def n_pairs(self) -> int:
        return self.n_experts // 2


CONFIGS = {
    "tiny": MoEConfig("tiny", 0, 64, 128, 2, 1, True),
    "mixtral": MoEConfig("mixtral", 1, 4096, 14336, 8, 2, True),
    "qwen15": MoEConfig("qwen15", 3, 2048, 1408, 60, 4, False),
    "deepseek": MoEConfig("deepseek", 3, 2048, 1408, 64, 6, False),
}


def seeds(cfg: MoEConfig) -> dict:
    base = SEED_BASE + 10 * cfg.index
    return {"weights": base + 1, "activations": base + 2, "logits": base + 3}


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


def to_bf16_values(x: np.ndarray) -> np.ndarray:
    """Round f32 values to bf16 with torch's CPU cast (a library routine), return f32."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t.to(torch.bfloat16).to(torch.float32).numpy()


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def pairing(cfg: MoEConfig, seed: int | None = None) -> tuple[list[tuple[int, int]], np.ndarray]:
    """Random disjoint pairing (the paper's default), smaller id at pos 0
    (reading R7). Returns (pairs, expert_slot[E] = 2*pair + pos)."""
    seed = seeds(cfg)["weights"] if seed is None else seed
    perm = _rng(seed, 7).permutation(cfg.n_experts)
    pairs = []
    slot = np.empty(cfg.n_experts, np.int32)
    for p in range(cfg.n_pairs):
        a, b = sorted((int(perm[2 * p]), int(perm[2 * p + 1])))
        pairs.append((a, b))
        slot[a] = 2 * p
        slot[b] = 2 * p + 1
    return pairs, slot


SLOTS = ("w1", "w3", "w2")


def slot_shape(cfg: MoEConfig, slot: str) -> tuple[int, int]:
    """(out, in) orientation (reading R11)."""
    return (cfg.d_ff, cfg.d_model) if slot in ("w1", "w3") else (cfg.d_model, cfg.d_ff)


def expert_pair_slot(cfg: MoEConfig, pair: int, slot: str, seed: int | None = None,
                     correlation: float = 0.0):
    """Two experts' bf16-valued weights for one linear slot of one pair, plus their
    Wanda norms (Eq. 4 input). W ~ N(0, 1/in); norms = 1 + |z|.

    correlation in [0,1): W_j = c W_i + sqrt(1-c^2) Z (Mixtral-like correlated experts,
    P:517-530); 0 = independent (Qwen/DeepSeek-like)."""
    seed = seeds(cfg)["weights"] if seed is None else seed
    rows, cols = slot_shape(cfg, slot)
    rng = _rng(seed, pair, SLOTS.index(slot))
    sigma = 1.0 / np.sqrt(cols)
    z_i = rng.standard_normal((rows, cols), dtype=np.float32)
    z_j = rng.standard_normal((rows, cols), dtype=np.float32)
    if correlation:
        z_j = np.float32(correlation) * z_i + np.float32(np.sqrt(1 - correlation ** 2)) * z_j
    w_i = to_bf16_values(z_i * np.float32(sigma))
    w_j = to_bf16_values(z_j * np.float32(sigma))
    n_i = (1.0 + np.abs(rng.standard_normal(cols, dtype=np.float32))).astype(np.float32)
    n_j = (1.0 + np.abs(rng.standard_normal(cols, dtype=np.float32))).astype(np.float32)
    return w_i, w_j, n_i, n_j


def hidden_bits(cfg: MoEConfig, T: int, seed: int | None = None, scale: float = 1.0) -> np.ndarray:
    seed = seeds(cfg)["activations"] if seed is None else seed
    x = _rng(seed, T).standard_normal((T, cfg.d_model), dtype=np.float32) * np.float32(scale)
    return to_bf16_bits(x)


def router_logits(cfg: MoEConfig, T: int, seed: int | None = None, skew: float = 0.0) -> np.ndarray:
    """N(0,1) fp32 logits (uniform expected load); skew adds a fixed per-expert bias."""
    seed = seeds(cfg)["logits"] if seed is None else seed
    rng = _rng(seed, T)
    lg = rng.standard_normal((T, cfg.n_experts), dtype=np.float32)
    if skew:
        lg += np.float32(skew) * _rng(seed, 99).standard_normal(cfg.n_experts, dtype=np.float32)
    return lg


def packed_statistical_torch(cfg: MoEConfig, device, seed: int):
    """Weights for the 32-layer stack / GPU-side bench (generator G2): expert weights
    drawn directly on the device with torch's generator (bf16 N(0, 1/in)), norms 1+|z|.
    Returns per-slot tuples (W_i, W_j, n_i, n_j) stacked over pairs:
      w1/w3: [P, f, d]; w2: [P, d, f]; norms [P, in]."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = {}
    for slot in SLOTS:
        rows, cols = slot_shape(cfg, slot)
        sigma = 1.0 / float(np.sqrt(cols))
        w_i = (torch.randn((cfg.n_pairs, rows, cols), generator=g, device=device) * sigma).to(torch.bfloat16)
        w_j = (torch.randn((cfg.n_pairs, rows, cols), generator=g, device=device) * sigma).to(torch.bfloat16)
        n_i = 1.0 + torch.randn((cfg.n_pairs, cols), generator=g, device=device).abs()
        n_j = 1.0 + torch.randn((cfg.n_pairs, cols), generator=g, device=device).abs()
        out[slot] = (w_i, w_j, n_i, n_j)
    return out
