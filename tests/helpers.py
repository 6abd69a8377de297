"""Test-side helpers: build oracle-packed layers from the seeded generator, upload them,
and compare GPU outputs with the oracle under the north-star tolerance."""
from __future__ import annotations

import functools

import numpy as np

import oracle
import synth

# BASELINE.json north_star: "max abs error <= 2e-2 and relative L2 <= 5e-3 against an
# fp32-accumulated oracle on bf16 inputs" (our oracle accumulates in f64, R16/R17).
MAX_ABS = 2e-2
REL_L2 = 5e-3


@functools.lru_cache(maxsize=8)
def oracle_packed_layer(cfg: synth.MoEConfig, seed: int | None = None, tau: float = 0.4):
    """Packed w13 [P,2,f,d], w2 [P,d,f] (uint16) merged + packed by the ORACLE from the
    generator's expert weights, plus expert_slot and pack stats."""
    _, slot = synth.pairing(cfg, seed)
    P, d, f = cfg.n_pairs, cfg.d_model, cfg.d_ff
    w13 = np.empty((P, 2, f, d), np.uint16)
    w2 = np.empty((P, d, f), np.uint16)
    stats = np.zeros(4, np.uint64)
    for p in range(P):
        for s_idx, slot_name in enumerate(synth.SLOTS):
            w_i, w_j, n_i, n_j = synth.expert_pair_slot(cfg, p, slot_name, seed)
            art = oracle.merge(w_i, w_j, n_i, n_j, tau)
            packed, st = oracle.pack_artifacts(art)
            stats += st
            if slot_name == "w1":
                w13[p, 0] = packed
            elif slot_name == "w3":
                w13[p, 1] = packed
            else:
                w2[p] = packed
            del art, w_i, w_j
    return w13, w2, slot, stats


def compare(gpu_out: np.ndarray, ref: np.ndarray) -> dict:
    g = gpu_out.astype(np.float64)
    r = ref.astype(np.float64)
    diff = g - r
    max_abs = float(np.abs(diff).max()) if diff.size else 0.0
    denom = float(np.linalg.norm(r)) or 1.0
    rel = float(np.linalg.norm(diff)) / denom
    return {"max_abs": max_abs, "rel_l2": rel}


def assert_close(gpu_out: np.ndarray, ref: np.ndarray, what: str = ""):
    m = compare(gpu_out, ref)
    assert m["max_abs"] <= MAX_ABS and m["rel_l2"] <= REL_L2, f"{what}: {m}"
    return m


@functools.lru_cache(maxsize=8)
def oracle_mixed_layer(cfg: synth.MoEConfig, n_merged: int, seed: int | None = None, tau: float = 0.4):
    """The 25%-ratio layout (reading R20): the generator's first `n_merged` pairs merged +
    packed by the ORACLE, every other expert kept as plain bf16 bits in a dense slot of its
    own; slots in a seeded random order. Returns w13 [P',2,f,d], w2 [P',d,f] (uint16),
    expert_slot [E] and pair_dense [P'] with P' = E - n_merged."""
    pairs, _ = synth.pairing(cfg, seed)
    d, f = cfg.d_model, cfg.d_ff
    n_slots = cfg.n_experts - n_merged
    order = np.random.default_rng(1234 + n_merged).permutation(n_slots)
    w13 = np.empty((n_slots, 2, f, d), np.uint16)
    w2 = np.empty((n_slots, d, f), np.uint16)
    slot = np.empty(cfg.n_experts, np.int32)
    dense = np.zeros(n_slots, np.uint8)
    nxt = 0
    for p, (a, b) in enumerate(pairs):
        per = {}
        for slot_name in synth.SLOTS:
            w_i, w_j, n_i, n_j = synth.expert_pair_slot(cfg, p, slot_name, seed)
            if p < n_merged:
                per[slot_name] = (oracle.pack_artifacts(oracle.merge(w_i, w_j, n_i, n_j, tau))[0],)
            else:
                per[slot_name] = (synth.to_bf16_bits(w_i), synth.to_bf16_bits(w_j))
        if p < n_merged:
            q = int(order[nxt]); nxt += 1
            w13[q, 0], w13[q, 1], w2[q] = per["w1"][0], per["w3"][0], per["w2"][0]
            slot[a], slot[b] = 2 * q, 2 * q + 1
        else:
            for j, e in enumerate((a, b)):
                q = int(order[nxt]); nxt += 1
                w13[q, 0], w13[q, 1], w2[q] = per["w1"][j], per["w3"][j], per["w2"][j]
                slot[e] = 2 * q
                dense[q] = 1
    return w13, w2, slot, dense


# ---- fixed-capacity EP index tables, restated from include/puzzlemoe.h (puzzle_ep_*) ----
# Plain numpy statements of what the three index kernels must produce; the GPU tests compare
# the kernels with these, the gloo tests use them as the CPU stand-in of the device ops.

def ep_dispatch_ref(hidden, assign_token, off, dest_pairs, cap, lb_max):
    """send_rows [G*(cap+1)][d] int16: per destination q, its rows then a header row whose first
    2*lb_max 16-bit words are the int32 counts of q's local buckets (everything unwritten 0)."""
    G = len(dest_pairs)
    R = cap + 1
    rows = np.zeros((G * R, hidden.shape[1]), np.int16)
    for q, (lo, hi) in enumerate(dest_pairs):
        a, b = off[2 * lo], off[2 * hi]
        rows[q * R:q * R + (b - a)] = hidden[assign_token[a:b]]
        counts = np.zeros(lb_max, np.int32)
        counts[:2 * (hi - lo)] = np.diff(off[2 * lo:2 * hi + 1])
        rows[q * R + cap, :2 * lb_max] = counts.view(np.int16)
    return rows


def ep_recv_plan_ref(recv_rows, world, lb, cap):
    """(local_off [lb+1], gather_idx [G*cap], return_idx [G*(cap+1)]) from the header counts of
    an int16 [G*(cap+1)][d] region buffer; local order (bucket, source)."""
    R = cap + 1
    rows = np.asarray(recv_rows).reshape(world, R, -1)
    rc = np.ascontiguousarray(rows[:, cap, :2 * lb]).view(np.int32).astype(np.int64).reshape(world, lb)
    local_off = np.concatenate([[0], np.cumsum(rc.sum(0))]).astype(np.int32)
    gidx = np.zeros(world * cap, np.int32)
    ridx = np.zeros(world * R, np.int32)
    l = 0
    for b in range(lb):
        for s in range(world):
            w0 = rc[s, :b].sum()
            for w in range(rc[s, b]):
                gidx[l] = s * R + w0 + w
                ridx[s * R + w0 + w] = l
                l += 1
    return local_off, gidx, ridx


def ep_home_index_ref(assign_of, gate, off, dest_pairs, slices, cap):
    """(aof_s [T*k*S], gate_s [T][k*S])."""
    T, k = gate.shape
    aof = np.asarray(assign_of).reshape(-1)
    aof_s = np.zeros(T * k * slices, np.int32)
    gate_s = np.zeros((T * k, slices), np.float32)
    for i, a in enumerate(aof):
        g = int(np.searchsorted(off, a, side="right")) - 1
        p = g // 2
        owners = [q for q, (lo, hi) in enumerate(dest_pairs) if lo <= p < hi]
        assert len(owners) == slices
        for s, q in enumerate(owners):
            aof_s[i * slices + s] = q * (cap + 1) + (a - off[2 * dest_pairs[q][0]])
            gate_s[i, s] = gate.reshape(-1)[i]
    return aof_s, gate_s.reshape(T, k * slices)
