#!/usr/bin/env python
"""PuzzleMoE packed-expert MoE layer benchmark (B200, sm_100a).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config mixtral] [--batch 64] [--no-extra]

One step = one puzzle_moe_forward over one batch: route + top-k gates (a3), gate/up
projections over the on-the-fly decoded packed experts with SwiGLU (a4), down projection
(a5), combine (a6) -- the whole hot path of SURVEY.md §8(a) (pack (a1) is offline; its
GB/s is reported under "aux"). Default workload = BASELINE.json configs[1]: one
Mixtral-8x7B MoE layer (4096 x 14336, 8 experts merged into 4 pairs, top-2) at decode
batch 64 on one B200. Weights are synthetic (seeded N(0, 1/in) experts merged + packed on
the GPU by puzzle_merge_experts_pack); the packed layer (1.41 GB) is >10x the 126 MB L2,
so no L2 flush is needed for the headline (smaller secondary configs flush L2 per step).

Rank 0 prints ONE JSON line. Under torchrun (N > 1) the layer runs expert-parallel: every
rank holds its share of the merged pairs and its own batch of tokens (weak scaling), tokens go
to the pair owners and back with NCCL all-to-all -- fixed-capacity dispatch (device-only,
CUDA-graph captured) for decode batches, variable splits for prefill -- and the time is the
max over ranks.

--impl reference times the CPU oracle (oracle/, plain C) on the host cores on a bounded
sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "MoE-layer tokens/s at 1/2/4/8 B200 (decode & prefill); % HBM / tensor roofline"
FALLBACK_HBM_GBS = 6650.0     # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)
FALLBACK_BF16_TFLOPS = 1590.0


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": FALLBACK_HBM_GBS, "bf16_tflops": FALLBACK_BF16_TFLOPS,
            "bf16_tflops_sustained": 1400.0, "source": "fallback (B200_PROFILING.md)"}


# --------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    """Samples SM clock + clock-event reasons every 20 ms on a thread (NVML)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device_index: int):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            want = str(getattr(torch.cuda.get_device_properties(device_index), "uuid", "")).lower()
            self.h = None
            for i in range(pynvml.nvmlDeviceGetCount()):
                h = pynvml.nvmlDeviceGetHandleByIndex(i)
                u = pynvml.nvmlDeviceGetUUID(h)
                u = (u.decode() if isinstance(u, bytes) else u).lower()
                if want and want in u:
                    self.h = h
                    break
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.nvml = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - reported in the JSON line
            self.err = repr(e)
        self._stop = threading.Event()
        self.mark = None

    def _run(self):
        n = self.nvml
        while not self._stop.is_set():
            try:
                mhz = n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)
                try:
                    reasons = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    reasons = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, reasons))
            except Exception:
                pass
            time.sleep(0.02)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self, t0: float, t1: float) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        use = inside if inside else self.samples
        mhz = [s[1] for s in use]
        mask = 0
        for s in use:
            mask |= s[2]
        reasons = [k for k, v in self.REASONS.items() if mask & v]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(use), "samples_in_timed_region": len(inside)}


# --------------------------------------------------------------------------- workload
def build_layer_gpu(pz, cfg, seed: int, device, ratio: float = 0.5):
    """Synthetic experts drawn on the GPU (generator G1 statistics) and merged + packed by
    puzzle_merge_experts_pack (Eq. 1-7 + pack, tau = 0.4). ratio 0.5: every pair merged;
    ratio 0.25 (reading R20): the first E/4 pairs merged, the other experts kept as
    dense bf16 slots (E/4 + E/2 = 3E/4 slots); ratio 1.0: the unmerged model, every expert a
    dense slot."""
    import torch
    pairs, slot = synth.pairing(cfg, seed)
    w = synth.packed_statistical_torch(cfg, device, seed)
    stats = pz.new_stats(device)
    n_merged = cfg.n_pairs if ratio == 0.5 else cfg.n_experts // 4 if ratio == 0.25 else 0  # 1.0: unmerged
    packed = {}
    for name, (w_i, w_j, n_i, n_j) in w.items():
        merged = pz.merge_experts_pack(w_i[:n_merged].contiguous(), w_j[:n_merged].contiguous(),
                                       n_i[:n_merged].contiguous(), n_j[:n_merged].contiguous(), 0.4, stats=stats)
        if n_merged < cfg.n_pairs:  # dense slots: expert i then expert j of each unmerged pair
            rest = torch.stack([w_i[n_merged:], w_j[n_merged:]], dim=1).flatten(0, 1).view(torch.int16)
            merged = torch.cat([merged, rest])
        packed[name] = merged
    del w
    dense = None
    if n_merged < cfg.n_pairs:
        for p, (a, b) in enumerate(pairs[n_merged:]):
            slot[a], slot[b] = 2 * (n_merged + 2 * p), 2 * (n_merged + 2 * p + 1)
        dense = torch.tensor([0] * n_merged + [1] * (2 * (cfg.n_pairs - n_merged)), dtype=torch.uint8, device=device)
    w13 = torch.stack([packed["w1"], packed["w3"]], dim=1).contiguous()
    layer = pz.PackedMoELayer(w13, packed["w2"].contiguous(), torch.from_numpy(slot).to(device), dense)
    torch.cuda.synchronize(device)
    return layer, stats.cpu().tolist()


def make_inputs(cfg, T: int, seed: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    hidden = torch.randn((T, cfg.d_model), generator=g, device=device).to(torch.bfloat16)
    logits = torch.randn((T, cfg.n_experts), generator=g, device=device)
    return hidden, logits


def touched_pairs(layer, logits, cfg) -> int:
    _, _, off, _, _ = layer.route(logits, cfg.top_k, cfg.renormalize)
    off = off.cpu().numpy()
    cnt = np.diff(off).reshape(-1, 2).sum(1)
    return int((cnt > 0).sum())


def algorithmic_bytes(cfg, n_touched: int, T: int) -> dict:
    """per touched pair the packed words are read once: w13 = 2*f*d*2 B,
    w2 = d*f*2 B; activations are <1% and counted separately."""
    w13 = n_touched * 2 * cfg.d_ff * cfg.d_model * 2
    w2 = n_touched * cfg.d_model * cfg.d_ff * 2
    acts = T * cfg.d_model * 2 + T * cfg.n_experts * 4 + T * cfg.d_model * 2
    return {"w13": w13, "w2": w2, "acts": acts, "total": w13 + w2 + acts}


def l2_bytes(device) -> int:
    import torch
    try:
        return int(torch.cuda.get_device_properties(device).L2_cache_size)
    except Exception:
        return 126 * 1024 * 1024


def l2_flusher(device):
    """L2 flush between timed steps, outside the events: write a buffer of 2x L2, then read
    another 2x L2 buffer, so L2 holds clean lines when the step starts (a write-only flush
    leaves ~L2 of dirty lines whose write-back would share HBM with the step's weight stream)."""
    import torch
    wbuf = torch.empty(2 * l2_bytes(device), dtype=torch.uint8, device=device)
    rbuf = torch.ones(2 * l2_bytes(device) // 4, dtype=torch.float32, device=device)

    def flush():
        wbuf.zero_()
        torch.amax(rbuf)
    return flush


def timed_steps(step, K: int, flush=None, stream=None):
    """Device time of K steps with CUDA events on the launching stream. Without flush:
    one event pair around the K back-to-back steps. With flush: an event pair per step,
    the L2 flush runs between timed steps outside the events."""
    import torch
    s = stream or torch.cuda.current_stream()
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(K):
            step()
        e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1)
    pairs = []
    for _ in range(K):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        step()
        e1.record(s)
        pairs.append((e0, e1))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in pairs)


def unpacked_baseline(pz, layer, cfg, hidden, logits, K: int, W: int):
    """The unpacked bf16 expert-FFN baseline on the same box, two arms:
      same_kernels -- THIS library on the unmerged layer (every expert a dense bf16 slot, R20):
                      the same route / decode-shape tcgen05 kernels / combine, CUDA-graph replay,
                      reading 2x the bytes -- the like-for-like ratio the paper's 1.28x is about;
      cublas       -- the experts decoded ONCE to dense bf16 (puzzle_unpack), each step torch
                      routing + every expert's cuBLAS bf16 matmuls over all tokens with the gate
                      as a per-token weight (0 for unrouted tokens): no host synchronisation,
                      captured in a CUDA graph (decode: every expert's weights are read once,
                      as in the routed form)."""
    import torch
    res = {}
    dense_layer, _ = build_layer_gpu(pz, cfg, synth.seeds(cfg)["weights"], hidden.device, ratio=1.0)
    out_d = torch.empty_like(hidden)
    ws_d = dense_layer.workspace(hidden.shape[0], cfg.top_k)
    fwd = lambda: dense_layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out_d, workspace=ws_d)
    for _ in range(W):
        fwd()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fwd()
    for _ in range(W):
        g.replay()
    torch.cuda.synchronize()
    ms = timed_steps(g.replay, K) / K
    nt = touched_pairs(dense_layer, logits, cfg)
    dense_bytes = nt * 3 * cfg.d_model * cfg.d_ff * 2  # dense slots touched x one expert's bf16 weights
    res["same_kernels"] = {"ms_per_step": ms, "tokens_per_s": hidden.shape[0] / (ms / 1e3), "weight_bytes": dense_bytes,
                           "achieved_gbs": dense_bytes / (ms / 1e3) / 1e9, "slots": dense_layer.n_pairs,
                           "how": "this library's forward on the unmerged layer (every expert a dense bf16 slot), "
                                  "CUDA-graph replay"}
    del dense_layer, ws_d
    torch.cuda.empty_cache()

    _, slot = synth.pairing(cfg, None)
    dev = hidden.device
    E, d, f = cfg.n_experts, cfg.d_model, cfg.d_ff
    w13 = torch.empty((E, 2 * f, d), dtype=torch.bfloat16, device=dev)
    w2 = torch.empty((E, d, f), dtype=torch.bfloat16, device=dev)
    slot_dev = layer.expert_slot.cpu().numpy()
    for e in range(E):
        p, pos = divmod(int(slot_dev[e]), 2)
        pz.unpack(layer.w13[p].reshape(-1), pos, out=w13[e].reshape(-1))
        pz.unpack(layer.w2[p].reshape(-1), pos, out=w2[e].reshape(-1))
    k, renorm = cfg.top_k, cfg.renormalize
    out = torch.empty_like(hidden)

    def step():
        if renorm:
            tv, ti = torch.topk(logits, k, dim=-1)
            gates = torch.softmax(tv, dim=-1)
        else:
            probs = torch.softmax(logits, dim=-1)
            gates, ti = torch.topk(probs, k, dim=-1)
        dense_g = torch.zeros((hidden.shape[0], E), dtype=torch.float32, device=dev).scatter_(1, ti, gates)
        acc = torch.zeros(hidden.shape, dtype=torch.float32, device=dev)
        for e in range(E):
            gu = hidden @ w13[e].T
            h = torch.nn.functional.silu(gu[:, :f]) * gu[:, f:]
            acc += (h @ w2[e].T).float() * dense_g[:, e:e + 1]
        out.copy_(acc)

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        step()
    g2.replay()
    torch.cuda.synchronize()
    ms2 = timed_steps(g2.replay, K) / K
    bytes2 = E * 3 * d * f * 2
    del w13, w2
    res["cublas"] = {"ms_per_step": ms2, "tokens_per_s": hidden.shape[0] / (ms2 / 1e3), "weight_bytes": bytes2,
                     "achieved_gbs": bytes2 / (ms2 / 1e3) / 1e9,
                     "how": "puzzle_unpack once -> dense bf16 experts; per step torch topk/softmax + every expert's "
                            "cuBLAS bf16 matmuls on all tokens weighted by the gate; CUDA-graph replay, no host sync"}
    return res


def cpu_oracle_timing(cfg, T_batch: int, budget_s: float = 12.0, max_calls: int | None = None,
                      one_core: bool = False):
    """Time the oracle (as it stands) on host cores on a bounded sample of the workload:
    `n` tokens of the same config with random packed words (timing is data-independent)."""
    import oracle
    threads = oracle.num_threads()
    rng = np.random.default_rng(0)
    P, d, f = cfg.n_pairs, cfg.d_model, cfg.d_ff
    w13 = rng.integers(0, 1 << 16, (P, 2, f, d), dtype=np.uint16)
    w2 = rng.integers(0, 1 << 16, (P, d, f), dtype=np.uint16)
    _, slot = synth.pairing(cfg)
    n = max(1, min(threads, T_batch))
    hb = synth.hidden_bits(cfg, n)
    lg = synth.router_logits(cfg, n)
    calls, t_total = 0, 0.0
    while True:
        t0 = time.perf_counter()
        oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize)
        t_total += time.perf_counter() - t0
        calls += 1
        if t_total >= budget_s or (max_calls and calls >= max_calls):
            break
    res = {"value": calls * n / t_total, "unit": "tokens/s", "cores": threads, "kind": "oracle",
           "sample": f"{calls} oracle calls x {n} tokens of {cfg.name} (d={d}, d_ff={f}, E={cfg.n_experts}, "
                     f"top-{cfg.top_k}) on random packed words; f64 accumulation, OpenMP over tokens",
           "seconds": t_total}
    if one_core and threads > 1:  # also a 1-core number (one token, one call)
        oracle.set_num_threads(1)
        try:
            t0 = time.perf_counter()
            oracle.moe_forward(w13, w2, slot, hb[:1], lg[:1], cfg.top_k, cfg.renormalize)
            res["one_core"] = {"value": 1 / (time.perf_counter() - t0), "unit": "tokens/s", "cores": 1,
                               "sample": "1 oracle call x 1 token"}
        finally:
            oracle.set_num_threads(threads)
    return res


def cpu_oracle_breakdown(budget_s: float = 2.0):
    """The oracle's other steps on the host cores: pack / unpack / merge
    elements per second (single-threaded C loops, 4 M elements) and the FFN tokens/s of every
    BASELINE config shape (OpenMP over tokens, a bounded sample each)."""
    import oracle
    rng = np.random.default_rng(1)
    n = 1 << 22
    w = np.abs(rng.standard_normal(n).astype(np.float32)) * 0.02
    planes = [rng.integers(0, 2, n, dtype=np.uint8) for _ in range(4)]
    out = {}
    t0 = time.perf_counter()
    words, _ = oracle.pack(w, *planes)
    out["pack_elems_per_s"] = n / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    oracle.unpack(words, 0)
    out["unpack_elems_per_s"] = n / (time.perf_counter() - t0)
    rows, cols = 1024, n // 1024
    wi = synth.to_bf16_values(rng.standard_normal((rows, cols)).astype(np.float32) * 0.02)
    wj = synth.to_bf16_values(rng.standard_normal((rows, cols)).astype(np.float32) * 0.02)
    ni = 1 + np.abs(rng.standard_normal(cols).astype(np.float32))
    t0 = time.perf_counter()
    oracle.merge(wi, wj, ni, ni, 0.4)
    out["merge_elems_per_s"] = n / (time.perf_counter() - t0)
    out["ffn_tokens_per_s"] = {}
    for name in ("tiny", "qwen15", "deepseek", "mixtral"):
        r = cpu_oracle_timing(synth.CONFIGS[name], 64, budget_s=budget_s, max_calls=3 if name != "tiny" else 200)
        out["ffn_tokens_per_s"][name] = {"value": r["value"], "sample": r["sample"]}
    out["cores"] = oracle.num_threads()
    out["note"] = "pack / unpack / merge: one thread (plain C loops); FFN: OpenMP over tokens"
    return out


# --------------------------------------------------------------------------- arms
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    import oracle
    oracle.build()
    threads = oracle.num_threads()
    rng = np.random.default_rng(0)
    P, d, f = cfg.n_pairs, cfg.d_model, cfg.d_ff
    w13 = rng.integers(0, 1 << 16, (P, 2, f, d), dtype=np.uint16)
    w2 = rng.integers(0, 1 << 16, (P, d, f), dtype=np.uint16)
    _, slot = synth.pairing(cfg)
    # size each step so that (warmup + steps) x step time stays within ~150 s: one token per
    # thread when that fits, else a single token per step
    hb1, lg1 = synth.hidden_bits(cfg, 1), synth.router_logits(cfg, 1)
    t_one = time.perf_counter()
    oracle.moe_forward(w13, w2, slot, hb1, lg1, cfg.top_k, cfg.renormalize)
    t_one = time.perf_counter() - t_one
    per_step = 150.0 / max(args.steps + args.warmup, 1)
    n = max(1, min(threads, args.batch)) if t_one <= per_step else 1
    hb = synth.hidden_bits(cfg, n)
    lg = synth.router_logits(cfg, n)
    step = lambda: oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    ms = dt / args.steps * 1e3
    value = n / (ms / 1e3)
    sample = (f"each step = {n} of the {args.batch} tokens of the {cfg.name} decode batch through the oracle "
              f"(plain C, f64, OpenMP over tokens), random packed words")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} single MoE layer {'decode' if args.batch <= 64 else 'prefill'}, batch {args.batch} (sampled {n} tokens/step)",
                       "d_model": d, "d_ff": f, "n_experts": cfg.n_experts, "top_k": cfg.top_k},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200 import build as pzbuild

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    # --ep1: the expert-parallel code path through a 1-rank NCCL group (tests the EP step on a
    # one-GPU box; not a multi-GPU measurement)
    dist_on = world > 1 or args.ep1
    if dist_on:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if "MASTER_PORT" not in os.environ:
                import socket
                with socket.socket() as sk:
                    sk.bind(("127.0.0.1", 0))
                    os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        import datetime
        # generous timeout: the non-zero ranks wait in barriers while rank 0 prints its line
        dist.init_process_group("nccl", device_id=device, timeout=datetime.timedelta(minutes=30))
    if rank == 0 and not os.path.exists(pz.LIB_PATH):
        pzbuild.build()
    if dist_on:
        dist.barrier()
    pz.load_library()
    pk = peaks()
    cfg = synth.CONFIGS[args.config]
    T, K, W = args.batch, args.steps, args.warmup
    seed = synth.seeds(cfg)["weights"]
    log("building layer", cfg.name)
    layer, pack_stats = build_layer_gpu(pz, cfg, seed, device, args.ratio)
    log("layer built", layer.packed_bytes)
    hidden, logits = make_inputs(cfg, T, seed + 100 * rank + 2, device)
    out = torch.empty_like(hidden)
    ws = layer.workspace(T, cfg.top_k)
    stream = torch.cuda.current_stream()
    ep = None
    if dist_on:
        # expert parallelism: this rank keeps only its pairs (or d_ff slice) of the layer
        from paper_2511_04805_b200.ep import ExpertParallelMoE, Partition, shard_dense, shard_packed
        part = Partition(layer.n_pairs, world)
        w13_l, w2_l = shard_packed(layer.w13, layer.w2, part, rank)
        local = pz.PackedMoELayer(w13_l, w2_l, torch.arange(2 * w13_l.shape[0], dtype=torch.int32, device=device),
                                  shard_dense(layer.pair_dense, part, rank))
        routing = pz.RoutingLayer(layer.n_pairs, cfg.d_model, cfg.d_ff, layer.expert_slot, w13_l)
        ep = ExpertParallelMoE(part, rank, routing, local, cfg.d_model)

    ep_fixed = ep is not None and T <= 64  # decode: static splits, no host sync, graph-capturable
    ep_capi = None  # the same fixed-capacity layer behind the C ABI (C-owned NCCL communicator)
    if ep is not None and args.ep_transport == "capi" and T <= 64:  # decode (prefill: variable splits)
        uid = [pz.ep_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ep_capi = pz.EpComm(world, rank, uid[0], device.index)
        ep_ws = ep_capi.workspace(routing, local, T, cfg.top_k)
        ep_out = torch.empty_like(hidden)
    ep_peer = None
    if ep_fixed and args.ep_transport == "peer":
        # rows / outputs stored straight into the owners' / home ranks' symmetric buffers by the
        # dispatch / return kernels (NVLink peer memory, no NCCL on the data path)
        from paper_2511_04805_b200.ep import make_peer_buffer
        try:
            ep_peer = make_peer_buffer(world, T * cfg.top_k, cfg.d_model, device)
            ep.attach_peer_buffer(ep_peer)
        except Exception as e:  # pragma: no cover
            log("peer buffer unavailable, NCCL transport:", repr(e))
            ep_peer = None

    def ep_forward(h, lg):
        if ep_capi is not None:
            return ep_capi.forward(routing, local, h, lg, cfg.top_k, cfg.renormalize, cap_tokens=T,
                                   out=ep_out if h is hidden else None, workspace=ep_ws,
                                   path=pz.PATH_GEMV if T <= 64 else pz.PATH_AUTO)
        if ep_peer is not None:
            return ep.forward_peer(h, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)
        if ep_fixed:
            return ep.forward_fixed(h, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)
        return ep.forward(h, lg, cfg.top_k, cfg.renormalize)

    def step():
        if ep is not None:
            ep_forward(hidden, logits)
        else:
            layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out, workspace=ws)

    log("workspace", ws.numel())
    n_touched = touched_pairs(layer, logits, cfg)
    log("touched pairs", n_touched)
    ab = algorithmic_bytes(cfg, n_touched, T)
    big = ab["w13"] + ab["w2"] > 4 * l2_bytes(device)
    flush = None if big else l2_flusher(device)

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    log("warmup done")
    graph = None
    if not args.no_graph and (ep is None or ep_fixed or ep_capi is not None):  # variable-split EP: eager
        # the whole forward (route .. combine) replayed as one CUDA graph: no host launch gaps
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for _ in range(W):
            graph.replay()
        torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.1)
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if graph is not None:
        total_ms = timed_steps(graph.replay, K, flush)
    else:
        with pz.profile_window() as prof:
            total_ms = timed_steps(step, K, flush)
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    t1 = time.perf_counter()
    if graph is not None:
        # per-kernel durations: the same K steps launched eagerly with library events on
        # the launching stream (graph replays carry no per-kernel events)
        with pz.profile_window() as prof:
            timed_steps(step, K, flush)
    # per-step distribution (separate pass, one event pair per step; the headline stays the
    # back-to-back average above)
    run1 = graph.replay if graph is not None else step
    ev_pairs = []
    for _ in range(min(K, 100)):
        if flush is not None:
            flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run1()
        b.record()
        ev_pairs.append((a, b))
    torch.cuda.synchronize()
    per_step = sorted(a.elapsed_time(b) for a, b in ev_pairs)
    pct = {q: per_step[min(len(per_step) - 1, int(round(q / 100 * (len(per_step) - 1))))] for q in (10, 50, 90)}
    time.sleep(0.05)
    clocks.stop()
    ms = total_ms / K
    log("timed", ms, prof.kernels)
    if dist_on:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = T * world / (ms / 1e3)

    # the peer-memory transport moves the same rows in the same order as the NCCL form, so the
    # two must agree bit for bit: a runtime self-check of the cross-rank protocol (all ranks)
    # the C-ABI and peer-memory transports move the same rows in the same order through the same
    # kernels as the torch.distributed NCCL form, so the outputs must agree bit for bit: a runtime
    # self-check of the cross-rank protocol on every rank (a mismatch aborts the run: its numbers
    # would not be of this layer)
    ep_peer_check = ep_capi_check = None
    if ep is not None and ep_fixed and (ep_peer is not None or ep_capi is not None):
        o_ref = ep.forward_fixed(hidden, logits, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)
        o_alt = ep_forward(hidden, logits).clone()
        ok = torch.tensor([1 if torch.equal(o_alt.view(torch.int16), o_ref.view(torch.int16)) else 0],
                          device=device, dtype=torch.int32)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ep_peer is not None:
            ep_peer_check = bool(ok.item()) and ep_peer.wait_timeouts() == 0
        else:
            ep_capi_check = bool(ok.item())
        if not (ep_peer_check or ep_capi_check):
            log("EP self-check FAILED: transport output differs from the torch.distributed NCCL form")
            dist.barrier()
            dist.destroy_process_group()
            return 3

    # roofline of the dominant kernel (largest share of the profiled step)
    kern = {k: {"launches": n, "total_ms": t, "avg_ms": t / max(n, 1)} for k, (n, t) in prof.kernels.items()}
    gpu_launches = sum(v["launches"] for v in kern.values())
    dom = max(kern, key=lambda k: kern[k]["total_ms"]) if kern else None
    per_launch_bytes = {"w13_gemv": ab["w13"], "w2_gemv": ab["w2"]}
    roof = None
    if dom in per_launch_bytes:
        # the projection's time includes its tail-reduce launch (the dynamic tail's partials)
        tail = dom.replace("_gemv", "_tail")
        dom_ms = kern[dom]["avg_ms"] + (kern[tail]["avg_ms"] if tail in kern else 0.0)
        achieved = per_launch_bytes[dom] / (dom_ms / 1e3) / 1e9
        traffic = ncu_traffic(cfg.name, T, dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "frac_of_nominal_8tbs": achieved / 8000.0,
                "traffic": traffic, "algorithmic_bytes_per_launch": per_launch_bytes[dom],
                "units_per_launch": n_touched, "unit_bytes": per_launch_bytes[dom] // max(n_touched, 1),
                "duration_ms": dom_ms, "duration_includes": [k for k in (dom, tail) if k in kern],
                "peak_source": pk["source"],
                "step_share": kern[dom]["total_ms"] / max(sum(v["total_ms"] for v in kern.values()), 1e-9)}
    elif dom in ("w13_tc", "w2_tc", "w13_ts", "w2_ts"):
        # prefill: tensor-bound; algorithmic flops = dense-equivalent FFN flops of the routed
        # assignments (unit: one assignment's 2*(2f)*d (w13) or 2*d*f (w2) flop)
        n_assign = T * cfg.top_k
        unit = 2 * 2 * cfg.d_ff * cfg.d_model if dom.startswith("w13") else 2 * cfg.d_model * cfg.d_ff
        achieved = unit * n_assign / (kern[dom]["avg_ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16_tflops"], "traffic": ncu_traffic(cfg.name, T, dom),
                "algorithmic_flops_per_launch": unit * n_assign, "units_per_launch": n_assign, "unit_flops": unit,
                "peak_source": pk["source"],
                "step_share": kern[dom]["total_ms"] / max(sum(v["total_ms"] for v in kern.values()), 1e-9)}
    step_gbs = (ab["w13"] + ab["w2"]) / (ms / 1e3) / 1e9

    # e2e through the public API with host buffers (pinned), copies inside the timed region.
    # Single GPU: a serving-style pipeline -- step i's inputs are copied in on a copy stream
    # while step i-1 computes, and its output is copied out on another while step i+1
    # computes (two buffer sets; every step still moves its own inputs and output across
    # PCIe inside the timed region). EP: sequential (host-side split sizes).
    h_host = [hidden.cpu().pin_memory() for _ in range(2)]
    l_host = [logits.cpu().pin_memory() for _ in range(2)]
    o_host = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
    h_dev = [torch.empty_like(hidden) for _ in range(2)]
    l_dev = [torch.empty_like(logits) for _ in range(2)]
    o_dev = [torch.empty_like(out) for _ in range(2)]
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "comp", "out")}
    e2e_graphs = [None, None]
    if ep is None and graph is not None:
        for b in range(2):
            layer.forward(h_dev[b], l_dev[b], cfg.top_k, cfg.renormalize, out=o_dev[b], workspace=ws)
            torch.cuda.synchronize()
            e2e_graphs[b] = torch.cuda.CUDAGraph()
            with torch.cuda.graph(e2e_graphs[b]):
                layer.forward(h_dev[b], l_dev[b], cfg.top_k, cfg.renormalize, out=o_dev[b], workspace=ws)
    it = [0]

    def e2e_step():
        b = it[0] & 1
        it[0] += 1
        if ep is not None:
            h_dev[0].copy_(h_host[0], non_blocking=True)
            l_dev[0].copy_(l_host[0], non_blocking=True)
            o_host[0].copy_(ep_forward(h_dev[0], l_dev[0]), non_blocking=True)
            return
        s_in.wait_event(ev["comp"][b])  # buffer set b's previous forward has read its inputs
        with torch.cuda.stream(s_in):
            h_dev[b].copy_(h_host[b], non_blocking=True)
            l_dev[b].copy_(l_host[b], non_blocking=True)
            ev["in"][b].record(s_in)
        comp.wait_event(ev["in"][b])
        comp.wait_event(ev["out"][b])  # o_dev[b] has been copied out
        if e2e_graphs[b] is not None:
            e2e_graphs[b].replay()
        else:
            layer.forward(h_dev[b], l_dev[b], cfg.top_k, cfg.renormalize, out=o_dev[b], workspace=ws)
        ev["comp"][b].record(comp)
        s_out.wait_event(ev["comp"][b])
        with torch.cuda.stream(s_out):
            o_host[b].copy_(o_dev[b], non_blocking=True)
            ev["out"][b].record(s_out)

    def e2e_drain():
        for b in range(2):
            comp.wait_event(ev["out"][b])

    for b in range(2):  # initial state: every event recorded once
        for k in ev:
            ev[k][b].record(comp)
    for _ in range(W):
        e2e_step()
    e2e_drain()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if flush is None:
        e0.record(comp)
        s_in.wait_event(e0)  # the first copy-in starts after e0
        for _ in range(K):
            e2e_step()
        e2e_drain()  # the last outputs are on the host
        e1.record(comp)
        e1.synchronize()
        e2e_ms = e0.elapsed_time(e1) / K
    else:  # small layers: L2 flushed between steps, each step timed alone (no overlap)
        tot = 0.0
        for _ in range(K):
            flush()
            e0.record(comp)
            s_in.wait_event(e0)
            e2e_step()
            e2e_drain()
            e1.record(comp)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        e2e_ms = tot / K
    o_ok = bool(torch.equal(o_host[0].view(torch.int16), out.cpu().view(torch.int16))) if ep is None else None
    if dist_on:
        t = torch.tensor([e2e_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    log("e2e", e2e_ms)
    e2e = {"value": T * world / (e2e_ms / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": h_host[0].numel() * 2 + l_host[0].numel() * 4,
           "d2h_bytes_per_step": o_host[0].numel() * 2, "ms_per_step": e2e_ms,
           "api": (("EpComm.forward -> puzzle_moe_forward_ep" if ep_capi is not None else
                    "ExpertParallelMoE." + ("forward_peer" if ep_peer is not None else "forward_fixed" if ep_fixed
                                            else "forward")) if ep is not None
                   else "PackedMoELayer.forward -> puzzle_moe_forward_ex") + " (host pinned buffers)",
           "pipelined": ep is None and flush is None,
           "note": "copy-in of step i+1 and copy-out of step i-1 overlap step i's forward (two buffer sets, "
                   "separate copy streams)" if ep is None and flush is None else "sequential copies",
           "output_matches_device_run": o_ok}

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded N(0,1/in) experts merged+packed on GPU, tau=0.4; N(0,1) hidden and logits)",
            "config": {"workload": f"{cfg.name} single MoE layer {'decode' if T <= 64 else 'prefill'}, batch {T} per GPU"
                                   + (" (25% ratio: merged pairs + dense bf16 slots)" if args.ratio == 0.25 else "")
                                   + (" (BASELINE.json configs[1])" if cfg.name == "mixtral" and T <= 64 else (" (BASELINE.json configs[2])" if cfg.name == "mixtral" else "")),
                       "d_model": cfg.d_model, "d_ff": cfg.d_ff, "n_experts": cfg.n_experts,
                       "n_pairs": cfg.n_pairs, "top_k": cfg.top_k, "batch_per_gpu": T,
                       "parallelism": f"ep{world} (pairs sharded, NCCL all-to-all dispatch/combine, "
                                      f"{T} tokens per rank, "
                                      + ("fixed-capacity dispatch, C-ABI NCCL communicator)" if ep_capi is not None
                                         else "fixed-capacity dispatch over NVLink peer memory)" if ep_peer is not None
                                         else "fixed-capacity dispatch, NCCL)" if ep_fixed
                                         else "variable-split dispatch, NCCL)")
                                      if dist_on else "single",
                       "l2": "inputs larger than L2 (packed layer %.2f GB)" % (layer.packed_bytes / 1e9) if big
                       else "L2 flushed between timed steps (2x L2 written, then 2x L2 read: clean lines)",
                       "launch": "CUDA graph replay of the whole forward" if graph is not None else "eager"},
            "roofline": roof, "step_weight_gbs": step_gbs, "gpu_launches": gpu_launches,
            **({"ep_peer_wait_timeouts": ep_peer.wait_timeouts(), "ep_peer_matches_nccl": ep_peer_check}
               if ep_peer is not None else {}),
            **({"ep_capi_matches_torch_nccl": ep_capi_check} if ep_capi is not None else {}),
            "step_ms_percentiles": {"p10": pct[10], "p50": pct[50], "p90": pct[90], "steps": len(per_step),
                                    "note": "one event pair per step, separate pass (rank-local)"},
            "kernels": kern, "e2e": e2e}
    if ep is not None and ep_fixed and not args.no_extra:
        # strong scaling (global decode batch fixed, split over the ranks)
        line.setdefault("aux", {})["strong_scaling"] = ep_strong_scaling(
            pz, args, cfg, device, rank, world, routing, local, ep, ep_capi, global_batch=args.batch)
    if dist_on and ((world > 1 and not args.no_extra) or args.stack_ep):
        stack_ep = stack_runs_ep(pz, args, device, part, rank, world, ep_capi)
        line.setdefault("aux", {})["stack32_ep"] = stack_ep
    if rank == 0:
        line["clocks"] = clocks.summary(t0, t1)
        line["aux"] = dict(line.get("aux", {}),
                           pack_stats=dict(zip(["rounded_up", "saturated", "nonfinite", "negative"], pack_stats)),
                           touched_pairs=n_touched)
        if not args.no_extra and not dist_on:  # single-GPU extras (the N = 1 run carries them)
            line["aux"]["host_call"] = host_call_cost(layer, cfg, hidden, logits, out, ws)
            try:
                line["aux"]["quant_forward"] = quant_forward_rates(pz, device, pk)
            except Exception as e:  # pragma: no cover
                line["aux"]["quant_forward"] = {"error": repr(e)}
            try:
                ub = unpacked_baseline(pz, layer, cfg, hidden, logits, min(K, 50), W)
                for arm in ("same_kernels", "cublas"):
                    ub[arm]["packed_speedup"] = ub[arm]["ms_per_step"] / ms
                line["aux"]["unpacked_bf16_baseline"] = ub
            except Exception as e:  # pragma: no cover
                line["aux"]["unpacked_bf16_baseline"] = {"error": repr(e)}
            line["aux"]["packer"] = packer_rates(pz, layer, device)
            line["aux"]["sweep"] = sweep(pz, args, device, pk)
            try:
                line["aux"]["calib"] = calib_run(pz, args, device, pk)
            except Exception as e:  # pragma: no cover
                line["aux"]["calib"] = {"error": repr(e)}
            try:
                del layer
                torch.cuda.empty_cache()
                line["aux"]["stack32"] = stack_runs(pz, args, device, pk)
            except Exception as e:  # pragma: no cover
                line["aux"]["stack32"] = {"error": repr(e)}
        if world == 1 and not args.no_cpu:
            try:
                line["cpu_baseline"] = cpu_oracle_timing(cfg, T, one_core=True)
                if not args.no_extra:
                    line["cpu_baseline"]["breakdown"] = cpu_oracle_breakdown()
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"error": repr(e)}
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def ncu_traffic(cfg_name: str, T: int, kernel: str):
    """dram bytes per launch from the committed ncu --set full capture, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        tab = json.load(fh)
    return tab.get(f"{cfg_name}/T{T}/{kernel}")


def quant_forward_rates(pz, device, pk, cases=(("mixtral", 64), ("mixtral", 1), ("qwen15", 64), ("deepseek", 64))):
    """NEXT-3: puzzle_moe_forward_quant (the quantised weight class through the decode-shape
    tcgen05 kernels) on full-size layers with seeded random code bytes (flags + 3-bit codes, bit 3
    zero) and group scales (timing is data-independent; parity: tests/test_gpu_quant_forward.py).
    Algorithmic bytes = the touched pairs' code bytes + scales (8.25 bits per merged element)."""
    import torch
    res = []
    g = torch.Generator(device=device)
    g.manual_seed(2511)
    for name, T in cases:
        cfg = synth.CONFIGS[name]
        P, d, f = cfg.n_pairs, cfg.d_model, cfg.d_ff
        rnd = lambda *shape: (torch.randint(0, 256, shape, generator=g, device=device, dtype=torch.int32) & 0xF7).to(torch.uint8)
        c13, c2 = rnd(P, 2, f, d), rnd(P, d, f)
        s13 = torch.rand((P, 2, f, d // 128), generator=g, device=device) * 0.01 + 1e-3
        s2 = torch.rand((P, d, f // 128), generator=g, device=device) * 0.01 + 1e-3
        _, slot = synth.pairing(cfg)
        layer = pz.QuantMoELayer(c13, s13, c2, s2, torch.from_numpy(slot).to(device))
        hidden, logits = make_inputs(cfg, T, synth.seeds(cfg)["activations"], device)
        out = torch.empty_like(hidden)
        ws = layer.workspace(T, cfg.top_k)
        fwd = lambda: layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
        fwd()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fwd()
        for _ in range(5):
            gr.replay()
        torch.cuda.synchronize()
        K = 50
        ms = timed_steps(gr.replay, K) / K
        with pz.profile_window() as prof:
            timed_steps(fwd, 20)
        kern = {k: round(t / n * 1e3, 2) for k, (n, t) in prof.kernels.items()}
        top = torch.topk(logits, cfg.top_k, dim=-1).indices.reshape(-1).cpu().numpy()
        nt = len(set(int(slot[e]) // 2 for e in top))
        per_pair = 3 * d * f + (2 * f * d // 128 + d * f // 128) * 4
        gbs = nt * per_pair / (ms / 1e3) / 1e9
        res.append({"config": name, "batch": T, "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3),
                    "touched_pairs": nt, "quant_bytes_per_pair": per_pair, "weight_gbs": gbs,
                    "frac_hbm": gbs / pk["hbm_gbs"], "kernel_avg_us": kern,
                    "bits_per_merged_element": 8 + 32 / 128})
        del layer, c13, c2, s13, s2
        torch.cuda.empty_cache()
    return res


def host_call_cost(layer, cfg, hidden, logits, out, ws, n: int = 50):
    """The un-captured C-ABI call: host time to enqueue one puzzle_moe_forward (argument checks,
    plan, tensor-map encodes, kernel launches; no synchronisation) and the device time per step
    of back-to-back eager calls (launch gaps included), next to the CUDA-graph replay headline."""
    import torch
    fwd = lambda: layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
    for _ in range(5):
        fwd()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fwd()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    eager_ms = timed_steps(fwd, n) / n
    return {"host_us_per_call": (t1 - t0) / n * 1e6, "eager_device_ms_per_step": eager_ms, "calls": n,
            "api": "PackedMoELayer.forward -> puzzle_moe_forward_ex (eager, no graph)"}


def ep_strong_scaling(pz, args, cfg, device, rank, world, routing, local, ep, ep_capi, global_batch: int):
    """The expert-parallel decode layer with the GLOBAL batch fixed (global_batch tokens split
    evenly over the ranks, at least 1 each): tokens/s = global_batch / max-over-ranks step time.
    Same transport as the headline (C-ABI communicator, or the torch.distributed NCCL form)."""
    import torch
    import torch.distributed as dist
    T_l = max(1, global_batch // world)
    seed = synth.seeds(cfg)["weights"]
    h, lg = make_inputs(cfg, T_l, seed + 100 * rank + 7, device)
    if ep_capi is not None:
        ws = ep_capi.workspace(routing, local, T_l, cfg.top_k)
        out = torch.empty_like(h)
        fwd = lambda: ep_capi.forward(routing, local, h, lg, cfg.top_k, cfg.renormalize, cap_tokens=T_l, out=out,
                                      workspace=ws, path=pz.PATH_GEMV)
    else:
        fwd = lambda: ep.forward_fixed(h, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)
    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fwd()
    for _ in range(max(3, args.warmup)):
        g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    K = max(10, min(args.steps, 100))
    ms = timed_steps(g.replay, K) / K
    t = torch.tensor([ms], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"scaling": "strong", "global_batch": T_l * world, "tokens_per_rank": T_l, "ms_per_step": ms,
            "value": T_l * world / (ms / 1e3), "unit": "tokens/s",
            "transport": "C-ABI NCCL communicator" if ep_capi is not None else "torch.distributed NCCL",
            "launch": "CUDA graph replay", "timing": "CUDA events, max over ranks"}


def packer_rates(pz, layer, device):
    import torch
    n = layer.w13.numel()
    src = layer.w13.reshape(-1)
    out = torch.empty(n, dtype=torch.bfloat16, device=device)
    for _ in range(2):
        pz.unpack(src, 0, out=out)
    torch.cuda.synchronize()
    ms = timed_steps(lambda: pz.unpack(src, 0, out=out), 5) / 5
    unpack_gbs = n * 4 / (ms / 1e3) / 1e9
    m = 1 << 28
    w = torch.rand(m, device=device)
    planes = [torch.randint(0, 2, (m,), dtype=torch.uint8, device=device) for _ in range(4)]
    po = torch.empty(m, dtype=torch.int16, device=device)
    pz.merge_pack(w, *planes, out=po)
    torch.cuda.synchronize()
    ms2 = timed_steps(lambda: pz.merge_pack(w, *planes, out=po), 5) / 5
    # NEXT-3 quantised packer pair on the same 2^28 elements as [2^15, 2^13] matrices
    w2d, pl2d = w.view(1 << 15, 1 << 13), [p.view(1 << 15, 1 << 13) for p in planes]
    codes, scales = pz.quant_pack(w2d, *pl2d)
    deq = pz.quant_unpack(codes, scales, 0)
    torch.cuda.synchronize()
    ms3 = timed_steps(lambda: pz.quant_pack(w2d, *pl2d), 5) / 5
    ms4 = timed_steps(lambda: pz.quant_unpack(codes, scales, 0), 5) / 5
    del deq
    qg = quant_gemv_rates(pz, w, planes, device)
    # NEXT-1 fused merge + pack (Eq. 1-7): a Mixtral w1 slot, 4 pairs x [14336, 4096] bf16 experts
    wi = (torch.randn(4, 14336, 4096, device=device) * 0.0156).to(torch.bfloat16)
    wj = (torch.randn(4, 14336, 4096, device=device) * 0.0156).to(torch.bfloat16)
    ni = 1 + torch.randn(4, 4096, device=device).abs()
    nj = 1 + torch.randn(4, 4096, device=device).abs()
    mo = pz.merge_experts_pack(wi, wj, ni, nj, 0.4)
    torch.cuda.synchronize()
    ms5 = timed_steps(lambda: pz.merge_experts_pack(wi, wj, ni, nj, 0.4, out=mo), 5) / 5
    me = wi.numel()
    del wi, wj, mo
    pk = peaks()
    return {"quant_gemv": qg, "unpack_gbs": unpack_gbs, "unpack_elems": n, "pack_gbs": m * 10 / (ms2 / 1e3) / 1e9, "pack_elems": m,
            "merge_gbs": me * 6 / (ms5 / 1e3) / 1e9, "merge_frac_hbm": me * 6 / (ms5 / 1e3) / 1e9 / pk["hbm_gbs"],
            "merge_elems": me, "merge_ms": ms5,
            "quant_pack_gbs": m * (9 + 4 / 128) / (ms3 / 1e3) / 1e9,
            "quant_unpack_gbs": m * (3 + 4 / 128) / (ms4 / 1e3) / 1e9,
            "note": "algorithmic bytes: unpack 4 B/elem, pack 10 B/elem, merge+pack 6 B/elem (W_i, W_j in, word out; norms per column), quant pack 9 B/elem (+ scales), "
                    "quant unpack 3 B/elem (+ scales); quant timings include the output allocation"}


def quant_gemv_rates(pz, w, planes, device):
    """NEXT-3 expert GEMV over the quantised format (puzzle_quant_gemv) on Mixtral w13-shaped
    merged pairs ([2 d_ff, d] = [28672, 4096] codes), 4 pairs cycled per launch round so the
    470 MB of codes exceed L2; tokens per expert n_i = n_j in {1, 8, 16}. Algorithmic bytes per
    pair: codes 1 B/elem + scales 4 B/128 elem + the token rows in and outputs out."""
    import torch
    rows, cols = 28672, 4096
    e = rows * cols
    pairs = [pz.quant_pack(w[k * e:(k + 1) * e].view(rows, cols), *[p[k * e:(k + 1) * e].view(rows, cols)
                           for p in planes]) for k in range(2)]
    pairs = pairs + [(c.clone(), s.clone()) for c, s in pairs]  # 4 distinct buffers (2^28 elements hold 2 pairs)
    out = []
    for n in (1, 8, 16):
        xi = torch.randn(n, cols, device=device).to(torch.bfloat16)
        xj = torch.randn(n, cols, device=device).to(torch.bfloat16)
        for c, s in pairs:
            pz.quant_gemv(c, s, xi, xj)
        torch.cuda.synchronize()
        reps = 10
        ms = timed_steps(lambda: [pz.quant_gemv(c, s, xi, xj) for c, s in pairs], reps) / (reps * len(pairs))
        nbytes = e * (1 + 4 / 128) + 2 * n * cols * 2 + 2 * n * rows * 4
        out.append({"tokens_per_expert": n, "us_per_pair": ms * 1e3, "gbs": nbytes / (ms / 1e3) / 1e9,
                    "bytes_per_pair": nbytes})
    return {"shape": [rows, cols], "pairs_cycled": len(pairs), "points": out,
            "note": "CUDA-core GEMV (k_quant_gemv); timings include the output allocation"}


def sweep(pz, args, device, pk):
    """Secondary configs: decode batches of BASELINE.json configs[1] and configs[3] shapes
    (HBM-bound, GB/s of packed weights), and prefill of configs[2] / configs[3] on the tcgen05
    path (tensor-bound, TFLOP/s of the dense-equivalent 2*3*d*f*T*k)."""
    import torch
    res = []
    layers = {}
    for name, T, ratio in (("mixtral", 1, 0.5), ("mixtral", 16, 0.5), ("mixtral", 128, 0.5), ("mixtral", 256, 0.5),
                           ("mixtral", 384, 0.5), ("mixtral", 512, 0.5), ("mixtral", 1024, 0.5), ("mixtral", 4096, 0.5),
                           ("qwen15", 1, 0.5), ("qwen15", 16, 0.5), ("qwen15", 64, 0.5), ("qwen15", 128, 0.5),
                           ("qwen15", 256, 0.5), ("qwen15", 512, 0.5), ("qwen15", 1024, 0.5), ("qwen15", 4096, 0.5),
                           ("deepseek", 1, 0.5), ("deepseek", 16, 0.5), ("deepseek", 64, 0.5), ("deepseek", 512, 0.5), ("deepseek", 1024, 0.5),
                           ("deepseek", 4096, 0.5),
                           ("mixtral", 64, 0.25), ("mixtral", 4096, 0.25), ("deepseek", 64, 0.25)):
        cfg = synth.CONFIGS[name]
        try:
            if (name, ratio) not in layers:
                layers.clear()
                torch.cuda.empty_cache()
                layers[(name, ratio)] = build_layer_gpu(pz, cfg, synth.seeds(cfg)["weights"], device, ratio)[0]
            layer = layers[(name, ratio)]
            hidden, logits = make_inputs(cfg, T, synth.seeds(cfg)["activations"], device)
            out = torch.empty_like(hidden)
            ws = layer.workspace(T, cfg.top_k)
            eager = lambda: layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
            eager()
            torch.cuda.synchronize()
            if args.no_graph:
                step = eager
            else:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    eager()
                step = g.replay
            nt = touched_pairs(layer, logits, cfg)
            ab = algorithmic_bytes(cfg, nt, T)
            flush = l2_flusher(device)
            for _ in range(5):
                step()
            torch.cuda.synchronize()
            K = 50 if T <= 64 else 20
            ms = timed_steps(step, K, flush) / K
            with pz.profile_window() as prof:
                timed_steps(eager, K, flush)
            kern = {k: round(t / n, 5) for k, (n, t) in prof.kernels.items()}
            gbs = (ab["w13"] + ab["w2"]) / (ms / 1e3) / 1e9
            row = {"config": name, "batch": T, "tokens_per_s": T / (ms / 1e3), "ms_per_step": ms,
                   "touched_pairs": nt, "kernel_avg_ms": kern}
            if ratio != 0.5:
                row.update({"compression": "25% (merged pairs + dense bf16 slots, R20)",
                            "slots": layer.n_pairs, "packed_gb": layer.packed_bytes / 1e9})
            if T <= 64:
                row.update({"weight_gbs": gbs, "frac_hbm": gbs / pk["hbm_gbs"]})
            else:
                row.update({"weight_gbs_step": gbs, "frac_hbm_step": gbs / pk["hbm_gbs"]})
                flops = 2 * 3 * cfg.d_model * cfg.d_ff * T * cfg.top_k
                tc_ms = sum(v for k, v in kern.items() if k.endswith("_tc") or k.endswith("_ts"))
                row.update({"path": "ts" if any(k.endswith("_ts") for k in kern) else
                                    "gemv" if any(k.endswith("_gemv") for k in kern) else "tc", "tflops_step": flops / (ms / 1e3) / 1e12,
                            "tflops_tc_kernels": flops / (tc_ms / 1e3) / 1e12 if tc_ms else None,
                            "frac_bf16_peak": flops / (tc_ms / 1e3) / 1e12 / pk["bf16_tflops"] if tc_ms else None})
            res.append(row)
            del flush
        except Exception as e:  # pragma: no cover
            res.append({"config": name, "batch": T, "ratio": ratio, "error": repr(e)})
    return res


def calib_run(pz, args, device, pk, T: int = 4096):
    """NEXT-4: one calibration batch (T tokens) through the UNMERGED Mixtral layer (8 dense bf16
    slots) with puzzle_moe_forward_calib: the forward plus the Eq. 4 column statistics of x and
    h per expert. The statistics kernel is HBM-bound: it reads the bucket-ordered x and h rows
    once (n_assign * (d + f) * 2 B per step, over its two launches)."""
    import torch
    cfg = synth.CONFIGS["mixtral"]
    layer, _ = build_layer_gpu(pz, cfg, synth.seeds(cfg)["weights"], device, ratio=1.0)
    hidden, logits = make_inputs(cfg, T, synth.seeds(cfg)["activations"], device)
    sx = torch.zeros((2 * layer.n_pairs, cfg.d_model), dtype=torch.float64, device=device)
    sh = torch.zeros((2 * layer.n_pairs, cfg.d_ff), dtype=torch.float64, device=device)
    step = lambda: layer.forward_calib(hidden, logits, cfg.top_k, cfg.renormalize, sx, sh)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    K = 10
    flush = l2_flusher(device)
    ms = timed_steps(step, K, flush) / K
    with pz.profile_window() as prof:
        timed_steps(step, K, flush)
    n_launch, total = prof.kernels.get("calib_colsumsq", (0, 0.0))
    kern = {k: round(t / n, 5) for k, (n, t) in prof.kernels.items()}
    n_assign = T * cfg.top_k
    stat_bytes = n_assign * (cfg.d_model + cfg.d_ff) * 2
    stat_ms = total / K if n_launch else 0.0  # both launches (x rows, h rows) of one step
    gbs = stat_bytes / (stat_ms / 1e3) / 1e9 if stat_ms else None
    out = {"config": "mixtral unmerged (8 dense slots)", "batch": T, "ms_per_step": ms,
           "tokens_per_s": T / (ms / 1e3), "kernel_avg_ms": kern, "stat_bytes_per_step": stat_bytes,
           "stat_gbs": gbs, "stat_frac_hbm": gbs / pk["hbm_gbs"] if gbs else None,
           "norms_finite": bool(torch.isfinite(sx).all().item() and torch.isfinite(sh).all().item())}
    del layer, flush
    torch.cuda.empty_cache()
    return out


def stack_runs(pz, args, device, pk):
    """BASELINE.json configs[4] on one B200: the 32-layer Mixtral-8x7B MoE stack at 50%
    compression (45.1 GB packed), x_{l+1} = x_l + MoE_l(x_l) with fixed per-layer router
    logits, batch-64 decode (graph replay) and 8192-token prefill."""
    import torch
    cfg = synth.CONFIGS["mixtral"]
    n_layers = 32
    layers = []
    for l in range(n_layers):
        layer, _ = build_layer_gpu(pz, cfg, 90000 + l, device)
        layers.append(layer)
    res = []
    for T in (64, 8192):
        g = torch.Generator(device=device)
        g.manual_seed(777 + T)
        x0 = torch.randn((T, cfg.d_model), generator=g, device=device).to(torch.bfloat16)
        logits = [torch.randn((T, cfg.n_experts), generator=g, device=device) for _ in range(n_layers)]
        bufs = [torch.empty_like(x0), torch.empty_like(x0)]
        ws = [layer.workspace(T, cfg.top_k) for layer in layers[:1]][0]
        need = max(layer.workspace_size(T, cfg.top_k) for layer in layers)
        if ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=device)

        def step():
            x = x0
            for l, layer in enumerate(layers):
                out = bufs[l % 2]
                layer.forward(x, logits[l], cfg.top_k, cfg.renormalize, residual=x, out=out, workspace=ws)
                x = out
            return x

        step()
        torch.cuda.synchronize()
        run = step
        if T <= 64 and not args.no_graph:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step()
            run = gr.replay
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        K = 20 if T <= 64 else 5
        ms = timed_steps(run, K) / K
        row = {"config": "mixtral_stack32", "batch": T, "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3),
               "layers": n_layers, "packed_gb": sum(l.packed_bytes for l in layers) / 1e9}
        if T <= 64:
            row["weight_gbs"] = row["packed_gb"] * 1e9 / (ms / 1e3) / 1e9  # upper bound: all pairs touched at B=64
        else:
            fl = 2 * 3 * cfg.d_model * cfg.d_ff * T * cfg.top_k * n_layers
            row["tflops_step"] = fl / (ms / 1e3) / 1e12
        res.append(row)
    del layers
    torch.cuda.empty_cache()
    return res


def stack_runs_ep(pz, args, device, part, rank, world, ep_capi=None):
    """BASELINE.json configs[4] as named: the 32-layer Mixtral-8x7B MoE stack at 50%
    compression, EXPERT-PARALLEL -- every rank holds its share of each layer's merged pairs and
    its own tokens (weak scaling), x_{l+1} = x_l + MoE_l(x_l). Batch-64 decode runs the
    fixed-capacity dispatch (device-only) replayed as one CUDA graph of all 32 layers; the
    8192-token prefill runs the variable-split dispatch eagerly. Time = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2511_04805_b200.ep import ExpertParallelMoE, shard_dense, shard_packed
    cfg = synth.CONFIGS["mixtral"]
    n_layers = 32
    eps = []
    for l in range(n_layers):
        layer, _ = build_layer_gpu(pz, cfg, 90000 + l, device)
        w13_l, w2_l = shard_packed(layer.w13, layer.w2, part, rank)
        local = pz.PackedMoELayer(w13_l, w2_l, torch.arange(2 * w13_l.shape[0], dtype=torch.int32, device=device),
                                  shard_dense(layer.pair_dense, part, rank))
        routing = pz.RoutingLayer(layer.n_pairs, cfg.d_model, cfg.d_ff, layer.expert_slot.clone(), w13_l)
        eps.append(ExpertParallelMoE(part, rank, routing, local, cfg.d_model))
        del layer
    torch.cuda.empty_cache()
    pb = None
    if args.ep_transport == "peer":  # one peer buffer serves every layer (calls are sequential)
        from paper_2511_04805_b200.ep import make_peer_buffer
        try:
            pb = make_peer_buffer(world, 64 * cfg.top_k, cfg.d_model, device)
            for ep in eps:
                ep.attach_peer_buffer(pb)
        except Exception as e:  # pragma: no cover
            log("peer buffer unavailable, NCCL transport:", repr(e))
            pb = None
    res = []
    for T in (64, 8192):
        g = torch.Generator(device=device)
        g.manual_seed(777 + T + 1000 * rank)
        x0 = torch.randn((T, cfg.d_model), generator=g, device=device).to(torch.bfloat16)
        logits = [torch.randn((T, cfg.n_experts), generator=g, device=device) for _ in range(n_layers)]
        fixed = T <= 64

        ws_c = None
        if fixed and ep_capi is not None:  # one communicator and workspace serve every layer
            ws_c = ep_capi.workspace(eps[0].route_layer, eps[0].local_layer, T, cfg.top_k)

        def step():
            x = x0
            for l, ep in enumerate(eps):
                if fixed and ws_c is not None:
                    x = ep_capi.forward(ep.route_layer, ep.local_layer, x, logits[l], cfg.top_k, cfg.renormalize,
                                        cap_tokens=T, residual=x, workspace=ws_c, path=pz.PATH_GEMV)
                elif fixed and pb is not None:
                    x = ep.forward_peer(x, logits[l], cfg.top_k, cfg.renormalize, residual=x, path=pz.PATH_GEMV)
                elif fixed:
                    x = ep.forward_fixed(x, logits[l], cfg.top_k, cfg.renormalize, residual=x, path=pz.PATH_GEMV)
                else:
                    x = ep.forward(x, logits[l], cfg.top_k, cfg.renormalize, residual=x)
            return x

        step()
        torch.cuda.synchronize()
        run = step
        if fixed and not args.no_graph:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step()
            run = gr.replay
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        dist.barrier()
        K = 20 if fixed else 5
        ms = timed_steps(run, K) / K
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        row = {"config": f"mixtral_stack32_ep{world}", "batch_per_rank": T, "ms_per_step": ms,
               "tokens_per_s": T * world / (ms / 1e3), "layers": n_layers,
               "dispatch": (("fixed-capacity, C-ABI NCCL communicator" if ws_c is not None else
                             "fixed-capacity over NVLink peer memory" if pb is not None else "fixed-capacity, NCCL")
                            + (", one CUDA graph of 32 layers" if not args.no_graph else ", eager")
                            if fixed else "variable-split, NCCL, eager")}
        if fixed and pb is not None:
            row["peer_wait_timeouts"] = pb.wait_timeouts()
        if not fixed:
            row["tflops_per_rank"] = 2 * 3 * cfg.d_model * cfg.d_ff * T * cfg.top_k * n_layers / (ms / 1e3) / 1e12
        res.append(row)
    del eps
    torch.cuda.empty_cache()
    return res


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(synth.CONFIGS), default="mixtral")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ratio", type=float, choices=[0.5, 0.25], default=0.5,
                    help="compression ratio of the timed layer: 0.5 (all pairs merged, the headline) or "
                         "0.25 (merged pairs + dense bf16 slots, R20)")
    ap.add_argument("--no-extra", action="store_true", help="skip the unpacked baseline / sweep / packer lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle timing")
    ap.add_argument("--ep1", action="store_true", help="run the expert-parallel path in a 1-rank NCCL group")
    ap.add_argument("--ep-transport", choices=["capi", "peer", "nccl"], default="capi",
                    help="EP decode transport: kernels storing into peer memory, or NCCL all-to-all")
    ap.add_argument("--stack-ep", action="store_true", help="with --ep1: also the expert-parallel 32-layer stack")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replays")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
