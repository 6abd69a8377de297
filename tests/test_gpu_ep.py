"""Expert-parallel path on the GPU through the real kernels and a 1-rank NCCL group (the pod
exposes one GPU; multi-rank host logic is covered by tests/test_ep_gloo.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
import synth
from helpers import assert_close, oracle_mixed_layer, oracle_packed_layer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [synth.MoEConfig("ep_small", 30, 256, 512, 8, 2, True),
                                 synth.MoEConfig("ep_fine", 31, 128, 256, 16, 4, False)], ids=lambda c: c.name)
def test_ep_world1_matches_forward_and_oracle(nccl_group, cfg):
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200.ep import ExpertParallelMoE, Partition, shard_packed
    w13, w2, slot, _ = oracle_packed_layer(cfg)
    w13_d = torch.from_numpy(w13.view(np.int16)).cuda()
    w2_d = torch.from_numpy(w2.view(np.int16)).cuda()
    slot_d = torch.from_numpy(slot).cuda()
    full = pz.PackedMoELayer(w13_d, w2_d, slot_d)
    part = Partition(cfg.n_pairs, 1)
    w13_l, w2_l = shard_packed(w13_d, w2_d, part, 0)
    local = pz.PackedMoELayer(w13_l, w2_l, torch.arange(2 * w13_l.shape[0], dtype=torch.int32, device="cuda"))
    route = pz.RoutingLayer(cfg.n_pairs, cfg.d_model, cfg.d_ff, slot_d, w13_l)
    ep = ExpertParallelMoE(part, 0, route, local, cfg.d_model)
    T = 37
    hb = synth.hidden_bits(cfg, T)
    lg = synth.router_logits(cfg, T)
    h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    l = torch.from_numpy(lg).cuda()
    out = ep.forward(h, l, cfg.top_k, cfg.renormalize)
    ref_fwd = full.forward(h, l, cfg.top_k, cfg.renormalize)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize)
    assert_close(out.float().cpu().numpy(), ref, "ep vs oracle")
    assert (out.float() - ref_fwd.float()).abs().max().item() <= 2e-2


# ---- fixed-capacity dispatch: the three index kernels against their header definitions ----

def _partitions():
    from paper_2511_04805_b200.ep import Partition
    for P, G in [(4, 1), (4, 3), (30, 8), (32, 4), (4, 8), (2, 4), (1, 2)]:
        part = Partition(P, G)
        yield P, G, part.slices, np.array([part.pairs_of(q) for q in range(G)], np.int32)


def _random_routing(rng, P, T, k):
    """bucket_off / assign_token / assign_of / gate of a random top-k routing (bucket-major)."""
    E = 2 * P
    idx = np.stack([rng.choice(E, size=min(k, E), replace=False) for _ in range(T)]) if T else np.zeros((0, k), np.int64)
    b = idx.reshape(-1)
    order = np.argsort(b, kind="stable")
    off = np.concatenate([[0], np.cumsum(np.bincount(b, minlength=E))]).astype(np.int32)
    tok = (order // k).astype(np.int32)
    aof = np.empty(T * k, np.int32)
    aof[order] = np.arange(T * k, dtype=np.int32)
    gate = rng.random((T, k)).astype(np.float32)
    return off, tok, aof, gate


@pytest.mark.parametrize("T,k,spare", [(1, 1, 0), (13, 2, 3), (64, 2, 0), (37, 6, 1), (0, 2, 2)])
def test_ep_dispatch_and_home_index_match_definition(T, k, spare):
    import paper_2511_04805_b200 as pz
    from helpers import ep_dispatch_ref, ep_home_index_ref
    rng = np.random.default_rng(1000 + T * 7 + k)
    d = 64
    for P, G, S, dest in _partitions():
        if k > 2 * P:
            continue
        off, tok, aof, gate = _random_routing(rng, P, T, k)
        cap = (T + spare) * k
        lb_max = int(2 * max(b - a for a, b in dest))
        hidden = rng.integers(-2**15, 2**15, size=(max(T, 1), d), dtype=np.int16)
        h_d = torch.from_numpy(hidden).cuda()
        tok_d, off_d = torch.from_numpy(tok).cuda(), torch.from_numpy(off).cuda()
        rows = torch.zeros((G * (cap + 1), d), dtype=torch.int16, device="cuda")
        rows = pz.ep_dispatch(h_d, tok_d, off_d, P, dest, cap, lb_max, send_rows=rows)
        r_ref = ep_dispatch_ref(hidden, tok, off, dest, cap, lb_max)
        assert np.array_equal(rows.cpu().numpy(), r_ref), (P, G)  # rows and header counts
        aof_s, gate_s = pz.ep_home_index(torch.from_numpy(aof).cuda(), torch.from_numpy(gate).cuda(), off_d, P, dest,
                                         S, cap)
        a_ref, g_ref = ep_home_index_ref(aof, gate, off, dest, S, cap)
        assert np.array_equal(aof_s.cpu().numpy(), a_ref), (P, G)
        assert np.array_equal(gate_s.cpu().numpy(), g_ref), (P, G)


@pytest.mark.parametrize("G,lb,cap,d", [(1, 8, 128, 64), (2, 4, 10, 64), (8, 2, 384, 64), (4, 60, 2048, 128),
                                        (3, 5, 0, 64), (8, 16, 64, 64), (2, 1024, 40, 2048)])
def test_ep_recv_plan_matches_definition(G, lb, cap, d):
    import paper_2511_04805_b200 as pz
    from helpers import ep_recv_plan_ref
    rng = np.random.default_rng(G * 100 + lb)
    R = cap + 1
    rows = rng.integers(-2**15, 2**15, size=(G * R, d), dtype=np.int16)  # payload is irrelevant
    for s in range(G):  # each source sends at most cap rows, some buckets empty
        n = int(rng.integers(0, cap + 1)) if cap else 0
        rc = np.zeros(lb, np.int32)
        if lb and n:
            cut = np.sort(rng.integers(0, n + 1, size=lb - 1))
            rc = np.diff(np.concatenate([[0], cut, [n]])).astype(np.int32)
        rows[s * R + cap, :2 * lb] = rc.view(np.int16)
    lo, gi, ri = pz.ep_recv_plan(torch.from_numpy(rows).cuda(), G, lb, cap)
    lo_r, gi_r, ri_r = ep_recv_plan_ref(rows, G, lb, cap)
    assert np.array_equal(lo.cpu().numpy(), lo_r)
    assert np.array_equal(gi.cpu().numpy(), gi_r)
    assert np.array_equal(ri.cpu().numpy(), ri_r)


def test_ep_fixed_argument_errors():
    import paper_2511_04805_b200 as pz
    h = torch.zeros((4, 64), dtype=torch.int16, device="cuda")
    tok = torch.zeros(8, dtype=torch.int32, device="cuda")
    off = torch.zeros(9, dtype=torch.int32, device="cuda")
    with pytest.raises(pz.PuzzleError):  # cap < T*k
        pz.ep_dispatch(h, tok, off, 4, [[0, 4]], 7, 8)
    with pytest.raises(pz.PuzzleError):  # pair range outside [0, n_pairs]
        pz.ep_dispatch(h, tok, off, 4, [[0, 5]], 8, 10)
    with pytest.raises(pz.PuzzleError):  # lb_max below a rank's local buckets
        pz.ep_dispatch(h, tok, off, 4, [[0, 2], [2, 4]], 8, 3)
    with pytest.raises(pz.PuzzleError):  # pair 3 has no owner
        pz.ep_home_index(tok, torch.zeros((4, 2), device="cuda"), off, 4, [[0, 3]], 1, 8)
    with pytest.raises(pz.PuzzleError):  # 4 * lb_max > 2 * d_model: the counts do not fit in a header row
        pz.ep_dispatch(h, tok, off, 4, [[0, 4]], 8, 33)
    with pytest.raises(pz.PuzzleError):  # n_local_buckets beyond what a 64-wide header row holds
        pz.ep_recv_plan(torch.zeros((9, 64), dtype=torch.int16, device="cuda"), 1, 33, 8)


def _ep_world1(cfg, n_merged=None):
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200.ep import ExpertParallelMoE, Partition, shard_dense, shard_packed
    if n_merged is None:
        w13, w2, slot, _ = oracle_packed_layer(cfg)
        dense = None
    else:  # 25% ratio: merged pairs + dense bf16 slots (R20)
        w13, w2, slot, dense = oracle_mixed_layer(cfg, n_merged)
    w13_d = torch.from_numpy(w13.view(np.int16)).cuda()
    w2_d = torch.from_numpy(w2.view(np.int16)).cuda()
    slot_d = torch.from_numpy(slot).cuda()
    n_slots = w13.shape[0]
    part = Partition(n_slots, 1)
    w13_l, w2_l = shard_packed(w13_d, w2_d, part, 0)
    dense_l = shard_dense(None if dense is None else torch.from_numpy(dense.astype(np.uint8)).cuda(), part, 0)
    local = pz.PackedMoELayer(w13_l, w2_l, torch.arange(2 * w13_l.shape[0], dtype=torch.int32, device="cuda"), dense_l)
    route = pz.RoutingLayer(n_slots, cfg.d_model, cfg.d_ff, slot_d, w13_l)
    return ExpertParallelMoE(part, 0, route, local, cfg.d_model), (w13, w2, slot, dense)


@pytest.mark.parametrize("cfg", [synth.MoEConfig("ep_small", 30, 256, 512, 8, 2, True),
                                 synth.MoEConfig("ep_fine", 31, 128, 256, 16, 4, False)], ids=lambda c: c.name)
@pytest.mark.parametrize("T,path", [(37, 0), (64, 1), (5, 1), (200, 0)])
def test_ep_fixed_world1_matches_oracle(nccl_group, cfg, T, path):
    ep, (w13, w2, slot, _) = _ep_world1(cfg)
    hb = synth.hidden_bits(cfg, T, seed=7)
    lg = synth.router_logits(cfg, T, seed=8)
    rb = synth.hidden_bits(cfg, T, seed=9)
    h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    r = torch.from_numpy(rb.view(np.int16)).cuda().view(torch.bfloat16)
    out = ep.forward_fixed(h, torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize, residual=r,
                           cap_tokens=T + 3, path=path)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, rb)
    assert_close(out.float().cpu().numpy(), ref, "fixed-capacity ep vs oracle")


@pytest.mark.parametrize("T,path", [(64, 1), (150, 0)])
def test_ep_fixed_world1_dense_slots_match_oracle(nccl_group, T, path):
    """25% ratio (merged pairs + dense bf16 slots) through the fixed-capacity dispatch."""
    cfg = synth.MoEConfig("ep25_gpu", 33, 256, 512, 8, 2, True)
    ep, (w13, w2, slot, dense) = _ep_world1(cfg, n_merged=2)
    hb = synth.hidden_bits(cfg, T, seed=11)
    lg = synth.router_logits(cfg, T, seed=12)
    h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    out = ep.forward_fixed(h, torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize, path=path)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, pair_dense=dense)
    assert_close(out.float().cpu().numpy(), ref, "fixed-capacity ep (dense slots) vs oracle")


def test_ep_fixed_graph_capture(nccl_group):
    """The fixed-capacity layer has no host sync: it captures into a CUDA graph (NCCL inside)
    and a replay on new inputs equals the oracle."""
    import paper_2511_04805_b200 as pz
    cfg = synth.MoEConfig("ep_graph", 32, 256, 512, 8, 2, True)
    ep, (w13, w2, slot, _) = _ep_world1(cfg)
    T = 16
    h = torch.empty((T, cfg.d_model), dtype=torch.bfloat16, device="cuda")
    lg = torch.empty((T, cfg.n_experts), dtype=torch.float32, device="cuda")

    def load(seed):
        hb = synth.hidden_bits(cfg, T, seed=seed)
        lb = synth.router_logits(cfg, T, seed=seed + 1)
        h.copy_(torch.from_numpy(hb.view(np.int16)).view(torch.bfloat16))
        lg.copy_(torch.from_numpy(lb))
        return hb, lb

    load(40)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside capture (workspaces, NCCL communicator)
        ep.forward_fixed(h, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = ep.forward_fixed(h, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)
    hb, lb = load(50)
    g.replay()
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lb, cfg.top_k, cfg.renormalize)
    assert_close(out.float().cpu().numpy(), ref, "graph-replayed fixed-capacity ep vs oracle")


@pytest.mark.parametrize("cfg,G,n_merged", [
    (synth.MoEConfig("sim_small", 34, 256, 512, 8, 2, True), 2, None),    # 4 pairs: 2 per rank
    (synth.MoEConfig("sim_small", 34, 256, 512, 8, 2, True), 3, None),    # uneven pair blocks
    (synth.MoEConfig("sim_small", 34, 256, 512, 8, 2, True), 8, None),    # world > pairs: d_ff slices
    (synth.MoEConfig("sim_fine", 35, 128, 256, 16, 4, False), 4, None),   # fine-grained, top-4
    (synth.MoEConfig("sim_25", 36, 256, 512, 8, 2, True), 3, 2),          # 25 %: pairs + dense slots
], ids=lambda v: str(v) if not hasattr(v, "name") else v.name)
def test_ep_fixed_simulated_world_matches_oracle(cfg, G, n_merged):
    """G ranks' fixed-capacity EP layers driven in ONE process through the real kernels, phase by
    phase (send -> exchange by slicing -> serve -> exchange -> finish; no rank waits on another
    inside a kernel): every rank's output equals the oracle on its own (ragged) tokens."""
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200.ep import ExpertParallelMoE, Partition, shard_dense, shard_packed
    if n_merged is None:
        w13, w2, slot, _ = oracle_packed_layer(cfg)
        dense = None
    else:
        w13, w2, slot, dense = oracle_mixed_layer(cfg, n_merged)
    n_slots = w13.shape[0]
    w13_d = torch.from_numpy(w13.view(np.int16)).cuda()
    w2_d = torch.from_numpy(w2.view(np.int16)).cuda()
    slot_d = torch.from_numpy(slot).cuda()
    dense_d = None if dense is None else torch.from_numpy(dense.astype(np.uint8)).cuda()
    part = Partition(n_slots, G)
    eps = []
    for r in range(G):
        w13_l, w2_l = shard_packed(w13_d, w2_d, part, r)
        local = pz.PackedMoELayer(w13_l, w2_l, torch.arange(2 * w13_l.shape[0], dtype=torch.int32, device="cuda"),
                                  shard_dense(dense_d, part, r))
        route = pz.RoutingLayer(n_slots, cfg.d_model, cfg.d_ff, slot_d, w13_l)
        eps.append(ExpertParallelMoE(part, r, route, local, cfg.d_model))
    T = 24
    inputs, sends, states = [], [], []
    for r in range(G):
        Tr = T - r if r < G - 1 or G < 3 else 0  # ragged per-rank batches (an idle rank at G >= 3), one capacity
        hb = synth.hidden_bits(cfg, Tr, seed=500 + r)
        lg = synth.router_logits(cfg, Tr, seed=600 + r)
        rb = synth.hidden_bits(cfg, Tr, seed=700 + r)
        inputs.append((hb, lg, rb))
        h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
        s, st = eps[r].fixed_send(h, torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize, cap_tokens=T)
        sends.append(s)
        states.append(st)
    R = T * cfg.top_k + 1  # rows per region
    recv = [torch.cat([sends[s][q * R:(q + 1) * R] for s in range(G)]) for q in range(G)]
    served = [eps[q].fixed_serve(recv[q], R - 1, path=pz.PATH_GEMV) for q in range(G)]
    for r in range(G):
        back = torch.cat([served[q][r * R:(r + 1) * R] for q in range(G)])
        hb, lg, rb = inputs[r]
        out = eps[r].fixed_finish(back, states[r], torch.from_numpy(rb.view(np.int16)).cuda().view(torch.bfloat16))
        torch.cuda.synchronize()
        if hb.shape[0] == 0:
            assert out.shape == (0, cfg.d_model)
            continue
        ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, rb, pair_dense=dense)
        assert_close(out.float().cpu().numpy(), ref, f"simulated world {G}, rank {r}")


# ---- the NVLink peer-memory form: transfers fused into the dispatch / return kernels ----

def _sim_world(cfg, G, n_merged=None):
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200.ep import ExpertParallelMoE, Partition, shard_dense, shard_packed
    if n_merged is None:
        w13, w2, slot, _ = oracle_packed_layer(cfg)
        dense = None
    else:
        w13, w2, slot, dense = oracle_mixed_layer(cfg, n_merged)
    n_slots = w13.shape[0]
    w13_d = torch.from_numpy(w13.view(np.int16)).cuda()
    w2_d = torch.from_numpy(w2.view(np.int16)).cuda()
    slot_d = torch.from_numpy(slot).cuda()
    dense_d = None if dense is None else torch.from_numpy(dense.astype(np.uint8)).cuda()
    part = Partition(n_slots, G)
    eps = []
    for r in range(G):
        w13_l, w2_l = shard_packed(w13_d, w2_d, part, r)
        local = pz.PackedMoELayer(w13_l, w2_l, torch.arange(2 * w13_l.shape[0], dtype=torch.int32, device="cuda"),
                                  shard_dense(dense_d, part, r))
        route = pz.RoutingLayer(n_slots, cfg.d_model, cfg.d_ff, slot_d, w13_l)
        eps.append(ExpertParallelMoE(part, r, route, local, cfg.d_model))
    return eps, (w13, w2, slot, dense)


@pytest.mark.parametrize("cfg,G,n_merged", [
    (synth.MoEConfig("peer_small", 37, 256, 512, 8, 2, True), 2, None),
    (synth.MoEConfig("peer_small", 37, 256, 512, 8, 2, True), 8, None),   # d_ff slices
    (synth.MoEConfig("peer_fine", 38, 128, 256, 16, 4, False), 4, None),
    (synth.MoEConfig("peer_25", 39, 256, 512, 8, 2, True), 3, 2),
], ids=lambda v: str(v) if not hasattr(v, "name") else v.name)
def test_ep_peer_simulated_world_matches_oracle(cfg, G, n_merged):
    """G ranks' peer buffers in one process (plain device memory standing in for the NVLink
    mappings), phases run rank after rank -- every wait is already satisfied when it runs, no
    rank waits on another inside a kernel. Two consecutive steps (the epochs advance)."""
    import paper_2511_04805_b200 as pz
    eps, (w13, w2, slot, dense) = _sim_world(cfg, G, n_merged)
    T = 20
    cap = T * cfg.top_k
    nbytes = pz.EpPeerBuffer.size(G, cap, cfg.d_model)
    bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(G)]
    ptrs = [b.data_ptr() for b in bufs]
    for r in range(G):
        eps[r].attach_peer_buffer(pz.EpPeerBuffer(bufs[r], ptrs, G, cap, cfg.d_model))
    for step in range(2):
        inputs, states = [], []
        for r in range(G):
            Tr = T - (r + step) % 3 if (r, step) != (G - 1, 1) else 0  # ragged; the last rank idle in step 1
            hb = synth.hidden_bits(cfg, Tr, seed=800 + 10 * step + r)
            lg = synth.router_logits(cfg, Tr, seed=900 + 10 * step + r)
            inputs.append((hb, lg))
            h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
            states.append(eps[r].peer_send(h, torch.from_numpy(lg).cuda(), cfg.top_k, cfg.renormalize))
        for r in range(G):
            eps[r].peer_serve(path=pz.PATH_GEMV)
        for r in range(G):
            if (r, step) == (0, 1):  # the two-call form: home-index tables + the plain combine
                st, ep = states[r], eps[r]
                aof_s, gate_s = pz.ep_home_index_peer(st["assign_of"], st["gate"], st["bucket_off"], ep.part.n_pairs,
                                                      ep.dest_pairs, ep.part.slices, ep.pb)
                out = pz.moe_combine(ep.pb.recv_y, aof_s, gate_s)
            else:
                out = eps[r].peer_finish(states[r])
            torch.cuda.synchronize()
            hb, lg = inputs[r]
            if hb.shape[0] == 0:
                assert out.shape == (0, cfg.d_model)
                continue
            ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, pair_dense=dense)
            assert_close(out.float().cpu().numpy(), ref, f"peer world {G}, step {step}, rank {r}")
    assert all(int(ep.pb.state[0].item()) == 2 for ep in eps)  # two steps published
    assert all(ep.pb.wait_timeouts() == 0 for ep in eps)


def test_ep_peer_world1_symmetric_memory_graph(nccl_group):
    """World 1 through torch symmetric memory (the multi-GPU allocation path) and a CUDA graph:
    the device-side epochs make replays correct without any reset."""
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200.ep import make_peer_buffer
    cfg = synth.MoEConfig("peer_graph", 40, 256, 512, 8, 2, True)
    ep, (w13, w2, slot, _) = _ep_world1(cfg)
    T = 16
    try:
        pb = make_peer_buffer(1, T * cfg.top_k, cfg.d_model, torch.device("cuda", 0))
    except Exception as e:  # pragma: no cover
        pytest.skip(f"torch symmetric memory unavailable here: {e!r}")
    ep.attach_peer_buffer(pb)
    h = torch.empty((T, cfg.d_model), dtype=torch.bfloat16, device="cuda")
    lg = torch.empty((T, cfg.n_experts), dtype=torch.float32, device="cuda")

    def load(seed):
        hb = synth.hidden_bits(cfg, T, seed=seed)
        lb = synth.router_logits(cfg, T, seed=seed + 1)
        h.copy_(torch.from_numpy(hb.view(np.int16)).view(torch.bfloat16))
        lg.copy_(torch.from_numpy(lb))
        return hb, lb

    hb, lb = load(60)
    out = ep.forward_peer(h, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)  # eager
    torch.cuda.synchronize()
    assert_close(out.float().cpu().numpy(), oracle.moe_forward(w13, w2, slot, hb, lb, cfg.top_k, cfg.renormalize),
                 "peer world 1 eager")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = ep.forward_peer(h, lg, cfg.top_k, cfg.renormalize, path=pz.PATH_GEMV)
    for seed in (70, 80):
        hb, lb = load(seed)
        g.replay()
        torch.cuda.synchronize()
        assert_close(out.float().cpu().numpy(), oracle.moe_forward(w13, w2, slot, hb, lb, cfg.top_k, cfg.renormalize),
                     f"peer world 1 replay {seed}")
    assert pb.wait_timeouts() == 0 and int(pb.state[0].item()) == 3


# ---- the same layer behind the C ABI: a C-owned NCCL communicator (puzzle_moe_forward_ep) ----

@pytest.fixture(scope="module")
def ep_comm():
    import paper_2511_04805_b200 as pz
    comm = pz.EpComm(1, 0, pz.ep_unique_id(), 0)
    yield comm
    comm.close()


@pytest.mark.parametrize("cfg", [synth.MoEConfig("ep_small", 30, 256, 512, 8, 2, True),
                                 synth.MoEConfig("ep_fine", 31, 128, 256, 16, 4, False)], ids=lambda c: c.name)
@pytest.mark.parametrize("T,path", [(37, 0), (64, 1), (5, 1), (200, 0), (0, 0)])
def test_ep_capi_world1_matches_oracle_and_python_form(nccl_group, ep_comm, cfg, T, path):
    """puzzle_moe_forward_ep on a 1-rank communicator: equal to the oracle under the tolerance
    and bit-identical to the torch.distributed fixed-capacity form (same kernels, same order)."""
    ep, (w13, w2, slot, _) = _ep_world1(cfg)
    hb = synth.hidden_bits(cfg, T, seed=7)
    lg = synth.router_logits(cfg, T, seed=8)
    rb = synth.hidden_bits(cfg, T, seed=9)
    h = torch.from_numpy(hb.view(np.int16)).cuda().view(torch.bfloat16)
    r = torch.from_numpy(rb.view(np.int16)).cuda().view(torch.bfloat16)
    l = torch.from_numpy(lg).cuda()
    cap = T + 3
    out = ep_comm.forward(ep.route_layer, ep.local_layer, h, l, cfg.top_k, cfg.renormalize, cap_tokens=cap,
                          residual=r, path=path)
    if T == 0:
        return
    py = ep.forward_fixed(h, l, cfg.top_k, cfg.renormalize, residual=r, cap_tokens=cap, path=path)
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, rb)
    assert_close(out.float().cpu().numpy(), ref, "C-ABI ep vs oracle")
    assert torch.equal(out.view(torch.int16), py.view(torch.int16))


def test_ep_capi_dense_slots_and_graph_capture(nccl_group, ep_comm):
    """25 % layout through the C-ABI layer, captured into a CUDA graph (NCCL inside) and
    replayed on new inputs."""
    cfg = synth.MoEConfig("ep25_capi", 33, 256, 512, 8, 2, True)
    ep, (w13, w2, slot, dense) = _ep_world1(cfg, n_merged=2)
    T = 24
    h = torch.empty((T, cfg.d_model), dtype=torch.bfloat16, device="cuda")
    lg = torch.empty((T, cfg.n_experts), dtype=torch.float32, device="cuda")

    def load(seed):
        hb = synth.hidden_bits(cfg, T, seed=seed)
        lb = synth.router_logits(cfg, T, seed=seed + 1)
        h.copy_(torch.from_numpy(hb.view(np.int16)).view(torch.bfloat16))
        lg.copy_(torch.from_numpy(lb))
        return hb, lb

    load(60)
    out = torch.empty_like(h)
    ws = ep_comm.workspace(ep.route_layer, ep.local_layer, T, cfg.top_k)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ep_comm.forward(ep.route_layer, ep.local_layer, h, lg, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ep_comm.forward(ep.route_layer, ep.local_layer, h, lg, cfg.top_k, cfg.renormalize, out=out, workspace=ws)
    hb, lb = load(70)
    g.replay()
    torch.cuda.synchronize()
    ref = oracle.moe_forward(w13, w2, slot, hb, lb, cfg.top_k, cfg.renormalize, pair_dense=dense)
    assert_close(out.float().cpu().numpy(), ref, "graph-replayed C-ABI ep (dense slots) vs oracle")


def test_ep_capi_rejects_mismatched_shard(nccl_group, ep_comm):
    import paper_2511_04805_b200 as pz
    cfg = synth.MoEConfig("ep_small", 30, 256, 512, 8, 2, True)
    ep, _ = _ep_world1(cfg)
    wrong = pz.PackedMoELayer(ep.local_layer.w13[:1].contiguous(), ep.local_layer.w2[:1].contiguous(),
                              torch.arange(2, dtype=torch.int32, device="cuda"))
    h = torch.zeros((4, cfg.d_model), dtype=torch.bfloat16, device="cuda")
    l = torch.zeros((4, cfg.n_experts), dtype=torch.float32, device="cuda")
    ws = torch.empty(1 << 26, dtype=torch.uint8, device="cuda")
    with pytest.raises(pz.PuzzleError) as e:
        ep_comm.forward(ep.route_layer, wrong, h, l, cfg.top_k, cfg.renormalize, workspace=ws)
    assert e.value.status == 2
