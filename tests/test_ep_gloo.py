"""Expert-parallel host logic (paper_2511_04805_b200/ep.py) on CPU: world size 2 over gloo.

The EP orchestration (partition, count exchange, variable-split dispatch, regroup into local
bucket order, un-permute, return, combine with d_ff-slice partials) is exactly the product
code; only the device ops are replaced by a CPU stand-in built on the oracle (test double).
Each rank's output must equal the single-process oracle forward on that rank's tokens."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from helpers import (ep_dispatch_ref, ep_home_index_ref, ep_recv_plan_ref, oracle_mixed_layer,
                     oracle_packed_layer)


class OracleOps:
    """CPU stand-in for the EP data-path kernels (tests only)."""

    def route(self, route_layer, logits, k, renorm):
        slot = route_layer["expert_slot"]
        idx, gate = oracle.route(logits.numpy(), k, renorm)
        T = idx.shape[0]
        b = slot[idx.reshape(-1)]
        order = np.argsort(b, kind="stable")           # bucket order, token order inside
        counts = np.bincount(b, minlength=2 * route_layer["n_pairs"])
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        assign_token = (order // k).astype(np.int32)
        assign_of = np.empty(T * k, np.int32)
        assign_of[order] = np.arange(T * k, dtype=np.int32)
        return (torch.from_numpy(idx), torch.from_numpy(gate.astype(np.float32)), torch.from_numpy(off),
                torch.from_numpy(assign_token), torch.from_numpy(assign_of))

    def gather_rows(self, src, index):
        return src[index.long()]

    def experts(self, local_layer, x_rows, bucket_off, path=None):
        w13, w2, dense = local_layer
        off = bucket_off.numpy()
        bits = x_rows.contiguous().view(torch.int16).numpy().view(np.uint16)
        y = np.zeros((x_rows.shape[0], w13.shape[3]), np.float32)
        for b in range(len(off) - 1):
            if off[b + 1] > off[b]:
                y[off[b]:off[b + 1]] = oracle.expert_ffn(w13, w2, b // 2, b % 2, bits[off[b]:off[b + 1]],
                                                         dense=dense is not None and bool(dense[b // 2]))
        return torch.from_numpy(y)

    def ep_dispatch(self, hidden, assign_token, bucket_off, n_pairs, dest_pairs, cap, lb_max):
        bits = hidden.contiguous().view(torch.int16).numpy()
        rows = ep_dispatch_ref(bits, assign_token.numpy(), bucket_off.numpy(), dest_pairs, cap, lb_max)
        return torch.from_numpy(rows).view(hidden.dtype)

    def ep_recv_plan(self, recv_rows, world, n_local_buckets, cap):
        bits = recv_rows.contiguous().view(torch.int16).numpy()
        return tuple(torch.from_numpy(a) for a in ep_recv_plan_ref(bits, world, n_local_buckets, cap))

    def ep_home_index(self, assign_of, gate, bucket_off, n_pairs, dest_pairs, slices, cap):
        return tuple(torch.from_numpy(a) for a in ep_home_index_ref(assign_of.numpy(), gate.numpy(),
                                                                     bucket_off.numpy(), dest_pairs, slices, cap))

    def combine(self, y, assign_of, gate, residual):
        T, k = gate.shape
        out = (y[assign_of.long()].reshape(T, k, -1).double() * gate.double()[:, :, None]).sum(1)
        if residual is not None:
            out = out + residual.double()
        return out


def _worker(rank, world, port, cfg_fields, T, outdir, n_merged=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_04805_b200.ep import ExpertParallelMoE, Partition, shard_dense, shard_packed
        cfg = synth.MoEConfig(*cfg_fields)
        if n_merged is None:
            w13, w2, slot, _ = oracle_packed_layer(cfg)
            dense = None
        else:  # 25% ratio: merged pairs + dense slots (R20)
            w13, w2, slot, dense = oracle_mixed_layer(cfg, n_merged)
        n_slots = w13.shape[0]
        part = Partition(n_slots, world)
        w13_l, w2_l = shard_packed(torch.from_numpy(w13.view(np.int16)), torch.from_numpy(w2.view(np.int16)), part, rank)
        dense_l = shard_dense(None if dense is None else torch.from_numpy(dense), part, rank)
        local = (w13_l.numpy().view(np.uint16), w2_l.numpy().view(np.uint16),
                 None if dense_l is None else dense_l.numpy())
        layer = ExpertParallelMoE(part, rank, {"expert_slot": slot, "n_pairs": n_slots}, local, cfg.d_model,
                                  ops=OracleOps())
        Tr = T - rank  # ragged: the ranks hold different token counts (fixed path: cap_tokens = T + 1)
        hb = synth.hidden_bits(cfg, Tr, seed=100 + rank)
        lg = synth.router_logits(cfg, Tr, seed=200 + rank)
        rb = synth.hidden_bits(cfg, Tr, seed=300 + rank)
        hidden = torch.from_numpy(hb.view(np.int16)).view(torch.bfloat16)
        resid = torch.from_numpy(oracle.bf16_bits_to_f32(rb))
        out = layer.forward(hidden, torch.from_numpy(lg), cfg.top_k, cfg.renormalize, residual=resid)
        ref = oracle.moe_forward(w13, w2, slot, hb, lg, cfg.top_k, cfg.renormalize, rb, pair_dense=dense)
        np.save(os.path.join(outdir, f"out{rank}.npy"), out.numpy())
        # fixed-capacity dispatch (device-side index tables; one spare token of capacity)
        outf = layer.forward_fixed(hidden, torch.from_numpy(lg), cfg.top_k, cfg.renormalize, residual=resid,
                                   cap_tokens=T + 1)
        np.save(os.path.join(outdir, f"outf{rank}.npy"), outf.numpy())
        np.save(os.path.join(outdir, f"ref{rank}.npy"), ref)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cfg_fields,T", [
    (("ep4", 20, 64, 128, 8, 2, True), 6),      # 4 pairs over 2 ranks: 2 pairs each
    (("ep2", 21, 64, 128, 4, 3, False), 5),     # 2 pairs over 2 ranks: 1 pair each
    (("ep1", 22, 64, 128, 2, 1, True), 7),      # 1 pair over 2 ranks: d_ff split in 2 slices
    (("ep1k2", 23, 64, 128, 2, 2, True), 4),    # both experts of the one pair, d_ff split
])
def test_ep_world2_matches_oracle(cfg_fields, T):
    _run_world2(cfg_fields, T, None)


@pytest.mark.parametrize("cfg_fields,T,n_merged", [
    (("ep25", 24, 64, 128, 8, 2, True), 9, 2),   # 2 merged pairs + 4 dense slots over 2 ranks
    (("ep25s", 25, 64, 128, 2, 1, True), 6, 0),  # 2 dense slots, one per rank
])
def test_ep_world2_dense_slots_match_oracle(cfg_fields, T, n_merged):
    _run_world2(cfg_fields, T, n_merged)


def _run_world2(cfg_fields, T, n_merged):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), cfg_fields, T, d, n_merged), nprocs=2, join=True)
        for r in range(2):
            out = np.load(os.path.join(d, f"out{r}.npy"))
            ref = np.load(os.path.join(d, f"ref{r}.npy"))
            np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)
            outf = np.load(os.path.join(d, f"outf{r}.npy"))
            np.testing.assert_allclose(outf, ref, rtol=1e-5, atol=1e-5)


def test_partition_layout():
    from paper_2511_04805_b200.ep import Partition
    p = Partition(30, 8)
    spans = [p.pairs_of(r) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 30
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert sorted(b - a for a, b in spans) == [3, 3, 4, 4, 4, 4, 4, 4]
    q = Partition(4, 8)
    assert q.slices == 2 and q.pairs_of(5) == (2, 3) and q.slice_of(5) == 1 and q.owners(2) == [4, 5]
    with pytest.raises(ValueError):
        _ = Partition(3, 8).slices
