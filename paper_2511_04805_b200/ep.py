"""Expert parallelism: PuzzleMoE merged pairs sharded over the GPUs of one node,
tokens dispatched to the pair owners and back with all-to-all (NCCL over NVLink in production,
gloo in the CPU tests).

Partition (the unit is a merged PAIR, so both experts of a pair stay co-resident and each
packed tile is still read once):
  world <= P : rank r owns pairs [floor(r P / G), floor((r+1) P / G)).
  world >  P : world % P == 0; each pair is split along d_ff into G/P slices (SwiGLU is
               elementwise in d_ff, so every slice computes an exact partial of W2 h; the
               partials are summed by the combine on the token's home rank).

Per layer (every rank holds T_local tokens of its own):
  1. route (a3) against the global pairing -> top-k, gates, global buckets (pair-major),
  2. rows gathered into bucket order (the buckets of a rank's pairs are contiguous),
  3. per-bucket counts exchanged (all_to_all), rows dispatched (all_to_all, variable splits),
  4. received rows regrouped into the owner's local bucket order, local experts (a4)+(a5),
  5. outputs un-permuted and sent home (all_to_all), combine (a6) with the home gates.
Every data-path step runs in libpuzzlemoe kernels (route, gather, experts, combine); torch
supplies the collectives and the host-side split sizes (one D2H copy of the bucket counts).

forward_fixed is the same layer with FIXED-CAPACITY dispatch: every rank reserves cap =
cap_tokens*top_k rows per destination, so both all-to-alls have equal splits known up front and
the index work of steps 3-5 runs in device kernels (puzzle_ep_dispatch / puzzle_ep_recv_plan /
puzzle_ep_home_index): no device->host copy, so a decode layer can be captured in a CUDA graph.
It moves world*(cap+1) rows per collective instead of the routed count (the price of static
splits; the extra row per destination carries its bucket counts, so no count exchange).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch
import torch.distributed as dist


@dataclasses.dataclass(frozen=True)
class Partition:
    n_pairs: int
    world: int

    @property
    def slices(self) -> int:
        """d_ff slices per pair (1 unless world > n_pairs)."""
        if self.world <= self.n_pairs:
            return 1
        if self.world % self.n_pairs:
            raise ValueError("expert parallelism with world > n_pairs needs world % n_pairs == 0")
        return self.world // self.n_pairs

    def pairs_of(self, rank: int) -> tuple[int, int]:
        """[first, last) global pair ids held (whole pairs, or one pair's d_ff slice)."""
        if self.slices == 1:
            return (rank * self.n_pairs) // self.world, ((rank + 1) * self.n_pairs) // self.world
        p = rank // self.slices
        return p, p + 1

    def slice_of(self, rank: int) -> int:
        return rank % self.slices

    def owners(self, pair: int) -> list[int]:
        if self.slices == 1:
            return [r for r in range(self.world) if self.pairs_of(r)[0] <= pair < self.pairs_of(r)[1]]
        return [pair * self.slices + j for j in range(self.slices)]


def shard_packed(w13: torch.Tensor, w2: torch.Tensor, part: Partition, rank: int):
    """Packed weights this rank holds: w13 [P,2,f,d] -> [p1-p0, 2, f/S, d]; w2 [P,d,f] ->
    [p1-p0, d, f/S] (a d_ff slice of a packed tensor is still a valid packed tensor: the
    decode is elementwise)."""
    p0, p1 = part.pairs_of(rank)
    S = part.slices
    f = w13.shape[2]
    if f % S or (f // S) % 64:
        raise ValueError("d_ff / slices must be a multiple of 64")
    fs = f // S
    j = part.slice_of(rank)
    w13_l = w13[p0:p1, :, j * fs:(j + 1) * fs, :].contiguous()
    w2_l = w2[p0:p1, :, j * fs:(j + 1) * fs].contiguous()
    return w13_l, w2_l


def shard_dense(pair_dense: torch.Tensor | None, part: Partition, rank: int):
    """This rank's slice of the dense-slot flags (25% ratio, reading R20); None stays None."""
    if pair_dense is None:
        return None
    p0, p1 = part.pairs_of(rank)
    return pair_dense[p0:p1].contiguous()


class CudaOps:
    """Device ops of the EP data path: libpuzzlemoe kernels."""

    def __init__(self):
        import paper_2511_04805_b200 as pz
        self.pz = pz

    def route(self, route_layer, logits, k, renorm):
        return route_layer.route(logits, k, renorm)

    def gather_rows(self, src, index):
        if src.dtype == torch.float32:  # 4-byte rows move as pairs of 16-bit columns
            return self.pz.gather_rows(src.view(torch.int16), index).view(torch.float32)
        return self.pz.gather_rows(src, index)

    def experts(self, local_layer, x_rows, bucket_off, path=None):
        return local_layer.experts(x_rows, bucket_off, path=self.pz.PATH_AUTO if path is None else path)

    def combine(self, y, assign_of, gate, residual):
        return self.pz.moe_combine(y, assign_of, gate, residual=residual)

    def ep_dispatch(self, hidden, assign_token, bucket_off, n_pairs, dest_pairs, cap, lb_max):
        return self.pz.ep_dispatch(hidden, assign_token, bucket_off, n_pairs, dest_pairs, cap, lb_max)

    def ep_recv_plan(self, recv_rows, world, n_local_buckets, cap):
        return self.pz.ep_recv_plan(recv_rows, world, n_local_buckets, cap)

    def ep_home_index(self, assign_of, gate, bucket_off, n_pairs, dest_pairs, slices, cap):
        return self.pz.ep_home_index(assign_of, gate, bucket_off, n_pairs, dest_pairs, slices, cap)

    # NVLink peer-memory form (transfers fused into the dispatch / return kernels)
    def ep_dispatch_peer(self, hidden, assign_token, bucket_off, n_pairs, dest_pairs, rank, pb, lb_max):
        self.pz.ep_dispatch_peer(hidden, assign_token, bucket_off, n_pairs, dest_pairs, rank, pb, lb_max)

    def ep_wait_dispatch(self, pb):
        self.pz.ep_wait_dispatch(pb)

    def ep_recv_plan_peer(self, pb, n_local_buckets):
        return self.pz.ep_recv_plan_peer(pb, n_local_buckets)

    def ep_return_peer(self, y_local, return_idx, rank, n_local_buckets, pb):
        self.pz.ep_return_peer(y_local, return_idx, rank, n_local_buckets, pb)

    def ep_home_index_peer(self, assign_of, gate, bucket_off, n_pairs, dest_pairs, slices, pb):
        return self.pz.ep_home_index_peer(assign_of, gate, bucket_off, n_pairs, dest_pairs, slices, pb)

    def ep_combine_peer(self, assign_of, gate, bucket_off, n_pairs, dest_pairs, pb, residual):
        return self.pz.ep_combine_peer(assign_of, gate, bucket_off, n_pairs, dest_pairs, pb, residual=residual)


class ExpertParallelMoE:
    """One MoE layer sharded by merged pairs over `world` ranks of `group`.

    route_layer: a layer descriptor whose routing metadata (n_experts, n_pairs, expert_slot)
                 is GLOBAL (route reads no weights); local_layer: this rank's packed shard."""

    def __init__(self, part: Partition, rank: int, route_layer, local_layer, d_model: int, group=None, ops=None):
        self.part, self.rank, self.world = part, rank, part.world
        self.route_layer, self.local_layer = route_layer, local_layer
        self.d = d_model
        self.group = group
        self.ops = ops if ops is not None else CudaOps()
        # local bucket b_local = 2 * (pair - p0) + pos
        self.p0, self.p1 = part.pairs_of(rank)
        self.n_local_buckets = 2 * (self.p1 - self.p0)
        # fixed-capacity dispatch tables (host): [world][2] pair ranges, count-table row stride
        self.dest_pairs = np.array([part.pairs_of(q) for q in range(part.world)], dtype=np.int32)
        self.lb_max = int(2 * max(b - a for a, b in self.dest_pairs))

    def _a2a(self, out, inp, out_splits, in_splits):
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def forward(self, hidden, logits, top_k: int, renormalize: bool, residual=None):
        ops, part, G, r = self.ops, self.part, self.world, self.rank
        dev = hidden.device
        T = hidden.shape[0]
        topk_idx, gate, bucket_off, assign_token, assign_of = ops.route(self.route_layer, logits, top_k, renormalize)
        off = bucket_off.cpu().numpy().astype(np.int64)  # the one D2H sync (split sizes)
        counts = np.diff(off)
        # ---- dispatch plan: rows for rank q = its pairs' buckets (duplicated for d_ff slices)
        send_index, send_split, send_counts = [], [], []
        for q in range(G):
            qa, qb = part.pairs_of(q)
            lo, hi = off[2 * qa], off[2 * qb]
            send_index.append(np.arange(lo, hi, dtype=np.int64))
            send_split.append(int(hi - lo))
            send_counts.append(counts[2 * qa:2 * qb])
        send_index = np.concatenate(send_index) if send_index else np.zeros(0, np.int64)
        x_perm = ops.gather_rows(hidden, assign_token)                   # bucket order
        if part.slices == 1:
            send_buf = x_perm                                            # already rank-major
        else:
            send_buf = ops.gather_rows(x_perm, torch.from_numpy(send_index.astype(np.int32)).to(dev))
        # ---- per-bucket counts: each rank learns [source][local bucket] counts
        lb = [2 * (part.pairs_of(q)[1] - part.pairs_of(q)[0]) for q in range(G)]
        c_send = torch.from_numpy(np.concatenate(send_counts).astype(np.int64)) if send_counts else torch.zeros(0, dtype=torch.int64)
        c_recv = torch.empty(G * lb[r], dtype=torch.int64)
        if dev.type == "cuda" and dist.get_backend(self.group) == "nccl":
            c_send_d, c_recv_d = c_send.to(dev), c_recv.to(dev)
            self._a2a(c_recv_d, c_send_d, [lb[r]] * G, lb)
            c_recv = c_recv_d.cpu()
        else:
            self._a2a(c_recv, c_send, [lb[r]] * G, lb)
        rc = c_recv.numpy().reshape(G, lb[r])                             # [source][local bucket]
        recv_split = rc.sum(1).astype(np.int64)
        # ---- rows to the owners
        x_recv = torch.empty((int(recv_split.sum()), self.d), dtype=hidden.dtype, device=dev)
        self._a2a(x_recv, send_buf, [int(v) for v in recv_split], send_split)
        # ---- regroup by local bucket: (bucket, source) order
        src_base = np.concatenate([[0], np.cumsum(recv_split)[:-1]]).astype(np.int64)
        within = np.concatenate([np.zeros((G, 1), np.int64), np.cumsum(rc, 1)[:, :-1]], 1)
        regroup = [src_base[s] + within[s, b] + np.arange(rc[s, b], dtype=np.int64)
                   for b in range(lb[r]) for s in range(G)]
        regroup = np.concatenate(regroup) if regroup else np.zeros(0, np.int64)
        local_off = np.concatenate([[0], np.cumsum(rc.sum(0))]).astype(np.int32)
        n_local = int(local_off[-1])
        if n_local > 0:
            x_local = ops.gather_rows(x_recv, torch.from_numpy(regroup.astype(np.int32)).to(dev))
            y_local = ops.experts(self.local_layer, x_local, torch.from_numpy(local_off).to(dev))
            inv = np.empty_like(regroup)
            inv[regroup] = np.arange(regroup.size)
            y_recv = ops.gather_rows(y_local, torch.from_numpy(inv.astype(np.int32)).to(dev))
        else:
            y_recv = torch.empty((0, self.d), dtype=torch.float32, device=dev)
        # ---- outputs home, aligned with send_buf rows
        y_back = torch.empty((int(sum(send_split)), self.d), dtype=torch.float32, device=dev)
        self._a2a(y_back, y_recv, send_split, [int(v) for v in recv_split])
        # ---- combine: every (t, j) sums its S partial rows with the full gate
        S = part.slices
        if S == 1:
            return ops.combine(y_back, assign_of, gate, residual)
        # row of assignment a's s-th copy inside send_buf / y_back
        pos_of = np.empty((off[-1], S), np.int64)
        seen = np.zeros(off[-1], np.int64)
        for i, a in enumerate(send_index):
            pos_of[a, seen[a]] = i
            seen[a] += 1
        aof = assign_of.cpu().numpy().astype(np.int64).reshape(T, top_k)
        aof_s = pos_of[aof].reshape(T, top_k * S).astype(np.int32)
        gate_s = gate.reshape(T, top_k, 1).expand(T, top_k, S).reshape(T, top_k * S).contiguous()
        return ops.combine(y_back, torch.from_numpy(aof_s).to(dev).reshape(-1), gate_s, residual)

    def _a2a_equal(self, out, inp):
        dist.all_to_all_single(out, inp, group=self.group)

    def forward_fixed(self, hidden, logits, top_k: int, renormalize: bool, residual=None,
                      cap_tokens: int | None = None, path=None):
        """The layer with fixed-capacity dispatch: device-only, no host synchronisation.

        cap_tokens (default: this rank's T) bounds every rank's token count and must be the same
        on all ranks; each rank sends world * (cap_tokens * top_k + 1) rows per all-to-all (the +1:
        a header row with the destination's bucket counts). path is
        passed to the local experts call (e.g. PATH_GEMV for decode-shape batches, whose owner
        receives up to world * cap rows)."""
        send_rows, state = self.fixed_send(hidden, logits, top_k, renormalize, cap_tokens)
        x_recv = torch.empty_like(send_rows)
        self._a2a_equal(x_recv, send_rows)
        y_recv = self.fixed_serve(x_recv, state["cap"], path)
        y_back = torch.empty_like(y_recv)
        self._a2a_equal(y_back, y_recv)
        return self.fixed_finish(y_back, state, residual)

    # The three local phases of forward_fixed, between which the two all-to-alls run (exposed so
    # a test can drive several ranks' phases in one process with the exchange done by slicing).
    def fixed_send(self, hidden, logits, top_k: int, renormalize: bool, cap_tokens: int | None = None):
        """route + dispatch: (send_rows [world*(cap+1)][d], state for fixed_finish)."""
        ops, part = self.ops, self.part
        T = hidden.shape[0]
        cap = (T if cap_tokens is None else int(cap_tokens)) * top_k  # row slots per destination (+1 header)
        if cap < T * top_k:
            raise ValueError("cap_tokens must be >= the number of tokens on this rank")
        topk_idx, gate, bucket_off, assign_token, assign_of = ops.route(self.route_layer, logits, top_k, renormalize)
        # every destination's rows (its pairs' buckets) into its fixed region, its bucket counts in
        # the region's header row: ONE all-to-all moves both
        send_rows = ops.ep_dispatch(hidden, assign_token, bucket_off, part.n_pairs, self.dest_pairs, cap, self.lb_max)
        return send_rows, {"cap": cap, "gate": gate, "bucket_off": bucket_off, "assign_of": assign_of}

    def fixed_serve(self, x_recv, cap: int, path=None):
        """owner: regroup the received regions into (local bucket, source) order, run the local
        experts, put the outputs back into the arrival slots (same region layout)."""
        ops = self.ops
        local_off, gidx, ridx = ops.ep_recv_plan(x_recv, self.world, self.n_local_buckets, cap)
        x_local = ops.gather_rows(x_recv, gidx)
        y_local = ops.experts(self.local_layer, x_local, local_off, path=path)
        return ops.gather_rows(y_local, ridx)

    def fixed_finish(self, y_back, state, residual=None):
        """home: region q of y_back = owner q's results for the rows sent to it -> combine."""
        part = self.part
        aof_s, gate_s = self.ops.ep_home_index(state["assign_of"], state["gate"], state["bucket_off"], part.n_pairs,
                                               self.dest_pairs, part.slices, state["cap"])
        return self.ops.combine(y_back, aof_s, gate_s, residual)

    # ---- the fixed-capacity layer over NVLink peer memory (no NCCL on the data path) ----
    def attach_peer_buffer(self, pb):
        """pb: paper_2511_04805_b200.EpPeerBuffer of this rank (see make_peer_buffer)."""
        self.pb = pb

    def forward_peer(self, hidden, logits, top_k: int, renormalize: bool, residual=None, path=None):
        """forward_fixed with the transfers fused into the dispatch / return kernels: rows are
        stored straight into the owners' peer buffers, outputs straight into the home ranks'
        (cap = the peer buffer's capacity; the same on every rank)."""
        state = self.peer_send(hidden, logits, top_k, renormalize)
        self.peer_serve(path)
        return self.peer_finish(state, residual)

    def peer_send(self, hidden, logits, top_k: int, renormalize: bool):
        ops, part, pb = self.ops, self.part, self.pb
        if hidden.shape[0] * top_k > pb.cap:
            raise ValueError("more assignments than the peer buffer's capacity")
        topk_idx, gate, bucket_off, assign_token, assign_of = ops.route(self.route_layer, logits, top_k, renormalize)
        ops.ep_dispatch_peer(hidden, assign_token, bucket_off, part.n_pairs, self.dest_pairs, self.rank, pb, self.lb_max)
        return {"gate": gate, "bucket_off": bucket_off, "assign_of": assign_of}

    def peer_serve(self, path=None):
        ops, pb = self.ops, self.pb
        local_off, gidx, ridx = ops.ep_recv_plan_peer(pb, self.n_local_buckets)  # waits for the dispatch
        x_local = ops.gather_rows(pb.recv_x, gidx)
        y_local = ops.experts(self.local_layer, x_local, local_off, path=path)
        ops.ep_return_peer(y_local, ridx, self.rank, self.n_local_buckets, pb)

    def peer_finish(self, state, residual=None):
        ops, part, pb = self.ops, self.part, self.pb
        # waits for every owner's return, combines from recv_y, advances the step (one kernel)
        return ops.ep_combine_peer(state["assign_of"], state["gate"], state["bucket_off"], part.n_pairs,
                                   self.dest_pairs, pb, residual)


def make_peer_buffer(world: int, cap: int, d_model: int, device, group=None):
    """This rank's EpPeerBuffer in torch symmetric memory (CUDA peer mappings over NVLink):
    every rank of `group` calls it with the same (world, cap, d_model)."""
    import paper_2511_04805_b200 as pz
    import torch.distributed._symmetric_memory as symm
    nbytes = pz.EpPeerBuffer.size(world, cap, d_model)
    group = group if group is not None else dist.group.WORLD
    name = group.group_name
    buf = symm.empty(nbytes, dtype=torch.uint8, device=device)
    hdl = symm.rendezvous(buf, name)
    buf.zero_()
    torch.cuda.synchronize(device)
    dist.barrier(group=group)
    return pz.EpPeerBuffer(buf, [int(p) for p in hdl.buffer_ptrs], world, cap, d_model)
