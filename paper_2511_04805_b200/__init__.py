"""B200-native PuzzleMoE packed-expert MoE FFN (arXiv 2511.04805).

Thin Python binding over the C ABI of ``libpuzzlemoe.so`` (declared in
``include/puzzlemoe.h``). Functions carry the C names without the ``puzzle_`` prefix
and only marshal torch CUDA tensors (pointer, size, current stream) into the library:
every step of the path runs in the library's sm_100a kernels. There is no CPU
fallback -- if the shared library is missing or no CUDA device is present, calls raise.

Build the library with ``python -m paper_2511_04805_b200.build`` (or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# PUZZLE_LIB points at an alternative build of the same library (tuning variants built by
# scripts/build_variant.py); by default the in-tree build is loaded.
LIB_PATH = os.environ.get("PUZZLE_LIB") or os.path.join(_HERE, "libpuzzlemoe.so")

PUZZLE_OK = 0
PUZZLE_ERR_NCCL = 6
EP_UNIQUE_ID_BYTES = 128
PATH_AUTO, PATH_GEMV, PATH_TC, PATH_TS = 0, 1, 2, 3

EXPORTED_SYMBOLS = (
    "puzzle_status_string", "puzzle_last_error", "puzzle_abi_version", "puzzle_merge_pack",
    "puzzle_unpack", "puzzle_merge_experts_pack", "puzzle_moe_workspace_size", "puzzle_moe_forward",
    "puzzle_moe_forward_ex", "puzzle_moe_route", "puzzle_moe_experts_workspace_size",
    "puzzle_moe_experts", "puzzle_moe_combine", "puzzle_gather_rows", "puzzle_profile_begin",
    "puzzle_profile_end", "puzzle_moe_route_workspace_size", "puzzle_group_colsumsq_workspace_size",
    "puzzle_group_colsumsq", "puzzle_moe_calib_workspace_size", "puzzle_moe_forward_calib",
    "puzzle_quant_pack", "puzzle_quant_unpack", "puzzle_quant_gemv", "puzzle_ep_dispatch", "puzzle_ep_recv_plan",
    "puzzle_ep_home_index", "puzzle_ep_peer_buffer_size", "puzzle_ep_dispatch_peer", "puzzle_ep_wait_dispatch",
    "puzzle_ep_return_peer", "puzzle_ep_home_index_peer", "puzzle_ep_recv_plan_peer", "puzzle_ep_combine_peer",
    "puzzle_ep_unique_id", "puzzle_ep_create", "puzzle_ep_destroy", "puzzle_ep_partition",
    "puzzle_moe_forward_ep_workspace_size", "puzzle_moe_forward_ep",
    "puzzle_moe_quant_workspace_size", "puzzle_moe_forward_quant",
)


class PuzzleError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {detail} (status {status})")
        self.status = status


class PackStats(ctypes.Structure):
    _fields_ = [("rounded_up", ctypes.c_ulonglong), ("saturated", ctypes.c_ulonglong),
                ("nonfinite", ctypes.c_ulonglong), ("negative", ctypes.c_ulonglong)]


class MoELayerDesc(ctypes.Structure):
    """puzzle_moe_layer."""
    _fields_ = [("n_experts", ctypes.c_int32), ("n_pairs", ctypes.c_int32), ("d_model", ctypes.c_int32),
                ("d_ff", ctypes.c_int32), ("w13", ctypes.c_void_p), ("w2", ctypes.c_void_p),
                ("expert_slot", ctypes.c_void_p), ("pair_dense", ctypes.c_void_p)]


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpuzzlemoe.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_2511_04805_b200.build` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        P, I, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        sig = {
            "puzzle_status_string": ([I], ctypes.c_char_p),
            "puzzle_last_error": ([], ctypes.c_char_p),
            "puzzle_abi_version": ([], I),
            "puzzle_merge_pack": ([P, P, P, P, P, I64, P, P, P], I),
            "puzzle_unpack": ([P, I, I64, P, P], I),
            "puzzle_merge_experts_pack": ([P, P, P, P, I64, I64, I64, ctypes.c_float, P, P, P], I),
            "puzzle_moe_workspace_size": ([P, I64, I], SZ),
            "puzzle_moe_forward": ([P, P, P, I64, I, I, P, P, P, SZ, P], I),
            "puzzle_moe_forward_ex": ([P, P, P, I64, I, I, P, P, P, SZ, I, P], I),
            "puzzle_moe_route": ([P, P, I64, I, I, P, P, P, P, P, P, SZ, P], I),
            "puzzle_moe_route_workspace_size": ([P], SZ),
            "puzzle_moe_experts_workspace_size": ([P, I64], SZ),
            "puzzle_moe_experts": ([P, P, P, I64, P, P, SZ, I, P], I),
            "puzzle_moe_combine": ([P, P, P, I64, I, I, P, P, P], I),
            "puzzle_gather_rows": ([P, P, I64, I64, P, P], I),
            "puzzle_group_colsumsq_workspace_size": ([I, I64], SZ),
            "puzzle_group_colsumsq": ([P, P, I, I64, P, P, SZ, P], I),
            "puzzle_moe_calib_workspace_size": ([P, I64, I], SZ),
            "puzzle_moe_forward_calib": ([P, P, P, I64, I, I, P, P, P, P, P, SZ, I, P], I),
            "puzzle_quant_pack": ([P, P, P, P, P, I64, I64, P, P, P], I),
            "puzzle_quant_unpack": ([P, P, I, I64, I64, P, P], I),
            "puzzle_quant_gemv": ([P, P, I64, I64, P, I64, P, I64, P, P, P], I),
            "puzzle_ep_dispatch": ([P, P, P, I, P, I, I64, I64, I, I, P, P], I),
            "puzzle_ep_recv_plan": ([P, I, I, I64, I, P, P, P, P], I),
            "puzzle_ep_home_index": ([P, P, P, I, P, I, I64, I64, I, P, P, P], I),
            "puzzle_ep_peer_buffer_size": ([I, I64, I], SZ),
            "puzzle_ep_dispatch_peer": ([P, P, P, I, P, I, I, I64, I64, I, I, P, P, P], I),
            "puzzle_ep_wait_dispatch": ([P, I, I64, I, P, P], I),
            "puzzle_ep_recv_plan_peer": ([P, I, I, I64, I, P, P, P, P, P], I),
            "puzzle_ep_combine_peer": ([P, P, P, I, P, I, I64, I64, I, I, P, P, P, P, P], I),
            "puzzle_ep_return_peer": ([P, P, I, I, I, I64, I, P, P, P], I),
            "puzzle_ep_home_index_peer": ([P, P, P, I, P, I, I64, I64, I, I, P, P, P, P, P], I),
            "puzzle_ep_unique_id": ([P], I),
            "puzzle_ep_create": ([ctypes.POINTER(ctypes.c_void_p), I, I, P, I], I),
            "puzzle_ep_destroy": ([P], I),
            "puzzle_ep_partition": ([I, I, P, P], I),
            "puzzle_moe_forward_ep_workspace_size": ([P, P, P, I64, I], SZ),
            "puzzle_moe_forward_ep": ([P, P, P, P, P, I64, I64, I, I, P, P, P, SZ, I, P], I),
            "puzzle_moe_quant_workspace_size": ([P, I64, I], SZ),
            "puzzle_moe_forward_quant": ([P, P, P, I64, I, I, P, P, P, SZ, P], I),
            "puzzle_profile_begin": ([], I),
            "puzzle_profile_end": ([ctypes.c_char_p, SZ], I),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def _check(rc: int, where: str) -> None:
    if rc != PUZZLE_OK:
        lib = load_library()
        raise PuzzleError(rc, where, f"{lib.puzzle_status_string(rc).decode()}: {lib.puzzle_last_error().decode()}")


def _p(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libpuzzlemoe takes CUDA tensors only (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream: torch.cuda.Stream | None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _u16(t: torch.Tensor) -> torch.Tensor:
    """bf16 / int16 / uint16 tensors share one bit view."""
    if t.dtype in (torch.bfloat16, torch.int16, torch.uint16, torch.float16):
        return t
    raise TypeError(f"expected a 16-bit tensor, got {t.dtype}")


# ---------------------------------------------------------------------------- pack / unpack
def merge_pack(w_merged, m0, m1, s0, s1, out=None, stats=None, stream=None) -> torch.Tensor:
    """puzzle_merge_pack: f32 magnitudes + uint8 bit-planes -> packed words (int16 tensor)."""
    assert w_merged.dtype == torch.float32
    for t in (m0, m1, s0, s1):
        assert t.dtype == torch.uint8 and t.shape == w_merged.shape
    out = torch.empty(w_merged.shape, dtype=torch.int16, device=w_merged.device) if out is None else out
    _check(load_library().puzzle_merge_pack(_p(w_merged), _p(m0), _p(m1), _p(s0), _p(s1), w_merged.numel(),
                                            _p(out), _p(stats), _stream(stream)), "puzzle_merge_pack")
    return out


def unpack(packed, pos: int, out=None, stream=None) -> torch.Tensor:
    """puzzle_unpack: Algorithm 1 -> bf16 tensor of expert ``pos``."""
    packed = _u16(packed)
    out = torch.empty(packed.shape, dtype=torch.bfloat16, device=packed.device) if out is None else out
    _check(load_library().puzzle_unpack(_p(packed), int(pos), packed.numel(), _p(out), _stream(stream)),
           "puzzle_unpack")
    return out


def merge_experts_pack(w_i, w_j, norms_i, norms_j, tau_sim: float = 0.4, out=None, stats=None,
                       stream=None) -> torch.Tensor:
    """puzzle_merge_experts_pack: bf16 [B, rows, cols] x2 + f32 norms [B, cols] -> packed."""
    assert w_i.dtype == torch.bfloat16 and w_j.dtype == torch.bfloat16 and w_i.shape == w_j.shape
    shp = w_i.shape if w_i.dim() == 3 else (1, *w_i.shape)
    n_mats, rows, cols = shp
    assert norms_i.dtype == torch.float32 and norms_i.numel() == n_mats * cols
    assert norms_j.dtype == torch.float32 and norms_j.numel() == n_mats * cols
    out = torch.empty(w_i.shape, dtype=torch.int16, device=w_i.device) if out is None else out
    _check(load_library().puzzle_merge_experts_pack(_p(w_i), _p(w_j), _p(norms_i), _p(norms_j), n_mats, rows,
                                                    cols, ctypes.c_float(tau_sim), _p(out), _p(stats),
                                                    _stream(stream)), "puzzle_merge_experts_pack")
    return out


def new_stats(device="cuda") -> torch.Tensor:
    """Zeroed device puzzle_pack_stats (4 x u64 as int64)."""
    return torch.zeros(4, dtype=torch.int64, device=device)


# ---------------------------------------------------------------------------- MoE layer
class PackedMoELayer:
    """Device tensors of one packed MoE layer plus its C descriptor.

    w13: packed [P, 2, d_ff, d_model]; w2: packed [P, d_model, d_ff]; expert_slot: int32 [E],
    E <= 2P; pair_dense: None or uint8 [P] (1 = the slot holds one unmerged expert's bf16
    weights, position 0 only: the 25% ratio, reading R20)."""

    def __init__(self, w13: torch.Tensor, w2: torch.Tensor, expert_slot: torch.Tensor, pair_dense=None):
        P, two, f, d = w13.shape
        assert two == 2 and tuple(w2.shape) == (P, d, f), (w13.shape, w2.shape)
        assert expert_slot.dtype == torch.int32 and 1 <= expert_slot.numel() <= 2 * P
        assert pair_dense is None or (pair_dense.dtype == torch.uint8 and pair_dense.numel() == P)
        self.w13, self.w2, self.expert_slot = _u16(w13).contiguous(), _u16(w2).contiguous(), expert_slot.contiguous()
        self.pair_dense = None if pair_dense is None else pair_dense.contiguous()
        self.n_pairs, self.n_experts, self.d_model, self.d_ff = P, expert_slot.numel(), d, f
        self.desc = MoELayerDesc(self.n_experts, P, d, f, self.w13.data_ptr(), self.w2.data_ptr(),
                                 self.expert_slot.data_ptr(),
                                 None if self.pair_dense is None else self.pair_dense.data_ptr())
        self._ws = None

    @property
    def packed_bytes(self) -> int:
        return self.w13.numel() * 2 + self.w2.numel() * 2

    def workspace_size(self, max_tokens: int, top_k: int) -> int:
        return int(load_library().puzzle_moe_workspace_size(ctypes.byref(self.desc), int(max_tokens), int(top_k)))

    def workspace(self, max_tokens: int, top_k: int) -> torch.Tensor:
        need = self.workspace_size(max_tokens, top_k)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.w13.device)
        return self._ws

    def forward(self, hidden, router_logits, top_k: int, renormalize: bool, residual=None, out=None,
                path: int = PATH_AUTO, workspace=None, stream=None) -> torch.Tensor:
        """puzzle_moe_forward_ex: bf16 [T, d] hidden, f32 [T, E] logits -> bf16 [T, d]."""
        T = hidden.shape[0]
        assert hidden.dtype == torch.bfloat16 and router_logits.dtype == torch.float32
        out = torch.empty_like(hidden) if out is None else out
        ws = self.workspace(T, top_k) if workspace is None else workspace
        _check(load_library().puzzle_moe_forward_ex(
            ctypes.byref(self.desc), _p(hidden), _p(router_logits), T, int(top_k), int(bool(renormalize)),
            _p(residual), _p(out), _p(ws), ws.numel(), int(path), _stream(stream)), "puzzle_moe_forward")
        return out

    __call__ = forward

    def forward_calib(self, hidden, router_logits, top_k: int, renormalize: bool, sumsq_x=None, sumsq_h=None,
                      residual=None, out=None, path: int = PATH_AUTO, stream=None) -> torch.Tensor:
        """puzzle_moe_forward_calib (NEXT-4): the forward, plus f64 per-bucket column sums of
        squares of x ([2P, d_model]) and of the SwiGLU rows ([2P, d_ff]) ACCUMULATED into
        sumsq_x / sumsq_h (either may be None)."""
        T = hidden.shape[0]
        assert hidden.dtype == torch.bfloat16 and router_logits.dtype == torch.float32
        for t, cols in ((sumsq_x, self.d_model), (sumsq_h, self.d_ff)):
            assert t is None or (t.dtype == torch.float64 and tuple(t.shape) == (2 * self.n_pairs, cols))
        out = torch.empty_like(hidden) if out is None else out
        need = int(load_library().puzzle_moe_calib_workspace_size(ctypes.byref(self.desc), T, int(top_k)))
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=hidden.device)
        _check(load_library().puzzle_moe_forward_calib(
            ctypes.byref(self.desc), _p(hidden), _p(router_logits), T, int(top_k), int(bool(renormalize)),
            _p(residual), _p(out), _p(sumsq_x), _p(sumsq_h), _p(ws), ws.numel(), int(path), _stream(stream)),
            "puzzle_moe_forward_calib")
        return out

    def route(self, router_logits, top_k: int, renormalize: bool, stream=None):
        """puzzle_moe_route -> (topk_idx, topk_gate, bucket_off, assign_token, assign_of)."""
        return _route(self.desc, self.n_pairs, router_logits, top_k, renormalize, stream)

    def experts(self, x_rows, bucket_off, y_rows=None, path: int = PATH_AUTO, workspace=None, stream=None):
        """puzzle_moe_experts: grouped bf16 rows -> unweighted f32 expert outputs."""
        n = x_rows.shape[0]
        y_rows = torch.empty((n, self.d_model), dtype=torch.float32, device=x_rows.device) if y_rows is None else y_rows
        if workspace is None:
            need = int(load_library().puzzle_moe_experts_workspace_size(ctypes.byref(self.desc), n))
            workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=x_rows.device)
        _check(load_library().puzzle_moe_experts(ctypes.byref(self.desc), _p(x_rows), _p(bucket_off), n,
                                                 _p(y_rows), _p(workspace), workspace.numel(), int(path),
                                                 _stream(stream)), "puzzle_moe_experts")
        return y_rows


class QuantLayerDesc(ctypes.Structure):
    """puzzle_moe_quant_layer."""
    _fields_ = [("n_experts", ctypes.c_int32), ("n_pairs", ctypes.c_int32), ("d_model", ctypes.c_int32),
                ("d_ff", ctypes.c_int32), ("w13_codes", ctypes.c_void_p), ("w13_scales", ctypes.c_void_p),
                ("w2_codes", ctypes.c_void_p), ("w2_scales", ctypes.c_void_p), ("expert_slot", ctypes.c_void_p)]


class QuantMoELayer:
    """NEXT-3: one MoE layer in the quantised weight class (puzzle_moe_forward_quant).

    w13_codes u8 [P, 2, d_ff, d_model], w13_scales f32 [P, 2, d_ff, d_model/128], w2_codes u8
    [P, d_model, d_ff], w2_scales f32 [P, d_model, d_ff/128] (puzzle_quant_pack's outputs per
    projection), expert_slot int32 [E]."""

    def __init__(self, w13_codes, w13_scales, w2_codes, w2_scales, expert_slot):
        P, two, f, d = w13_codes.shape
        assert two == 2 and w13_codes.dtype == torch.uint8 and w2_codes.dtype == torch.uint8
        assert tuple(w2_codes.shape) == (P, d, f) and tuple(w13_scales.shape) == (P, 2, f, d // 128)
        assert tuple(w2_scales.shape) == (P, d, f // 128) and w13_scales.dtype == torch.float32
        self.tensors = [t.contiguous() for t in (w13_codes, w13_scales, w2_codes, w2_scales, expert_slot)]
        self.n_pairs, self.n_experts, self.d_model, self.d_ff = P, expert_slot.numel(), d, f
        self.desc = QuantLayerDesc(self.n_experts, P, d, f, *[t.data_ptr() for t in self.tensors])
        self._ws = None

    @property
    def quant_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.tensors[:4])

    def workspace(self, max_tokens: int, top_k: int) -> torch.Tensor:
        need = int(load_library().puzzle_moe_quant_workspace_size(ctypes.byref(self.desc), int(max_tokens), int(top_k)))
        if need == 0:
            raise PuzzleError(1, "puzzle_moe_quant_workspace_size", "invalid layer")
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.tensors[0].device)
        return self._ws

    def forward(self, hidden, router_logits, top_k: int, renormalize: bool, residual=None, out=None, workspace=None,
                stream=None) -> torch.Tensor:
        T = hidden.shape[0]
        out = torch.empty_like(hidden) if out is None else out
        ws = self.workspace(T, top_k) if workspace is None else workspace
        _check(load_library().puzzle_moe_forward_quant(
            ctypes.byref(self.desc), _p(hidden), _p(router_logits), T, int(top_k), int(bool(renormalize)),
            _p(residual), _p(out), _p(ws), ws.numel(), _stream(stream)), "puzzle_moe_forward_quant")
        return out


class RoutingLayer:
    """Routing-only view of a layer for expert parallelism: GLOBAL n_experts / n_pairs /
    expert_slot (puzzle_moe_route reads nothing else); `anchor` is any 16-byte aligned 16-bit
    device tensor standing in for the weight pointers, which routing never dereferences."""

    def __init__(self, n_pairs: int, d_model: int, d_ff: int, expert_slot: torch.Tensor, anchor: torch.Tensor):
        assert expert_slot.dtype == torch.int32 and 1 <= expert_slot.numel() <= 2 * n_pairs
        self.expert_slot, self.anchor = expert_slot.contiguous(), anchor
        self.n_pairs = n_pairs
        self.desc = MoELayerDesc(expert_slot.numel(), n_pairs, d_model, d_ff, anchor.data_ptr(), anchor.data_ptr(),
                                 self.expert_slot.data_ptr(), None)

    def route(self, router_logits, top_k: int, renormalize: bool, stream=None):
        return _route(self.desc, self.n_pairs, router_logits, top_k, renormalize, stream)


def _route(desc, n_pairs, router_logits, top_k, renormalize, stream=None):
    """puzzle_moe_route -> (topk_idx, topk_gate, bucket_off, assign_token, assign_of)."""
    T = router_logits.shape[0]
    dev = router_logits.device
    idx = torch.empty((T, top_k), dtype=torch.int32, device=dev)
    gate = torch.empty((T, top_k), dtype=torch.float32, device=dev)
    off = torch.empty(2 * n_pairs + 1, dtype=torch.int32, device=dev)
    tok = torch.empty(T * top_k, dtype=torch.int32, device=dev)
    aof = torch.empty(T * top_k, dtype=torch.int32, device=dev)
    need = int(load_library().puzzle_moe_route_workspace_size(ctypes.byref(desc)))
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
    _check(load_library().puzzle_moe_route(ctypes.byref(desc), _p(router_logits), T, int(top_k),
                                           int(bool(renormalize)), _p(idx), _p(gate), _p(off), _p(tok),
                                           _p(aof), _p(ws), ws.numel(), _stream(stream)), "puzzle_moe_route")
    return idx, gate, off, tok, aof


def moe_combine(y_rows, assign_of, topk_gate, residual=None, out=None, stream=None) -> torch.Tensor:
    T, k = topk_gate.shape
    d = y_rows.shape[1]
    out = torch.empty((T, d), dtype=torch.bfloat16, device=y_rows.device) if out is None else out
    _check(load_library().puzzle_moe_combine(_p(y_rows), _p(assign_of), _p(topk_gate), T, k, d, _p(residual),
                                             _p(out), _stream(stream)), "puzzle_moe_combine")
    return out


def gather_rows(src, index, out=None, stream=None) -> torch.Tensor:
    n = index.numel()
    out = torch.empty((n, src.shape[1]), dtype=src.dtype, device=src.device) if out is None else out
    _check(load_library().puzzle_gather_rows(_p(src), _p(index), n, src.shape[1], _p(out), _stream(stream)),
           "puzzle_gather_rows")
    return out


def _dest_pairs(dest_pairs):
    """[world][2] host int32 array -> ctypes pointer (kept alive by the returned array)."""
    import numpy as np
    a = np.ascontiguousarray(np.asarray(dest_pairs, dtype=np.int32).reshape(-1, 2))
    return a, a.ctypes.data_as(ctypes.c_void_p), a.shape[0]


def ep_dispatch(hidden, assign_token, bucket_off, n_pairs: int, dest_pairs, cap: int, lb_max: int,
                send_rows=None, stream=None):
    """puzzle_ep_dispatch -> send_rows [world*(cap+1)][d] (per destination: cap row slots, then the
    header row whose first 4*lb_max bytes are the int32 bucket counts)."""
    arr, dp, world = _dest_pairs(dest_pairs)
    d = hidden.shape[1]
    if send_rows is None:
        send_rows = torch.empty((world * (cap + 1), d), dtype=hidden.dtype, device=hidden.device)
    _check(load_library().puzzle_ep_dispatch(_p(hidden), _p(assign_token), _p(bucket_off), int(n_pairs), dp, world,
                                             assign_token.numel(), int(cap), int(lb_max), d, _p(send_rows),
                                             _stream(stream)), "puzzle_ep_dispatch")
    return send_rows


def ep_header_counts(rows, world: int, cap: int, lb: int):
    """The int32 bucket counts carried by the header rows of a [world*(cap+1)][d] region buffer
    (a view for inspection / tests)."""
    return rows.view(world, cap + 1, -1)[:, cap].contiguous().view(torch.int32)[:, :lb]


def ep_recv_plan(recv_rows, world: int, n_local_buckets: int, cap: int, stream=None):
    """puzzle_ep_recv_plan -> (local_off [lb+1], gather_idx [world*cap], return_idx [world*(cap+1)])."""
    dev = recv_rows.device
    local_off = torch.empty(n_local_buckets + 1, dtype=torch.int32, device=dev)
    gidx = torch.empty(max(world * cap, 1), dtype=torch.int32, device=dev)[:world * cap]
    ridx = torch.empty(world * (cap + 1), dtype=torch.int32, device=dev)
    _check(load_library().puzzle_ep_recv_plan(_p(recv_rows), int(world), int(n_local_buckets), int(cap),
                                              recv_rows.shape[1], _p(local_off), _p(gidx), _p(ridx), _stream(stream)),
           "puzzle_ep_recv_plan")
    return local_off, gidx, ridx


def ep_home_index(assign_of, topk_gate, bucket_off, n_pairs: int, dest_pairs, slices: int, cap: int, stream=None):
    """puzzle_ep_home_index -> (aof_s [T*k*S] i32, gate_s [T][k*S] f32)."""
    arr, dp, world = _dest_pairs(dest_pairs)
    T, k = topk_gate.shape
    dev = topk_gate.device
    aof_s = torch.empty(T * k * slices, dtype=torch.int32, device=dev)
    gate_s = torch.empty((T, k * slices), dtype=torch.float32, device=dev)
    _check(load_library().puzzle_ep_home_index(_p(assign_of), _p(topk_gate), _p(bucket_off), int(n_pairs), dp, world,
                                               int(cap), T, k, _p(aof_s), _p(gate_s), _stream(stream)),
           "puzzle_ep_home_index")
    return aof_s, gate_s


class EpPeerBuffer:
    """This rank's peer buffer (puzzle_ep_peer_buffer_size bytes) + its view of every peer's
    buffer address + the private step state. `buffer` may come from torch symmetric memory
    (multi-GPU) or be a plain device tensor (peers in one process, tests)."""

    def __init__(self, buffer: torch.Tensor, peer_ptrs, world: int, cap: int, d_model: int):
        import numpy as np
        need = int(load_library().puzzle_ep_peer_buffer_size(world, cap, d_model))
        if buffer.numel() * buffer.element_size() < need:
            raise ValueError(f"peer buffer of {buffer.numel()} bytes < {need}")
        self.buffer, self.world, self.cap, self.d = buffer, world, cap, d_model
        self.peers = np.ascontiguousarray(np.asarray(peer_ptrs, dtype=np.uint64))
        assert self.peers.size == world
        self.state = torch.zeros(8, dtype=torch.int32, device=buffer.device)
        R = cap + 1
        self.recv_x = buffer.view(torch.uint8)[:world * R * d_model * 2].view(torch.bfloat16).view(world * R, d_model)
        off_y = (world * R * d_model * 2 + 255) // 256 * 256
        self.recv_y = buffer.view(torch.uint8)[off_y:off_y + world * R * d_model * 4].view(torch.float32).view(world * R, d_model)

    def wait_timeouts(self) -> int:
        """Cross-rank waits that gave up (state[4]); nonzero = some step's outputs are invalid."""
        return int(self.state[4].item())

    @staticmethod
    def size(world: int, cap: int, d_model: int) -> int:
        return int(load_library().puzzle_ep_peer_buffer_size(world, cap, d_model))

    def _peers(self):
        return self.peers.ctypes.data_as(ctypes.c_void_p)


def ep_dispatch_peer(hidden, assign_token, bucket_off, n_pairs: int, dest_pairs, rank: int, pb: EpPeerBuffer,
                     lb_max: int, stream=None):
    arr, dp, world = _dest_pairs(dest_pairs)
    _check(load_library().puzzle_ep_dispatch_peer(_p(hidden), _p(assign_token), _p(bucket_off), int(n_pairs), dp, world,
                                                  int(rank), assign_token.numel(), pb.cap, int(lb_max), pb.d,
                                                  pb._peers(), _p(pb.state), _stream(stream)), "puzzle_ep_dispatch_peer")


def ep_wait_dispatch(pb: EpPeerBuffer, stream=None):
    _check(load_library().puzzle_ep_wait_dispatch(_p(pb.buffer), pb.world, pb.cap, pb.d, _p(pb.state), _stream(stream)),
           "puzzle_ep_wait_dispatch")


def ep_recv_plan_peer(pb: "EpPeerBuffer", n_local_buckets: int, stream=None):
    """wait for this step's dispatch into pb, then puzzle_ep_recv_plan on pb.recv_x (one kernel)."""
    dev = pb.buffer.device
    world, cap = pb.world, pb.cap
    local_off = torch.empty(n_local_buckets + 1, dtype=torch.int32, device=dev)
    gidx = torch.empty(max(world * cap, 1), dtype=torch.int32, device=dev)[:world * cap]
    ridx = torch.empty(world * (cap + 1), dtype=torch.int32, device=dev)
    _check(load_library().puzzle_ep_recv_plan_peer(_p(pb.buffer), world, int(n_local_buckets), cap, pb.d,
                                                   _p(pb.state), _p(local_off), _p(gidx), _p(ridx), _stream(stream)),
           "puzzle_ep_recv_plan_peer")
    return local_off, gidx, ridx


def ep_return_peer(y_local, return_idx, rank: int, n_local_buckets: int, pb: EpPeerBuffer, stream=None):
    _check(load_library().puzzle_ep_return_peer(_p(y_local), _p(return_idx), pb.world, int(rank), int(n_local_buckets),
                                                pb.cap, pb.d,
                                                pb._peers(), _p(pb.state), _stream(stream)), "puzzle_ep_return_peer")


def ep_combine_peer(assign_of, topk_gate, bucket_off, n_pairs: int, dest_pairs, pb: EpPeerBuffer, residual=None,
                    out=None, stream=None):
    """puzzle_ep_combine_peer -> out [T][d] bf16 (waits for the returns; advances the step)."""
    arr, dp, world = _dest_pairs(dest_pairs)
    T, k = topk_gate.shape
    out = torch.empty((T, pb.d), dtype=torch.bfloat16, device=topk_gate.device) if out is None else out
    _check(load_library().puzzle_ep_combine_peer(_p(assign_of), _p(topk_gate), _p(bucket_off), int(n_pairs), dp, world,
                                                 pb.cap, T, k, pb.d, _p(pb.buffer), _p(residual), _p(out),
                                                 _p(pb.state), _stream(stream)), "puzzle_ep_combine_peer")
    return out


def ep_home_index_peer(assign_of, topk_gate, bucket_off, n_pairs: int, dest_pairs, slices: int, pb: EpPeerBuffer,
                       stream=None):
    arr, dp, world = _dest_pairs(dest_pairs)
    T, k = topk_gate.shape
    dev = topk_gate.device
    aof_s = torch.empty(max(T * k * slices, 1), dtype=torch.int32, device=dev)[:T * k * slices]
    gate_s = torch.empty((T, k * slices), dtype=torch.float32, device=dev)
    _check(load_library().puzzle_ep_home_index_peer(_p(assign_of), _p(topk_gate), _p(bucket_off), int(n_pairs), dp,
                                                    world, pb.cap, T, k, pb.d, _p(pb.buffer), _p(aof_s), _p(gate_s),
                                                    _p(pb.state), _stream(stream)), "puzzle_ep_home_index_peer")
    return aof_s, gate_s


class profile_window:
    """Context manager over puzzle_profile_begin/end: per-kernel CUDA-event timings of every
    library launch inside the window, recorded on the launching stream.
    After exit, ``.kernels`` maps kernel name -> (launches, total_ms)."""

    def __enter__(self):
        _check(load_library().puzzle_profile_begin(), "puzzle_profile_begin")
        self.kernels = {}
        return self

    def __exit__(self, *exc):
        buf = ctypes.create_string_buffer(1 << 16)
        _check(load_library().puzzle_profile_end(buf, len(buf)), "puzzle_profile_end")
        for line in buf.value.decode().splitlines():
            name, n, ms = line.split()
            self.kernels[name] = (int(n), float(ms))
        return False


def group_colsumsq(rows, group_off, sumsq, stream=None) -> torch.Tensor:
    """puzzle_group_colsumsq (NEXT-4): sumsq[g] += column sums of squares of bf16 rows
    [group_off[g], group_off[g+1]); sumsq f64 [G, cols] (accumulated, returned)."""
    rows = _u16(rows)
    G = group_off.numel() - 1
    cols = rows.shape[-1]
    assert group_off.dtype == torch.int32 and sumsq.dtype == torch.float64 and tuple(sumsq.shape) == (G, cols)
    need = int(load_library().puzzle_group_colsumsq_workspace_size(G, cols))
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=rows.device)
    _check(load_library().puzzle_group_colsumsq(_p(rows), _p(group_off), G, cols, _p(sumsq), _p(ws), ws.numel(),
                                                _stream(stream)), "puzzle_group_colsumsq")
    return sumsq


def quant_pack(w_merged, m0, m1, s0, s1, stream=None):
    """puzzle_quant_pack (NEXT-3): f32 [rows, cols] magnitudes + uint8 bit-planes -> (uint8
    codes [rows, cols], f32 scales [rows, cols / 128])."""
    assert w_merged.dtype == torch.float32 and w_merged.dim() == 2
    rows, cols = w_merged.shape
    for t in (m0, m1, s0, s1):
        assert t.dtype == torch.uint8 and t.shape == w_merged.shape
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=w_merged.device)
    scales = torch.empty((rows, max(cols // 128, 0)), dtype=torch.float32, device=w_merged.device)
    _check(load_library().puzzle_quant_pack(_p(w_merged), _p(m0), _p(m1), _p(s0), _p(s1), rows, cols, _p(codes),
                                            _p(scales), _stream(stream)), "puzzle_quant_pack")
    return codes, scales


def quant_unpack(codes, scales, pos: int, stream=None) -> torch.Tensor:
    """puzzle_quant_unpack: dequantised bf16 [rows, cols] of expert ``pos``."""
    assert codes.dtype == torch.uint8 and codes.dim() == 2 and scales.dtype == torch.float32
    rows, cols = codes.shape
    out = torch.empty((rows, cols), dtype=torch.bfloat16, device=codes.device)
    _check(load_library().puzzle_quant_unpack(_p(codes), _p(scales), int(pos), rows, cols, _p(out), _stream(stream)),
           "puzzle_quant_unpack")
    return out


def quant_gemv(codes, scales, x_i, x_j, stream=None):
    """puzzle_quant_gemv (NEXT-3): both experts of one quantised merged pair on their routed
    tokens, x_i / x_j bf16 [n, cols] -> (y_i, y_j) f32 [n, rows]."""
    assert codes.dtype == torch.uint8 and codes.dim() == 2 and scales.dtype == torch.float32
    rows, cols = codes.shape
    for x in (x_i, x_j):
        assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.shape[1] == cols and x.is_contiguous()
    y_i = torch.empty((x_i.shape[0], rows), dtype=torch.float32, device=codes.device)
    y_j = torch.empty((x_j.shape[0], rows), dtype=torch.float32, device=codes.device)
    _check(load_library().puzzle_quant_gemv(_p(codes), _p(scales), rows, cols, _p(x_i), x_i.shape[0], _p(x_j),
                                            x_j.shape[0], _p(y_i), _p(y_j), _stream(stream)), "puzzle_quant_gemv")
    return y_i, y_j


# ---- expert parallelism behind the C ABI (puzzle_ep_*, puzzle_moe_forward_ep) ----
def ep_unique_id() -> bytes:
    """puzzle_ep_unique_id: the 128-byte NCCL bootstrap id (rank 0; broadcast it to the others)."""
    buf = ctypes.create_string_buffer(EP_UNIQUE_ID_BYTES)
    _check(load_library().puzzle_ep_unique_id(buf), "puzzle_ep_unique_id")
    return buf.raw


def ep_partition(world: int, n_pairs: int):
    """puzzle_ep_partition -> (dest_pairs int32 [world][2] numpy, slices)."""
    import numpy as np
    dest = np.zeros((world, 2), np.int32)
    slices = ctypes.c_int(0)
    _check(load_library().puzzle_ep_partition(int(world), int(n_pairs), dest.ctypes.data_as(ctypes.c_void_p),
                                              ctypes.byref(slices)), "puzzle_ep_partition")
    return dest, int(slices.value)


class EpComm:
    """A C-owned NCCL communicator (puzzle_ep_create / puzzle_ep_destroy) and the expert-parallel
    layer over it (puzzle_moe_forward_ep). Collective: every rank constructs it with the same
    unique id (from ep_unique_id() on rank 0, broadcast by the caller)."""

    def __init__(self, world: int, rank: int, unique_id: bytes, device: int):
        assert len(unique_id) == EP_UNIQUE_ID_BYTES
        self.world, self.rank, self.device = world, rank, device
        h = ctypes.c_void_p(None)
        _check(load_library().puzzle_ep_create(ctypes.byref(h), int(world), int(rank), unique_id, int(device)),
               "puzzle_ep_create")
        self.handle = h
        self._ws = None

    def close(self):
        if self.handle:
            _check(load_library().puzzle_ep_destroy(self.handle), "puzzle_ep_destroy")
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def workspace(self, route_layer, local_layer, cap_tokens: int, top_k: int) -> torch.Tensor:
        need = int(load_library().puzzle_moe_forward_ep_workspace_size(
            self.handle, ctypes.byref(route_layer.desc), ctypes.byref(local_layer.desc), int(cap_tokens), int(top_k)))
        if need == 0:
            raise PuzzleError(1, "puzzle_moe_forward_ep_workspace_size", "invalid arguments")
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=torch.device("cuda", self.device))
        return self._ws

    def forward(self, route_layer, local_layer, hidden, router_logits, top_k: int, renormalize: bool,
                cap_tokens: int | None = None, residual=None, out=None, path: int = PATH_AUTO, workspace=None,
                stream=None) -> torch.Tensor:
        """puzzle_moe_forward_ep: this rank's tokens through the expert-parallel layer."""
        T = hidden.shape[0]
        cap_tokens = T if cap_tokens is None else int(cap_tokens)
        out = torch.empty_like(hidden) if out is None else out
        ws = self.workspace(route_layer, local_layer, cap_tokens, top_k) if workspace is None else workspace
        _check(load_library().puzzle_moe_forward_ep(
            self.handle, ctypes.byref(route_layer.desc), ctypes.byref(local_layer.desc), _p(hidden),
            _p(router_logits), T, cap_tokens, int(top_k), int(bool(renormalize)), _p(residual), _p(out), _p(ws),
            ws.numel(), int(path), _stream(stream)), "puzzle_moe_forward_ep")
        return out
