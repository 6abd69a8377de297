"""PuzzleMoE CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. It shares no code with the CUDA
path (``paper_2511_04805_b200``); the product path never imports it.

The arithmetic lives in ``puzzle_oracle.c`` (plain C, f32 merge per S:188, f64 FFN);
this module only marshals numpy arrays through ctypes. ``analysis`` holds the
Appendix B closed form.

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "puzzle_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

GCC_FLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            I = ctypes.c_int
            lib.oracle_bf16_round.argtypes = [P, I64, P]
            lib.oracle_merge.argtypes = [P, P, P, P, I64, I64, ctypes.c_float, P, P, P, P, P, P, P]
            lib.oracle_pack.argtypes = [P, P, P, P, P, I64, P, P]
            lib.oracle_unpack.argtypes = [P, I, I64, P]
            lib.oracle_route.argtypes = [P, I64, I, I, I, P, P]
            lib.oracle_moe_forward.argtypes = [P, P, P, P, I, I, I, P, P, I64, I, I, I, P, P]
            lib.oracle_expert_ffn.argtypes = [P, P, I, I, I, I, I, P, I64, P]
            lib.oracle_expert_ffn.restype = I
            lib.oracle_calib_sumsq.argtypes = [P, P, P, I, I, I, P, P, I64, I, I, I, P, P]
            lib.oracle_quant_pack.argtypes = [P, P, P, P, P, I64, I64, P, P]
            lib.oracle_quant_pack.restype = I
            lib.oracle_quant_unpack.argtypes = [P, P, I, I64, I64, P]
            lib.oracle_quant_unpack.restype = I
            lib.oracle_calib_sumsq.restype = I
            lib.oracle_num_threads.restype = I
            lib.oracle_set_num_threads.argtypes = [I]
            for name in ("oracle_bf16_round", "oracle_merge", "oracle_pack", "oracle_unpack",
                         "oracle_route", "oracle_moe_forward"):
                getattr(lib, name).restype = I
            _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags.c_contiguous, "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def bf16_round(x) -> np.ndarray:
    """f32 -> bf16 bits (uint16), round-to-nearest-even (reading R3)."""
    x = _c(x, np.float32)
    out = np.empty(x.shape, np.uint16)
    _load().oracle_bf16_round(_ptr(x), x.size, _ptr(out))
    return out


def bf16_bits_to_f32(h) -> np.ndarray:
    h = _c(h, np.uint16)
    return (h.astype(np.uint32) << 16).view(np.float32)


def merge(w_i, w_j, norms_i, norms_j, tau_sim: float = 0.4) -> dict:
    """Eq. 1-7 for one linear slot of one expert pair.

    w_i, w_j: (rows, cols) = (out, in); norms: (cols,). Returns a dict with
    w_merged (f32), m_sim, m_sal_i, m_i, m_j, s_i, s_j (uint8 0/1)."""
    w_i = _c(w_i, np.float32)
    w_j = _c(w_j, np.float32)
    if w_i.shape != w_j.shape or w_i.ndim != 2:
        raise ValueError("ShapeMismatch: W_i and W_j must share one 2-D shape")
    rows, cols = w_i.shape
    n_i = _c(norms_i, np.float32).reshape(-1)
    n_j = _c(norms_j, np.float32).reshape(-1)
    if n_i.size != cols or n_j.size != cols:
        raise ValueError("ShapeMismatch: norms must have length in_features")
    out = {"w_merged": np.empty((rows, cols), np.float32)}
    for key in ("m_sim", "m_sal_i", "m_i", "m_j", "s_i", "s_j"):
        out[key] = np.empty((rows, cols), np.uint8)
    rc = _load().oracle_merge(_ptr(w_i), _ptr(w_j), _ptr(n_i), _ptr(n_j), rows, cols,
                              ctypes.c_float(tau_sim), _ptr(out["w_merged"]), _ptr(out["m_sim"]),
                              _ptr(out["m_sal_i"]), _ptr(out["m_i"]), _ptr(out["m_j"]),
                              _ptr(out["s_i"]), _ptr(out["s_j"]))
    if rc != 0:
        raise ValueError("InvalidThreshold: tau_sim must lie in [0, 1]")
    out["m_sal_j"] = (1 - out["m_sal_i"]).astype(np.uint8)
    return out


def pack(w_merged, m0, m1, s0, s1) -> tuple[np.ndarray, np.ndarray]:
    """(a1) merged magnitude + 4 bit-planes -> packed uint16 words, and stats
    [rounded_up(e<112), saturated(e>143), nonfinite, negative]."""
    w = _c(w_merged, np.float32)
    planes = [_c(p, np.uint8) for p in (m0, m1, s0, s1)]
    for p in planes:
        if p.shape != w.shape:
            raise ValueError("ShapeMismatch: all five merge artifacts must share one shape")
    out = np.empty(w.shape, np.uint16)
    stats = np.zeros(4, np.uint64)
    _load().oracle_pack(_ptr(w), _ptr(planes[0]), _ptr(planes[1]), _ptr(planes[2]),
                        _ptr(planes[3]), w.size, _ptr(out), _ptr(stats))
    return out, stats


def pack_artifacts(art: dict) -> tuple[np.ndarray, np.ndarray]:
    """pos 0 = expert i, pos 1 = expert j (reading R7)."""
    return pack(art["w_merged"], art["m_i"], art["m_j"], art["s_i"], art["s_j"])


def unpack(packed, pos: int) -> np.ndarray:
    """(a2) Algorithm 1 over a whole tensor -> bf16 bits of expert ``pos``."""
    p = _c(packed, np.uint16)
    out = np.empty(p.shape, np.uint16)
    if _load().oracle_unpack(_ptr(p), int(pos), p.size, _ptr(out)) != 0:
        raise ValueError("expert_pos must be 0 or 1")
    return out


def route(logits, k: int, renormalize: bool) -> tuple[np.ndarray, np.ndarray]:
    """Top-k expert ids (ties -> lower index) and f64 gates per token."""
    lg = _c(logits, np.float32)
    T, E = lg.shape
    idx = np.empty((T, k), np.int32)
    gate = np.empty((T, k), np.float64)
    if _load().oracle_route(_ptr(lg), T, E, k, int(bool(renormalize)), _ptr(idx), _ptr(gate)) != 0:
        raise ValueError("bad routing arguments")
    return idx, gate


def moe_forward(w13, w2, expert_slot, hidden_bits, logits, k: int, renormalize: bool,
                residual_bits=None, pair_dense=None) -> np.ndarray:
    """f64 [T, d] = residual + sum_j gate_j * FFN_{e_j}(x) over packed pairs.

    w13: uint16 [P, 2, f, d]; w2: uint16 [P, d, f]; expert_slot: int32 [E]
    (2*pair+pos, E <= 2P, distinct); hidden_bits / residual_bits: uint16 bf16 bits
    [T, d]; logits: f32 [T, E]; pair_dense: None or uint8 [P], 1 = the slot holds one
    unmerged expert's plain bf16 weights at position 0 (25% ratio, reading R20)."""
    w13 = _c(w13, np.uint16)
    w2 = _c(w2, np.uint16)
    P, two, f, d = w13.shape
    assert two == 2 and w2.shape == (P, d, f), (w13.shape, w2.shape)
    slot = _c(expert_slot, np.int32)
    hb = _c(hidden_bits, np.uint16)
    lg = _c(logits, np.float32)
    T = hb.shape[0]
    E = lg.shape[1]
    assert hb.shape == (T, d) and lg.shape == (T, E) and slot.shape == (E,)
    res = None if residual_bits is None else _c(residual_bits, np.uint16)
    dense = None if pair_dense is None else _c(pair_dense, np.uint8).reshape(-1)
    assert dense is None or dense.shape == (P,)
    out = np.empty((T, d), np.float64)
    rc = _load().oracle_moe_forward(_ptr(w13), _ptr(w2), _ptr(slot), _ptr(dense), P, d, f, _ptr(hb), _ptr(lg),
                                    T, E, k, int(bool(renormalize)), _ptr(res), _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_moe_forward failed rc={rc}")
    return out


def expert_ffn(w13, w2, pair: int, pos: int, x_bits, dense: bool = False) -> np.ndarray:
    """f64 [n, d] = W2_pos (silu(W1_pos x) * (W3_pos x)) for rows already routed to expert
    (pair, pos); no gate, no residual. dense: the slot holds plain bf16 weights (R20)."""
    w13 = _c(w13, np.uint16)
    w2 = _c(w2, np.uint16)
    P, two, f, d = w13.shape
    xb = _c(x_bits, np.uint16).reshape(-1, d)
    y = np.empty((xb.shape[0], d), np.float64)
    if _load().oracle_expert_ffn(_ptr(w13), _ptr(w2), int(pair), int(pos), int(bool(dense)), d, f, _ptr(xb), xb.shape[0], _ptr(y)) != 0:
        raise ValueError("bad expert position")
    return y


def calib_sumsq(w13, expert_slot, hidden_bits, logits, k: int, renormalize: bool, pair_dense=None,
                want_h: bool = True) -> tuple[np.ndarray, np.ndarray | None]:
    """NEXT-4, Eq. 4 statistics: per slot b, f64 sums of squares per input
    column of the activations routed to it -- x for W1/W3 ([2P, d]) and the SwiGLU
    intermediate h for W2 ([2P, f]); ||X||_2 = sqrt of these."""
    w13 = _c(w13, np.uint16)
    P, two, f, d = w13.shape
    slot = _c(expert_slot, np.int32)
    hb = _c(hidden_bits, np.uint16)
    lg = _c(logits, np.float32)
    T, E = lg.shape
    assert hb.shape == (T, d) and slot.shape == (E,)
    dense = None if pair_dense is None else _c(pair_dense, np.uint8).reshape(-1)
    sx = np.empty((2 * P, d), np.float64)
    sh = np.empty((2 * P, f), np.float64) if want_h else None
    rc = _load().oracle_calib_sumsq(_ptr(w13), _ptr(slot), _ptr(dense), P, d, f, _ptr(hb), _ptr(lg), T, E, k,
                                    int(bool(renormalize)), _ptr(sx), _ptr(sh))
    if rc != 0:
        raise ValueError(f"oracle_calib_sumsq failed rc={rc}")
    return sx, sh


def group_colsumsq(rows_bits, group_off) -> np.ndarray:
    """NEXT-4 building block, the plain definition: f64 [G, cols] with row g = the column sums
    of squares of the bf16 rows [group_off[g], group_off[g+1])."""
    x = bf16_bits_to_f32(_c(rows_bits, np.uint16)).astype(np.float64)
    off = np.asarray(group_off, np.int64)
    out = np.zeros((off.size - 1, x.shape[1]), np.float64)
    for g in range(off.size - 1):
        for r in range(off[g], off[g + 1]):
            out[g] += x[r] * x[r]
    return out


def quant_pack(w_merged, m0, m1, s0, s1) -> tuple[np.ndarray, np.ndarray]:
    """NEXT-3 (Appendix A.3; readings R21-R23): merged magnitudes [rows, cols]
    (cols % 128 == 0) + bit-planes -> codes u8 [rows, cols] (S_i S_j M_i M_j 0 q2 q1 q0) and
    f32 scales [rows, cols / 128] (max / 7 per group of 128, 1 for an all-zero group)."""
    w = _c(w_merged, np.float32)
    rows, cols = w.shape
    planes = [_c(p, np.uint8) for p in (m0, m1, s0, s1)]
    codes = np.empty((rows, cols), np.uint8)
    scales = np.empty((rows, cols // 128), np.float32)
    if _load().oracle_quant_pack(_ptr(w), *[_ptr(p) for p in planes], rows, cols, _ptr(codes), _ptr(scales)) != 0:
        raise ValueError("quant_pack: cols must be a multiple of 128")
    return codes, scales


def quant_unpack(codes, scales, pos: int) -> np.ndarray:
    """Dequantised bf16 bits of expert `pos`: (-1)^S * M * bf16_rne(code * scale)."""
    codes = _c(codes, np.uint8)
    scales = _c(scales, np.float32)
    rows, cols = codes.shape
    out = np.empty((rows, cols), np.uint16)
    if _load().oracle_quant_unpack(_ptr(codes), _ptr(scales), int(pos), rows, cols, _ptr(out)) != 0:
        raise ValueError("quant_unpack: bad position or shape")
    return out


def quant_gemv(codes, scales, x_i, x_j) -> tuple[np.ndarray, np.ndarray]:
    """NEXT-3 expert GEMV over the quantised format (Appendix A.3; reading R23:
    the dequantised Ŵ_pos is the bf16 operand of the expert matmul, as Algorithm 1's output
    is). The tokens routed to expert i of the pair (x_i, bf16 bits [n_i, cols]) see Ŵ_0, those
    routed to j (x_j [n_j, cols]) see Ŵ_1: y_i = x_i Ŵ_0^T, y_j = x_j Ŵ_1^T, in f64
    ([n_i, rows], [n_j, rows])."""
    def bf16(bits):
        return (np.asarray(bits, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    w0 = bf16(quant_unpack(codes, scales, 0))
    w1 = bf16(quant_unpack(codes, scales, 1))
    return bf16(x_i) @ w0.T, bf16(x_j) @ w1.T
