"""GPU timeline of one CUDA-graph replay of the forward (needs a PZ_TRACE build of route.cu and
gemv_tc.cu: python scripts/build_variant.py trace route.cu,gemv_tc.cu -DPZ_TRACE=5; run with
PUZZLE_LIB=...). Prints each kernel's [first CTA start, pdl_wait return, last CTA end] in us
relative to the route kernel's start."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mixtral"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda:0")
layer, _ = bench.build_layer_gpu(pz, cfg, 1, dev)
hidden, logits = bench.make_inputs(cfg, T, 2, dev)
out = torch.empty_like(hidden)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, out=out)
lib = pz.load_library()
for name in ("puzzle_debug_rt", "puzzle_debug_cta", "puzzle_debug_wait"):
    getattr(lib, name).restype = ctypes.c_int
lib.puzzle_debug_rt.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
lib.puzzle_debug_cta.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
lib.puzzle_debug_wait.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
rt = np.zeros((4, 2), np.uint64)
cta = np.zeros((2, 1024, 4), np.uint64)
wt = np.zeros((2, 1024), np.uint64)
assert lib.puzzle_debug_rt(None, 0, 1) == 0
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    ev0.record(s)
    g.replay()
    ev1.record(s)
torch.cuda.synchronize()
assert lib.puzzle_debug_rt(rt.ctypes.data, rt.nbytes, 0) == 0
assert lib.puzzle_debug_cta(cta.ctypes.data, cta.nbytes) == 0
assert lib.puzzle_debug_wait(wt.ctypes.data, wt.nbytes) == 0
t0 = int(min(rt[0, 0], rt[3, 0]))
print(f"{cfg.name} T={T}: graph replay {ev0.elapsed_time(ev1) * 1e3:.1f} us (events)")
def us(x):
    return (int(x) - t0) / 1e3
if int(rt[3, 1]) > 0:
    print(f"  topk    start {us(rt[3,0]):7.2f}  end {us(rt[3,1]):7.2f}")
print(f"  route   start {us(rt[0,0]):7.2f}  end {us(rt[0,1]):7.2f}   (single-CTA route, or the decode scatter+gather)")
if int(rt[1, 1]) > 0:
    print(f"  gather  start {us(rt[1,0]):7.2f}  end {us(rt[1,1]):7.2f}")
for name, k in (("w13", 1), ("w2", 0)):
    v = cta[k]
    n = int((v[:, 3] > 0).sum())
    starts = v[:n, 0].astype(np.int64)
    waits = wt[k, :n].astype(np.int64)
    ends = v[:n, 3].astype(np.int64)
    print(f"  {name:6s}  start {(starts.min() - t0)/1e3:7.2f}  wait-ret min {(waits.min() - t0)/1e3:7.2f} "
          f"max {(waits.max() - t0)/1e3:7.2f}  end min {(ends.min() - t0)/1e3:7.2f} med {(np.median(ends) - t0)/1e3:7.2f} "
          f"max {(ends.max() - t0)/1e3:7.2f}   ({n} CTAs)")
print(f"  combine start {us(rt[2,0]):7.2f}  end {us(rt[2,1]):7.2f}")

if len(sys.argv) > 3:
    sm = np.zeros((2, 1024), np.uint32)
    lib.puzzle_debug_smid.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert lib.puzzle_debug_smid(sm.ctypes.data, sm.nbytes) == 0
    for name, k in (("w13", 1), ("w2", 0)):
        v = cta[k]
        n = int((v[:, 3] > 0).sum())
        dur = (v[:n, 3].astype(np.int64) - wt[k, :n].astype(np.int64)) / 1e3
        smid = sm[k, :n]
        print(f"{name}: duration after wait: mean {dur.mean():.1f} std {dur.std():.1f} min {dur.min():.1f} max {dur.max():.1f}")
        # per SM: the two CTAs on it
        per_sm = {}
        for i in range(n):
            per_sm.setdefault(int(smid[i]), []).append(float(dur[i]))
        sm_mean = np.array([np.mean(per_sm[s]) for s in sorted(per_sm)])
        print(f"  per-SM mean duration: min {sm_mean.min():.1f} max {sm_mean.max():.1f}; CTAs per SM "
              f"{sorted(set(len(x) for x in per_sm.values()))}")
        order = np.argsort(sm_mean)
        keys = sorted(per_sm)
        print("  slowest SMs:", [(keys[i], round(sm_mean[i], 1)) for i in order[-8:]])
        print("  fastest SMs:", [(keys[i], round(sm_mean[i], 1)) for i in order[:8]])
        # by CTA index halves
        print(f"  CTA idx < {n//2}: mean {dur[:n//2].mean():.1f}; >= : mean {dur[n//2:].mean():.1f}")
        # within-SM difference
        diffs = [abs(x[0] - x[1]) for x in per_sm.values() if len(x) == 2]
        print(f"  |CTA a - CTA b| on the same SM: mean {np.mean(diffs):.1f} max {np.max(diffs):.1f}")
        # dump durations in SM order for a correlation by GPC (SM id // 16 approx)
        gpc = {}
        for s_, d_ in per_sm.items():
            gpc.setdefault(s_ // 18, []).append(np.mean(d_))
        print("  by SM-id block of 18:", {k2: round(float(np.mean(v2)), 1) for k2, v2 in sorted(gpc.items())})

if os.environ.get("TIMELINE_DUMP"):
    sm = np.zeros((2, 1024), np.uint32)
    lib.puzzle_debug_smid.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert lib.puzzle_debug_smid(sm.ctypes.data, sm.nbytes) == 0
    red = np.zeros((2, 1024, 8), np.uint64)
    lib.puzzle_debug_red.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert lib.puzzle_debug_red(red.ctypes.data, red.nbytes) == 0
    np.savez(os.environ["TIMELINE_DUMP"], cta=cta, wt=wt, sm=sm, rt=rt, red=red,
             logits=logits.float().cpu().numpy(), slot=layer.expert_slot.cpu().numpy())
