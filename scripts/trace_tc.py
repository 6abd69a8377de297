"""Pipeline timeline of the prefill tcgen05 kernels (PZ_TRACE build of gemm_tc.cu:
python scripts/build_variant.py tctrace gemm_tc.cu -DPZ_TRACE=5; run with PUZZLE_LIB=...).
CTA 5 of the w13 kernel: per stage TMA issue (0), decode done (1), MMAs issued (2); per tile
epilogue start (3) / end (4). All CTAs of both kernels: start (after pdl_wait) / end."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "qwen15"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = torch.device("cuda:0")
layer, _ = bench.build_layer_gpu(pz, cfg, 1, dev)
hidden, logits = bench.make_inputs(cfg, T, 2, dev)
for _ in range(3):
    layer.forward(hidden, logits, cfg.top_k, cfg.renormalize)
torch.cuda.synchronize()
lib = pz.load_library()
ev = np.zeros((6, 4096), np.uint64)
cc = np.zeros((2, 1024, 2), np.uint64)
lib.puzzle_debug_tc.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t]
assert lib.puzzle_debug_tc(ev.ctypes.data, ev.nbytes, cc.ctypes.data, cc.nbytes) == 0
for name, k in (("w13", 1), ("w2", 0)):
    v = cc[k].astype(np.int64)
    n = int((v[:, 1] > 0).sum())
    v = v[:n]
    t0 = v[:, 0].min()
    d = (v[:, 1] - v[:, 0]) / 1e3
    print(f"{name}: {n} CTAs, start spread {(v[:,0].max()-t0)/1e3:.1f} us, duration min {d.min():.1f} "
          f"med {np.median(d):.1f} max {d.max():.1f} us; kernel span {(v[:,1].max()-t0)/1e3:.1f} us")
n = int((ev[2] > 0).sum())
e = ev[:, :n].astype(np.int64)
t0 = e[0, 0]
e = e - t0
ne = int((ev[4] > 0).sum())
print(f"CTA 5 w13: {n} stages, {ne} tiles, span {e[2, n-1]/1e3:.1f} us, per stage {e[2, n-1]/max(n,1):.0f} ns")
print("  TMA issue -> decode done   med ns", np.median(e[1] - e[0]))
print("  decode done -> MMA issued  med ns", np.median(e[2] - e[1]))
print("  MMA issue interval         med ns", np.median(np.diff(e[2])))
print("  decode-done interval       med ns", np.median(np.diff(e[1])))
epi = (ev[4, :ne].astype(np.int64) - ev[3, :ne].astype(np.int64))
print("  epilogue (wait tmem_full .. tmem_empty) per tile us:", np.round(epi / 1e3, 2)[:12])
for i in range(min(n, 40)):
    print(i, " ".join(f"{x/1e3:8.2f}" for x in e[:3, i]))
