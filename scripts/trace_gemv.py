"""Pipeline timeline of one CTA of the tcgen05 decode w13 kernel (needs a PZ_TRACE build:
python scripts/build_variant.py trace gemv_tc.cu -DPZ_TRACE=<cta>; run with PUZZLE_LIB=...).

Events per stage t (globaltimer ns): 0 W TMA issued, 1 X TMA issued, 2 decoder sees W,
3 decoder sees A buffer free, 4 decoder A-full arrive, 6 MMA warp sees X, 5 MMA warp sees A
full, 7 MMAs + commits issued."""
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
for _ in range(5):
    layer.forward(hidden, logits, cfg.top_k, cfg.renormalize)
torch.cuda.synchronize()
lib = pz.load_library()
buf = np.zeros((8, 4096), np.uint64)
lib.puzzle_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.puzzle_debug_trace(buf.ctypes.data, buf.nbytes) == 0
n = int((buf[7] > 0).sum())
ev = buf[:, :n].astype(np.int64)
t0 = ev[0, 0]
ev = ev - t0
names = {0: "W issue", 1: "X issue", 2: "dec sees W", 3: "dec A free", 4: "dec A full", 6: "mma sees X",
         5: "mma sees A", 7: "mma issued"}
print(f"stages {n}, span {ev[7, n-1]/1e3:.1f} us, per stage {ev[7, n-1]/n:.0f} ns")
def med(a):
    return float(np.median(a))
print("W latency (issue -> decoder sees)      med ns", med(ev[2] - ev[0]))
print("X latency (issue -> mma sees)          med ns", med(ev[6] - ev[1]))
print("decode (sees W -> A full)              med ns", med(ev[4] - ev[2]))
print("  of which wait A free (sees W -> A)   med ns", med(ev[3] - ev[2]))
print("A full -> mma sees                     med ns", med(ev[5] - ev[4]))
print("mma issue time                         med ns", med(ev[7] - ev[5]))
print("X issue lag behind W issue             med ns", med(ev[1] - ev[0]))
print("W issue interval                       med ns", med(np.diff(ev[0])))
print("A free seen - mma issued 3 stages ago  med ns", med(ev[3, 3:] - ev[7, :-3]))
print("first 24 stages (us):")
for t in range(min(24, n)):
    print(t, " ".join(f"{names[e]}={ev[e, t]/1e3:7.2f}" for e in (0, 1, 2, 3, 4, 6, 5, 7)))
mid = int(sys.argv[3]) if len(sys.argv) > 3 else n // 2
print("middle stages:")
for t in range(mid, min(mid + 12, n)):
    print(t, " ".join(f"{names[e]}={ev[e, t]/1e3:7.2f}" for e in (0, 1, 2, 3, 4, 6, 5, 7)))

cta = np.zeros((2, 1024, 4), np.uint64)
lib.puzzle_debug_cta.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.puzzle_debug_cta(cta.ctypes.data, cta.nbytes) == 0
for kname, k in (("w13", 1), ("w2", 0)):
    v = cta[k].astype(np.int64)
    n = int((v[:, 3] > 0).sum())
    v = v[:n]
    t0 = v[:, 0].min()
    v = v - t0
    print(f"{kname}: {n} CTAs; start spread {v[:,0].max()/1e3:.1f} us; first W issue med {np.median(v[:,1])/1e3:.1f} "
          f"max {v[:,1].max()/1e3:.1f}; producer done min {v[:,2].min()/1e3:.1f} med {np.median(v[:,2])/1e3:.1f} "
          f"max {v[:,2].max()/1e3:.1f}; end min {v[:,3].min()/1e3:.1f} med {np.median(v[:,3])/1e3:.1f} max {v[:,3].max()/1e3:.1f} us")
    print("  end-time percentiles (us):", [round(float(np.percentile(v[:,3], q))/1e3, 1) for q in (0, 10, 25, 50, 75, 90, 99, 100)])
