"""Pipeline timeline of the TS prefill kernel (PZ_TRACE build of gemm_ts.cu:
python scripts/build_variant.py tstrace gemm_ts.cu -DPZ_TRACE=4; run with PUZZLE_LIB=...).
CTA PZ_TRACE of the w13 kernel: per stage W TMA issue (0), X0 TMA issue (1), decoder words (2),
decoder A free (3), decoder afull (4), MMA0 xfull (5), MMA0 afull (6), MMA0 issued (7); per
item epilogue start (8) / end (9). All CTAs: start / end."""
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
    layer.forward(hidden, logits, cfg.top_k, cfg.renormalize, path=pz.PATH_TS)
torch.cuda.synchronize()
lib = pz.load_library()
ev = np.zeros((18, 4096), np.uint64)
cc = np.zeros((2, 1024, 2), np.uint64)
lib.puzzle_debug_ts.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t]
assert lib.puzzle_debug_ts(ev.ctypes.data, ev.nbytes, cc.ctypes.data, cc.nbytes) == 0
for name, k in (("w13", 1), ("w2", 0)):
    v = cc[k].astype(np.int64)
    n = int((v[:, 1] > 0).sum())
    v = v[:n]
    t0 = v[:, 0].min()
    d = (v[:, 1] - v[:, 0]) / 1e3
    print(f"{name}: {n} CTAs, start spread {(v[:,0].max()-t0)/1e3:.1f} us, duration min {d.min():.1f} "
          f"med {np.median(d):.1f} max {d.max():.1f} us; kernel span {(v[:,1].max()-t0)/1e3:.1f} us")
n = int((ev[7] > 0).sum())
e = ev[:, :].astype(np.int64)
t0 = e[0, 0]
print(f"stages traced {n}; per-stage (us since first W issue):")
names = ["Wiss", "X0iss", "Dwords", "DAfree", "Dafull", "Mxfull", "Mafull", "Missued"]
print("  s  " + " ".join(f"{x:>8}" for x in names) + "   dt(Missued)")
for s in list(range(0, 12)) + list(range(n // 2, n // 2 + 12)) + list(range(n - 6, n)):
    row = [(e[i, s] - t0) / 1e3 if e[i, s] else float("nan") for i in range(8)]
    dt = (e[7, s] - e[7, s - 1]) / 1e3 if s > 0 else 0
    print(f"{s:4d} " + " ".join(f"{x:8.2f}" for x in row) + f"   {dt:.3f}")
m = e[7, 1:n] - e[7, :n - 1]
print(f"MMA issue interval: median {np.median(m)/1e3:.3f} us, mean {m.mean()/1e3:.3f} us")
for a, b, lab in ((0, 2, "W issue -> words"), (1, 5, "X issue -> MMA xfull"), (2, 3, "words -> A free"),
                  (3, 4, "A free -> afull"), (4, 6, "afull -> MMA sees"), (5, 6, "MMA xfull -> afull"),
                  (6, 7, "MMA afull -> issued")):
    dd = (e[b, :n] - e[a, :n]) / 1e3
    print(f"  {lab:24s} median {np.median(dd):.3f} us  p90 {np.percentile(dd, 90):.3f}")
ni = int((ev[9] > 0).sum())
if ni:
    ep = (e[9, :ni] - e[8, :ni]) / 1e3
    print(f"items {ni}: epilogue median {np.median(ep):.2f} us, starts at " + " ".join(f"{(x - t0)/1e3:.1f}" for x in e[8, :ni]))
# A-ring cycle (kAStages = 4): MMA(s) issued -> its completion frees A buffer s % 4, seen by the
# decoder as "A free" of stage s + 4
A = int(os.environ.get('TS_ASTAGES', 4))
ss = np.arange(20, n - 8)
def med(x):
    return f"{np.median(x)/1e3:.3f}"
print("A-ring cycle (us): issue(s)->Afree(s+4)", med(e[3, ss + A] - e[7, ss]),
      "| Afree->afull(s+4)", med(e[4, ss + A] - e[3, ss + A]),
      "| afull(s+4)->MMA sees", med(e[6, ss + A] - e[4, ss + A]),
      "| MMA sees->issued(s+4)", med(e[7, ss + A] - e[6, ss + A]),
      "| issued(s+4)-issued(s)", med(e[7, ss + A] - e[7, ss]))
print("X-ring (3 slots) : issued(s)->X issue(s+3)", med(e[1, ss + 3] - e[7, ss]),
      "| X issue->xfull seen(s+3)", med(e[5, ss + 3] - e[1, ss + 3]))
print("W: decoder words(s)->W issue(s+4)", med(e[0, ss + 4] - e[2, ss]), "| W issue->words", med(e[2, ss] - e[0, ss]))
print("decoder: reach(s)->words(s)", med(e[2, ss] - e[13, ss]), "(W wait) | W issue(s)->reach(s)", med(e[13, ss] - e[0, ss]),
      "| Afree(s)-words(s)", med(e[3, ss] - e[2, ss]), "(A wait) | afull(s)->reach(s+1)", med(e[13, ss + 1] - e[4, ss]))
print("MMA0: issued(s)->xfull(s+1)", med(e[5, ss + 1] - e[7, ss]), "| xfull->afull", med(e[6, ss] - e[5, ss]))

# epilogue internals per item (events 8 accfull[0] seen, 14 first TMEM load landed, 15 half 0
# processed, 17 accfull[1] seen, 16 half 1 processed, 9 item end); MMA0 first issue of the next item
ni = int((ev[9] > 0).sum())
if ni and (ev[15, :ni] > 0).all():
    E = ev[:, :ni].astype(np.int64)
    print("epilogue internals (median us): accfull0->first load %.2f | first load->half0 processed %.2f | "
          "half0 processed->item end %.2f | accfull1 - accfull0 %.2f | accfull1->half1 processed %.2f" % (
              np.median(E[14] - E[8]) / 1e3, np.median(E[15] - E[14]) / 1e3, np.median(E[9] - E[15]) / 1e3,
              np.median(E[17] - E[8]) / 1e3, np.median(E[16] - E[17]) / 1e3))
