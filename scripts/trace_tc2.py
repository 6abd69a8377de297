"""Per-stage timeline of cluster 0 of the CTA-pair prefill kernel (PZ_TRACE build of
gemm_tc2.cu; run with PUZZLE_LIB=... PUZZLE_PREFILL_IMPL=pair)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, synth  # noqa: E402
import paper_2511_04805_b200 as pz  # noqa: E402
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mixtral"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = torch.device("cuda:0")
layer, _ = bench.build_layer_gpu(pz, cfg, 1, dev)
hidden, logits = bench.make_inputs(cfg, T, 2, dev)
for _ in range(3):
    layer.forward(hidden, logits, cfg.top_k, cfg.renormalize)
torch.cuda.synchronize()
lib = pz.load_library()
ev = np.zeros((2, 4, 2048), np.uint64)
lib.puzzle_debug_tc2.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.puzzle_debug_tc2(ev.ctypes.data, ev.nbytes) == 0
n = int((ev[0, 2] > 0).sum())
t0 = int(ev[0, 0, 0])
e = ev[:, :, :n].astype(np.int64) - t0
print(f"stages {n}; per stage (leader MMA issue) {e[0,2,n-1]/n:.0f} ns")
for r in (0, 1):
    print(f"rank {r}: TMA->full seen med {np.median(e[r,3]-e[r,0]):.0f} ns, full->decoded {np.median(e[r,1]-e[r,3]):.0f}, "
          f"TMA issue interval {np.median(np.diff(e[r,0])):.0f}")
print("leader: decoded(both max) -> MMA issued med", np.median(e[0,2] - np.maximum(e[0,1], e[1,1])))
for i in list(range(0, 12)) + list(range(100, 108)):
    if i < n:
        print(i, " ".join(f"{x/1e3:8.2f}" for x in (e[0,0,i], e[1,0,i], e[0,3,i], e[1,3,i], e[0,1,i], e[1,1,i], e[0,2,i])))
