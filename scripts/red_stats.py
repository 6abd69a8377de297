"""Reducer timing from a step_timeline.py TIMELINE_DUMP (PZ_TRACE build): per kernel, the split
items' reducers' wait for the other pieces and their reduction time, and reducer vs other CTA
end times (us from the first pdl_wait return)."""
import sys

import numpy as np

for path in sys.argv[1:]:
    d = np.load(path)
    print(path)
    for k, kn in ((1, "w13"), (0, "w2")):
        red = d["red"][k].astype(np.int64)
        wt = d["wt"][k].astype(np.int64)
        cta = d["cta"][k].astype(np.int64)
        n = int((cta[:, 3] > 0).sum())
        idx = np.flatnonzero(red[:n, 3] > 0)
        t0 = wt[:n].min()
        r = (red[idx] - t0) / 1e3
        e = (cta[:n, 3] - t0) / 1e3
        non = np.setdiff1d(np.arange(n), idx)
        print(f"  {kn}: reducers {len(idx)}; wait med {np.median(r[:, 2] - r[:, 1]):.1f} max {np.max(r[:, 2] - r[:, 1]):.1f}; "
              f"reduce med {np.median(r[:, 3] - r[:, 2]):.1f} max {np.max(r[:, 3] - r[:, 2]):.1f} us; end: reducers med "
              f"{np.median(e[idx]):.1f} max {e[idx].max():.1f}, others med {np.median(e[non]):.1f} max {e[non].max():.1f}")
        if red.shape[-1] > 4 and (red[idx, 6] > 0).all():
            print(f"    counter seen -> loads landed (warp 0 / 4) med {np.median(r[:, 4] - r[:, 2]):.1f} / "
                  f"{np.median(r[:, 5] - r[:, 2]):.1f}; -> barrier {np.median(r[:, 6] - r[:, 2]):.1f}; "
                  f"barrier -> end {np.median(r[:, 3] - r[:, 6]):.1f} us")
