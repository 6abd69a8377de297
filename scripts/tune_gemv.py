"""Sweep GEMV split / n-tile knobs (env overrides) on one config; prints per-kernel times."""
import itertools, json, os, subprocess, sys
cfg, T = sys.argv[1], sys.argv[2]
combos = [dict(zip(["PUZZLE_GEMV_KS13", "PUZZLE_GEMV_KS2", "PUZZLE_GEMV_NT"], c)) for c in
          itertools.product(*(v.split(",") for v in sys.argv[3:6]))]
for env in combos:
    e = dict(os.environ, **{k: v for k, v in env.items() if v != "-"})
    out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--batch", T, "--steps", "100", "--warmup", "5",
                          "--no-cpu", "--no-extra"], capture_output=True, text=True, env=e)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if not line:
        print(env, "FAILED", out.stderr[-500:]); continue
    d = json.loads(line[0])
    k = {n: round(v["avg_ms"] * 1e3, 1) for n, v in d["kernels"].items()}
    print(env, "step_us", round(d["ms_per_step"] * 1e3, 1), "kern_us", k, flush=True)
