import json, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.log"
for line in open(path):
    if line.startswith("[bench] timed"):
        print(line.strip()[:300])
    if line.startswith("{"):
        d = json.loads(line)
        r = d.get("roofline") or {}
        print("value %.0f tok/s  ms %.4f  roof %s %.0f GB/s frac %.3f  e2e %.0f" % (d["value"], d["ms_per_step"], r.get("kernel"), r.get("achieved", 0), r.get("frac", 0), d["e2e"]["value"]))
        aux = d.get("aux", {})
        if "unpacked_bf16_baseline" in aux: print("unpacked baseline ms", aux["unpacked_bf16_baseline"].get("ms_per_step"))
        for s in aux.get("sweep", []): print("  ", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in s.items()})
        print("clocks", d.get("clocks"))
