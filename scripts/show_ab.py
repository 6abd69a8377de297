import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        print(l.strip()); continue
    if "max_abs_diff" in d:
        print("   diff", d["max_abs_diff"]); continue
    print(d.get("config"), d.get("T"), d.get("path"), d.get("ms_step"), d.get("tflops_proj"), d.get("frac_bf16_peak"),
          {k: v for k, v in d.get("kernel_us", {}).items() if k.startswith("w")})
