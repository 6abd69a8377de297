"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes per launch) per kernel."""
import csv, json, sys
from collections import defaultdict
path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit")
idi = hdr.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[1:]:
    if len(r) <= vi: continue
    try: v = float(r[vi].replace(",", ""))
    except ValueError: continue
    unit = r[ui]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    per[r[idi]][r[mi]] = v * scale
    names[r[idi]] = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
agg = defaultdict(lambda: defaultdict(float)); cnt = defaultdict(int)
for i, m in per.items():
    n = names[i]; cnt[n] += 1
    for k, v in m.items(): agg[n][k] += v
tot = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
out = {}
print(f"{'kernel':40s} {'launches':>8s} {'avg_us':>10s} {'share':>7s} {'dram_rd_MB/launch':>18s} {'dram_wr_MB/launch':>18s}")
for n, a in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
    c = cnt[n]; t = a.get("gpu__time_duration.sum", 0)
    rd = a.get("dram__bytes_read.sum", 0) / c; wr = a.get("dram__bytes_write.sum", 0) / c
    print(f"{n[:40]:40s} {c:8d} {t / c:10.2f} {t / tot:7.1%} {rd / 1e6:18.2f} {wr / 1e6:18.2f}")
    out[n] = {"launches": c, "avg_us": t / c, "share": t / tot, "dram_read_bytes_per_launch": rd, "dram_write_bytes_per_launch": wr}
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
