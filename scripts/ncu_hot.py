import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]; which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(out.splitlines()):
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}; blocks.append(cur); continue
    if cur is not None: cur["rows"].append(row)
b = blocks[which]; hdr = b["rows"][0]; rows = b["rows"][1:]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_src = hdr.index("Source"); i_ex = hdr.index("Instructions Executed"); i_addr = hdr.index("Address")
data = []
for r in rows:
    try: data.append((int(r[i_s]), int(r[i_ex]), r[i_addr], r[i_src].strip()))
    except (ValueError, IndexError): pass
tot = sum(d[0] for d in data); totex = sum(d[1] for d in data)
print(b["name"][:80], "samples", tot, "executed", totex)
c = Counter(); ce = Counter()
for s, ex, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    c[op] += s; ce[op] += ex
print("by opcode (samples):", c.most_common(14))
print("by opcode (executed):", ce.most_common(14))
if len(sys.argv) > 3:
    for s, ex, a, src in sorted(data, key=lambda x: -x[1])[:int(sys.argv[3])]: print(ex, s, a[-5:], src)
