"""Static SASS checks on the built library.

1. Self-branches in the middle of a function: ptxas places `BRA .` where it proved a path
   unreachable (undefined behaviour in the source, e.g. an out-of-bounds loop); the normal
   end-of-function padding (`EXIT/RET/BRA; BRA .; NOP...`) is ignored.
2. Evidence of the Blackwell instructions the design relies on (UTCHMMA / UTMALDG / LDTM /
   HMMA)."""
import re
import subprocess
import sys

obj = sys.argv[1] if len(sys.argv) > 1 else "paper_2511_04805_b200/libpuzzlemoe.so"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs, fn = {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        funcs[fn] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m and fn:
        funcs[fn].append((int(m.group(1), 16), m.group(2).strip()))
bad, counts = 0, {}
for fn, ins in funcs.items():
    for i, (addr, txt) in enumerate(ins):
        for key in ("UTCHMMA", "UTMALDG", "LDTM", "HMMA", "UTCBAR"):
            if key in txt:
                counts[key] = counts.get(key, 0) + 1
        b = re.match(r"BRA\s+0x([0-9a-f]+)$", txt)
        if b and int(b.group(1), 16) == addr:
            tail = [t for _, t in ins[i + 1:] if not t.startswith("NOP")]
            if tail:
                print(f"SELF-BRANCH mid-function (unreachable code / UB) in {fn} at {addr:#x}; next: {tail[0]}")
                bad += 1
print("instruction evidence:", counts)
sys.exit(1 if bad else 0)
