"""Static SASS mix of the hottest loop of a kernel in libreax.so (the smallest
backward-branch region holding >= 30 DFMA): python tools/sass_loop.py k_nonbonded"""
import re, subprocess, sys
from collections import Counter
kern = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "-" else "paper_1706_07772_b200/libreax.so"
OPC = sys.argv[3] if len(sys.argv) > 3 else "DFMA"
MINC = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
f = [x for x in funcs if x.split("\n")[0].find(kern) >= 0][0]
ins = []
for line in f.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
    if m and m.group(1):
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            n = i - addr[tgt]
            ndfma = sum(1 for _, u in ins[addr[tgt]:i + 1] if OPC in u)
            if ndfma >= MINC and (best is None or n < best[0]):
                best = (n, addr[tgt], i)
n, lo, hi = best
c = Counter()
for a, t in ins[lo:hi + 1]:
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    op = t.split()[0]
    c[op.split(".")[0]] += 1
dp = sum(v for k, v in c.items() if k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
print(f"loop [{lo},{hi}] {n + 1} instructions, DP {dp}, other {n + 1 - dp}")
for k, v in c.most_common():
    print(f"  {k:10s} {v}")
