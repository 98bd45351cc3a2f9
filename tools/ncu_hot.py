"""Top stall instructions of one kernel in an ncu report (source page, SASS).
python tools/ncu_hot.py report.ncu-rep [kernel-regex] [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
k = sys.argv[2] if len(sys.argv) > 2 else "."
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + k],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, isrc, ist = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[ia].isdigit()]
tot = sum(int(r[ist]) for r in data)
print("total warp inst", sum(int(r[ia]) for r in data), "stall samples", tot)
order = {id(r): i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -int(r[ist]))[:N]:
    print(f"{order[id(r)]:5d} {100 * int(r[ist]) / tot:5.1f}% exec={r[ia]:>8} {r[isrc][:90]}")
