"""FP64 thread-instruction count of one kernel in an ncu report, from the
SASS source page (predicated-on thread instructions of DFMA/DMUL/DADD and the
other D* FP64-pipe opcodes).  usage: python tools/ncu_dp.py report.ncu-rep kernel_regex [units]"""
import csv
import io
import subprocess
import sys


def dp_count(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    tot = warp = 0
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        src = r[hdr.index("Source")].strip()
        if src.startswith("@"):
            src = src.split(" ", 1)[1]
        op = src.split(" ")[0].split(".")[0]
        if op in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DSET"):
            try:
                tot += int(r[hdr.index("Predicated-On Thread Instructions Executed")])
                warp += int(r[hdr.index("Instructions Executed")])
            except ValueError:
                pass
    return tot, warp


if __name__ == "__main__":
    t, w = dp_count(sys.argv[1], sys.argv[2])
    units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    print({"dp_thread_inst": t, "dp_warp_inst": w, "dp_thread_inst_per_unit": t / units})
