"""Regenerate profiles/ncu_summary.json (c4, c3_qeq entries) and
profiles/r02_summary.md from the committed round-2 captures."""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from ncu_dp import dp_count  # noqa: E402

NAMES = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
         "launch__registers_per_thread", "launch__grid_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
         "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def metrics(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    for row in r[2:]:
        if kernel in row[h.index("Kernel Name")]:
            m = {}
            for n in NAMES:
                v = float(row[h.index(n)])
                unit = u[h.index(n)]
                if n == "gpu__time_duration.sum":
                    v = v * {"ms": 1e3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}.get(unit, 1.0)
                if n.startswith("dram__bytes"):
                    v = v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(unit, 1.0)
                m[n] = v
            return m
    raise KeyError(kernel)


def entry(rep, kernel):
    m = metrics(os.path.join(ROOT, rep), kernel)
    return {"duration_us_cold": m["gpu__time_duration.sum"],
            "issue_active_pct": m["smsp__issue_active.avg.pct_of_peak_sustained_active"],
            "warps_active_pct": m["sm__warps_active.avg.pct_of_peak_sustained_active"],
            "sm_active_over_elapsed": m["sm__cycles_active.avg"] / m["gpc__cycles_elapsed.max"],
            "fp64_pipe_pct": m["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"],
            "xu_pipe_pct": m["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"],
            "warp_inst": m["smsp__inst_executed.sum"], "registers": m["launch__registers_per_thread"],
            "grid": m["launch__grid_size"],
            "dram_bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
            "dram_pct_of_peak": m["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]}


def main():
    N4, P4, N3, P3 = 16588000, 3394496961, 1039360, 212344633
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    s = json.load(open(summ_path))
    nbr = entry("profiles/r02_ncu_full_nbr_c4.ncu-rep", "k_nbr_build")
    nb = entry("profiles/r02_ncu_full_nonbonded_c4.ncu-rep", "k_nonbonded")
    q = entry("profiles/r02_ncu_full_qeq_c3.ncu-rep", "k_qeq_spmv")
    nbr["warp_inst_per_row"] = nbr["warp_inst"] / N4
    nb["warp_inst_per_row"] = nb["warp_inst"] / N4
    t, _ = dp_count(os.path.join(ROOT, "profiles/r02_ncu_full_nonbonded_c4.ncu-rep"), "k_nonbonded")
    nb["dp_thread_inst"] = t
    nb["dp_thread_inst_per_pair"] = t / P4
    q["spmv_bytes_alg"] = 2 * P3 * 12 + N3 * 32
    q["achieved_gbs_alg"] = q["spmv_bytes_alg"] / (q["duration_us_cold"] * 1e-6) / 1e9
    s["c4"] = {"_source": "profiles/r02_ncu_full_nbr_c4.ncu-rep, profiles/r02_ncu_full_nonbonded_c4.ncu-rep (round 2, "
                          "final code: ncu --set full --clock-control none --import-source on, tools/kbench.py 4 1, one "
                          "cold launch each); DP count from the SASS source page (tools/ncu_dp.py); launch list of the "
                          "bench step: profiles/r02_launches_c4.csv",
               "k_nbr_build": nbr, "k_nonbonded": nb}
    s["c3_qeq"] = {"_source": "profiles/r02_ncu_full_qeq_c3.ncu-rep (tools/qeqbench.py 3, first k_qeq_spmv launch)",
                   "k_qeq_spmv": q}
    json.dump(s, open(summ_path, "w"), indent=1)
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_c4.json")))
    L = ["# Round 2 profile summary (c4 = bench workload, 16,588,000 atoms, 3.39e9 half pairs)", "",
         f"Bench line (`bench.py --steps 5 --warmup 3`, CUDA-graph step, L2 flushed): {d['value'] / 1e6:.1f}M atom-steps/s, "
         f"{d['ms_per_step']:.2f} ms/step; k_nonbonded roofline frac {d['roofline']['frac']:.3f} (W_nb = 200 DP/pair vs the "
         f"live DFMA probe {d['roofline']['peak']:.2f} T/s); k_nbr_build frac {d['roofline_kernels'][0]['frac']:.3f} "
         f"(SURVEY 8(d) 900 B/atom vs {d['roofline_kernels'][0]['peak']} GB/s); e2e {d['e2e']['value'] / 1e6:.1f}M "
         f"atom-steps/s; c1 {d['c1']['value'] / 1e6:.1f}M ({d['c1']['ms_per_step'] * 1e3:.1f} us/step); cpu_baseline "
         f"{d['cpu_baseline']['value']:.0f} atom-steps/s on {d['cpu_baseline']['cores']} threads.", "",
         "| kernel | cold ms | issue active | warps active | FP64 pipe | XU pipe | warp inst / row | DRAM bytes |",
         "|---|---|---|---|---|---|---|---|"]
    for k, e in (("k_nbr_build", nbr), ("k_nonbonded", nb)):
        L.append(f"| {k} | {e['duration_us_cold'] / 1000:.2f} | {e['issue_active_pct']:.1f}% | {e['warps_active_pct']:.1f}% | "
                 f"{e['fp64_pipe_pct']:.1f}% | {e['xu_pipe_pct']:.1f}% | {e['warp_inst_per_row']:.0f} | "
                 f"{e['dram_bytes_per_launch'] / 1e9:.2f} GB |")
    L += ["", f"k_nonbonded executes {nb['dp_thread_inst_per_pair']:.1f} FP64 thread instructions per pair (SASS count, "
              "tools/ncu_dp.py).", "",
          f"QEq SpMV (c3, 2.12e8 half pairs, both right-hand sides in one pass over the doubly stored H): "
          f"{q['duration_us_cold']:.0f} us cold, {q['achieved_gbs_alg']:.0f} GB/s of algorithmic bytes "
          f"({q['achieved_gbs_alg'] / 6533.5:.2f} of the measured HBM bandwidth), issue active {q['issue_active_pct']:.1f}%, "
          f"warps active {q['warps_active_pct']:.1f}%.", "",
          "Launch list of the bench step: `r02_launches_c4.csv` (ncu --metrics gpu__time_duration.sum --clock-control "
          "none; cold, serialised).", "",
          "Binning, bond chain and finalize at c4 (`r02_ncu_full_chain_c4.ncu-rep`, `r02_ncu_full_chain2_c4.ncu-rep`; one cold launch each):", "",
          "| kernel | cold ms | issue active | warps active | DRAM bytes | DRAM % of peak |", "|---|---|---|---|---|---|"]
    chain = {}
    for k in ("k_cell_gather", "k_bond_eval", "k_bond_fill", "k_bond_rank", "k_bond_delta", "k_bond_correct",
              "k_finalize"):
        e = None
        for rep in ("profiles/r02_ncu_full_chain_c4.ncu-rep", "profiles/r02_ncu_full_chain2_c4.ncu-rep"):
            try:
                e = entry(rep, k)
                break
            except KeyError:
                continue
        if e is None:
            continue
        chain[k] = e
        L.append(f"| {k} | {e['duration_us_cold'] / 1000:.3f} | {e['issue_active_pct']:.1f}% | "
                 f"{e['warps_active_pct']:.1f}% | {e['dram_bytes_per_launch'] / 1e9:.2f} GB | {e['dram_pct_of_peak']:.1f}% |")
    s["c4"]["chain"] = chain
    json.dump(s, open(summ_path, "w"), indent=1)
    L += ["",
          "Rejected list-build variants and the reasons are in DESIGN.md §6 (k_nbr_build in round 2)."]
    open(os.path.join(ROOT, "profiles", "r02_summary.md"), "w").write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
