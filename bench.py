#!/usr/bin/env python
"""Benchmark of the B200 ReaxFF hot path (list build + bond orders + nonbonded).

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
One rank per GPU (torchrun for N > 1).  A step = one reax_step (lists rebuilt,
bond orders, nonbonded energies and forces) on the synthetic PETN-shaped
config C (default BASELINE.json configs[1], 32,480 atoms).  N > 1 runs
independent replicas ("replicas only": north_star keeps the path on one GPU).
Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (the
reference arm of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "atom-steps/s (list build+bond orders+nonbonded forces); % FP64/HBM roofline"
# Algorithmic work per unit:
W_NB_DP_PER_PAIR = 200.0    # FP64-pipe thread instructions per half pair (N1-N6, formula-minimal)
NBR_BYTES_PER_ATOM_FIXED = 16 + 4 + 4   # read fp32 local coords; write row length; bond-candidate count
NBR_BYTES_PER_PAIR = 2                  # one uint16 window slot per half-list entry
NBR_BYTES_PER_BONDCAND = 4
FLUSH_BYTES = 512 << 20                 # > 126 MB L2


def workload_name(k, c):
    return f"c{k}: {c['n']:,} atoms PETN-shaped (C5H8N4O12), box {'x'.join(str(b) for b in c['box'])} A"


def sample_clocks_start(dev_index):
    cmd = ["nvidia-smi", f"--id={dev_index}",
           "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
           "--format=csv,noheader,nounits", "-lms", "100"]
    try:
        return subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except Exception:
        return None


REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def sample_clocks_stop(p):
    if p is None:
        return None
    p.terminate()
    try:
        out, _ = p.communicate(timeout=5)
    except Exception:
        return None
    sm, mx, reasons = [], [], set()
    for line in out.strip().splitlines():
        f = [x.strip() for x in line.split(",")]
        if len(f) < 4:
            continue
        try:
            s, m = float(f[0]), float(f[1])
            r = int(f[3], 16)
        except ValueError:
            continue
        mx.append(m)
        if r & 0x1:   # idle samples say nothing about clocks under load
            continue
        sm.append(s)
        for bit, name in REASONS.items():
            if r & bit:
                reasons.add(name)
    if not mx:
        return None
    return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx), "samples_under_load": len(sm),
            "reasons": sorted(reasons)}


def max_over_ranks(vals, world, device):
    """Element-wise max over the ranks (a multi-GPU job takes as long as its
    slowest rank; timings are device-measured per rank, never wall clock)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def replica_throughput(n_atoms, steps, world, max_ms):
    """Whole-job atom-steps/s of `world` independent replicas (weak scaling,
    DESIGN.md "Multi-GPU": replicas only): every rank evaluates n_atoms per
    step; the job time is the slowest rank's."""
    return n_atoms * steps * world / (max_ms * 1e-3)


def run_cpu_oracle(k, evals):
    import gen
    import oracle
    params = gen.make_params()
    s = gen.make_config(k)
    oracle.build()
    t0 = time.perf_counter()
    for _ in range(evals):
        oracle.evaluate(s, params, gen.CUTOFFS)
    dt = time.perf_counter() - t0
    return len(s.pos) * evals / dt, dt, len(s.pos)


def reference_arm(args, rank, world):
    """The tier's reference arm: the CPU oracle as it stands, on the host cores."""
    import gen
    import oracle
    if rank != 0:
        return
    c = gen.CONFIGS[args.config]
    params = gen.make_params()
    oracle.build()
    # one full oracle evaluation of the config per step if that fits ~150 s
    # for W + K steps, else a smaller system from the same recipe (density,
    # generator, parameters, cutoffs): a bounded sample of the workload
    full = gen.make_config(args.config)
    t0 = time.perf_counter()
    oracle.evaluate(full, params, gen.CUTOFFS)
    t_full = time.perf_counter() - t0
    budget = 150.0 / max(1, args.steps + args.warmup)
    if t_full <= budget:
        s, sample = full, f"one full oracle evaluation of {workload_name(args.config, c)} per step"
    else:
        frac = max(budget / t_full, 0.02)
        n = max(2088, int(round(c["n"] * frac / 29)) * 29)
        L = (n / 0.0978) ** (1 / 3)
        s = gen.make_system(n, (L, L, L), gen.SEED_BASE + 100 + args.config)
        sample = (f"per step one full oracle evaluation of a {n:,}-atom system from the same recipe "
                  f"(cube {L:.2f} A, density 0.0978/A^3, same generator/params/cutoffs): bounded sample of c{args.config}")
    for _ in range(args.warmup):
        oracle.evaluate(s, params, gen.CUTOFFS)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.evaluate(s, params, gen.CUTOFFS)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = len(s.pos) * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "atom-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, c), "n_atoms": c["n"], "impl_detail": "C oracle (oracle/oracle.c), gcc -O2 -ffp-contract=off, 1 thread"},
        "cpu_baseline": {"value": value, "unit": "atom-steps/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "atom-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="direct launches instead of CUDA-graph replay")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # timing rule: W >= 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    import paper_1706_07772_b200 as rx
    from tools import build_tools

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    c = gen.CONFIGS[args.config]
    params = gen.make_params()
    s = gen.make_config(args.config)   # replicas: every rank the same synthetic instance
    n = len(s.pos)
    peak_dfma = build_tools.dfma_rate(5)

    ctx = rx.Reax(n, s.box, params, gen.CUTOFFS, device=dev)
    pos = torch.from_numpy(s.pos).to(dev)
    typ = torch.from_numpy(s.type).to(dev)
    q = torch.from_numpy(s.q).to(dev)
    F = torch.empty((n, 3), dtype=torch.float64, device=dev)
    E = torch.empty(2, dtype=torch.float64, device=dev)
    ctx.step(pos, typ, q, F, E)        # synchronous first call: validates, sizes capacities
    torch.cuda.synchronize()
    P, B = ctx.pair_count()
    ctx.set_async(True)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    clk = sample_clocks_start(local)
    for _ in range(args.warmup):
        flush.fill_(1.0)
        ctx.step(pos, typ, q, F, E)
    ctx.check()
    launches = ctx.launches_per_step()
    graph = tgraph = None
    if not args.no_graph:
        # the whole step as one CUDA graph (c1 is launch-bound with direct launches)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            ctx.step(pos, typ, q, F, E)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            ctx.step(pos, typ, q, F, E)
        # same step with the library's per-kernel CUDA events captured as
        # external event nodes (read back after each replay)
        ctx.set_timing(True)
        ctx.kernel_ms(reset=True)
        tgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(tgraph):
            ctx.step(pos, typ, q, F, E)
        ctx.set_timing(False)
        for _ in range(2):
            graph.replay()
            tgraph.replay()
        torch.cuda.synchronize()

    def one_step():
        if graph is not None:
            graph.replay()
        else:
            ctx.step(pos, typ, q, F, E)

    # pass 1 (value): K steps back to back, L2 flushed between them, each
    # bracketed by CUDA events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(float(k))          # L2 flush between timed steps (outside the events)
        ev[k][0].record()
        one_step()
        ev[k][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ctx.check()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    # pass 2 (kernel breakdown): the same K steps with per-kernel events live
    kms_acc = {k: 0.0 for k in rx.KERNEL_GROUPS}
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if tgraph is None:
        ctx.set_timing(True)
        ctx.kernel_ms(reset=True)
    for k in range(args.steps):
        flush.fill_(float(k))
        ev2[k][0].record()
        if tgraph is not None:
            tgraph.replay()
        else:
            ctx.step(pos, typ, q, F, E)
        ev2[k][1].record()
        if tgraph is not None:
            ev2[k][1].synchronize()
            for name, (ms, _) in ctx.kernel_ms(peek=True).items():
                kms_acc[name] += ms
    torch.cuda.synchronize()
    if tgraph is None:
        kms_acc = {name: ms for name, (ms, _) in ctx.kernel_ms(reset=True).items()}
        ctx.set_timing(False)
    ctx.check()
    pass2_ms = sum(a.elapsed_time(b) for a, b in ev2) / args.steps
    kms = {name: (kms_acc[name], args.steps) for name in kms_acc}
    tot_ms_max = max_over_ranks([sum(step_ms)], world, dev)[0]
    value = replica_throughput(n, args.steps, world, tot_ms_max)

    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(s.pos).pin_memory()
        ht = torch.from_numpy(s.type).pin_memory()
        hq = torch.from_numpy(s.q).pin_memory()
        hF = torch.empty((n, 3), dtype=torch.float64).pin_memory()
        hE = torch.empty(2, dtype=torch.float64).pin_memory()
        for _ in range(2):
            ctx.step_host(hp, ht, hq, hF, hE)
        eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.fill_(float(k))
            eev[k][0].record()
            ctx.step_host(hp, ht, hq, hF, hE)
            eev[k][1].record()
        torch.cuda.synchronize()
        e_ms = sum(a.elapsed_time(b) for a, b in eev)
        e_ms_max = max_over_ranks([e_ms], world, dev)[0]
        e2e = {"value": replica_throughput(n, args.steps, world, e_ms_max), "unit": "atom-steps/s",
               "h2d_bytes_per_step": hp.numel() * 8 + ht.numel() * 4 + hq.numel() * 8,
               "d2h_bytes_per_step": hF.numel() * 8 + hE.numel() * 8,
               "api": "reax_step_host (pinned host buffers in/out, copies inside the timed region)"}
    clocks = sample_clocks_stop(clk)

    # NEXT-1 (outside `value`): reax_bond_energy on the step's bond list, K
    # calls bracketed by events on the launching stream
    bond_energy = None
    try:
        bp = gen.make_bond_params()
        Fb = torch.empty((n, 3), dtype=torch.float64, device=dev)
        Eb = torch.empty(1, dtype=torch.float64, device=dev)
        one_step()
        for _ in range(3):
            ctx.bond_energy(bp, Fb, Eb)
        bev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.fill_(float(k))
            bev[k][0].record()
            ctx.bond_energy(bp, Fb, Eb)
            bev[k][1].record()
        torch.cuda.synchronize()
        ctx.check()
        b_ms = sum(a.elapsed_time(b) for a, b in bev) / args.steps
        bond_energy = {"row": "NEXT-1 bond energy + forces (reax_bond_energy), timed separately", "ms_per_call": b_ms,
                       "bond_entries": B, "bonds_per_s": (B / 2) / (b_ms * 1e-3), "launches_per_call": 3}
    except Exception as ex:   # reported, never silently dropped
        bond_energy = {"error": str(ex)}
    # NEXT-3 (outside `value`): reax_interaction_lists (counts + lists, both
    # synchronous), K calls bracketed by events
    ilists = None
    try:
        for _ in range(2):
            ctx.interaction_lists()
        torch.cuda.synchronize()
        iev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        sizes = None
        for k in range(args.steps):
            flush.fill_(float(k))
            iev[k][0].record()
            ao, ak, ho, hz = ctx.interaction_lists()
            iev[k][1].record()
            sizes = (len(ak), len(hz))
        torch.cuda.synchronize()
        ilists = {"row": "NEXT-3 3-body + H-bond lists (reax_interaction_counts + reax_interaction_lists), timed separately",
                  "ms_per_call": sum(a.elapsed_time(b) for a, b in iev) / args.steps,
                  "angle_entries": sizes[0], "hbond_entries": sizes[1]}
    except Exception as ex:   # reported, never silently dropped
        ilists = {"error": str(ex)}
    nb_ms, _ = kms["nonbonded"]
    nb_avg_s = nb_ms / args.steps * 1e-3
    achieved = W_NB_DP_PER_PAIR * P / nb_avg_s
    # list build on its own (the reax_build_lists path: k_nbr_build), timed
    # after the passes above (not part of `value`) for its roofline line
    lev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    lctx = rx.Reax(n, s.box, params, gen.CUTOFFS, device=dev)
    lctx.build_lists(pos, typ)
    lctx.set_async(True)
    lctx.set_timing(True)
    lctx.kernel_ms(reset=True)
    for k in range(10):
        flush.fill_(float(k))
        lctx.build_lists(pos, typ)
    torch.cuda.synchronize()
    lctx.check()
    lk = lctx.kernel_ms(reset=True)
    nbr_avg_s = lk["nbr"][0] / 10 * 1e-3
    # k_nonbonded on its own (the reax_nonbonded path: no concurrent bond
    # chain), same lists, for the kernel's isolated roofline line
    lctx.bond_orders()
    Fi = torch.empty((n, 3), dtype=torch.float64, device=dev)
    Ei = torch.empty(2, dtype=torch.float64, device=dev)
    lctx.nonbonded(pos, typ, q, Fi, Ei)
    lctx.kernel_ms(reset=True)
    for k in range(10):
        flush.fill_(float(k))
        lctx.nonbonded(pos, typ, q, Fi, Ei)
    torch.cuda.synchronize()
    lctx.check()
    nb_iso_s = lctx.kernel_ms(reset=True)["nonbonded"][0] / 10 * 1e-3
    del lctx
    nbr_bytes = n * NBR_BYTES_PER_ATOM_FIXED + P * NBR_BYTES_PER_PAIR + 2.9 * n * NBR_BYTES_PER_BONDCAND
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm_peak = 6650.0   # B200_PROFILING.md fallback
    traffic = nbr_traffic = dp_exec = None
    try:   # from the committed ncu capture of this workload (profiles/ncu_summary.json)
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))).get(f"c{args.config}", {})
        traffic = prof.get("k_nonbonded", {}).get("dram_bytes_per_launch")
        nbr_traffic = prof.get("k_nbr_build", {}).get("dram_bytes_per_launch")
        dp_exec = prof.get("k_nonbonded", {}).get("dp_thread_inst_per_pair")
    except Exception:
        pass
    step_total_ms = sum(v[0] for v in kms.values())
    line = {
        "metric": METRIC, "value": value, "unit": "atom-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, c), "n_atoms": n, "half_pairs": P, "bond_entries": B,
                   "evals_timed": args.steps, "lists": "rebuilt every step", "l2": "flushed (512 MB write) between timed steps",
                   "parallelism": "replicas" if world > 1 else "single GPU",
                   "launch": "direct launches" if args.no_graph else "CUDA graph replay of reax_step (async mode)"},
        "ns_per_atom_step": 1e9 / value * world if value else None,
        "roofline": {"bound": "alu", "kernel": "k_nonbonded (a7)",
                     "achieved": achieved / 1e12, "peak": peak_dfma / 1e12,
                     "unit": "T FP64-pipe thread-instructions/s", "frac": achieved / peak_dfma,
                     "traffic": traffic, "work": f"{W_NB_DP_PER_PAIR:.0f} DP inst/pair x {P} pairs per launch",
                     "peak_source": "DFMA probe measured in this run (tools/peak.cu); MEASURED_PEAKS.json has no FP64 entry",
                     "avg_launch_ms": nb_avg_s * 1e3,
                     "executed_dp_per_pair": dp_exec,
                     "fp64_pipe_frac": (dp_exec * P / nb_avg_s / peak_dfma) if dp_exec else None,
                     "note": "achieved/frac count the formula-minimal work W_nb = 200 FP64 inst/pair (SURVEY.md 8(d)); "
                             "the kernel executes executed_dp_per_pair (ncu DFMA+DMUL+DADD), fp64_pipe_frac is that rate "
                             "over the same peak"},
        "roofline_kernels": [
            {"kernel": "k_nbr_build (a3-a4; reax_build_lists path, timed separately)", "bound": "hbm", "achieved": nbr_bytes / nbr_avg_s / 1e9, "peak": hbm_peak,
             "unit": "GB/s", "frac": nbr_bytes / nbr_avg_s / 1e9 / hbm_peak, "avg_launch_ms": nbr_avg_s * 1e3,
             "bytes_per_launch": nbr_bytes, "traffic": nbr_traffic},
            {"kernel": "k_nonbonded (a7) on its own (reax_nonbonded path, no concurrent bond chain)", "bound": "alu",
             "achieved": W_NB_DP_PER_PAIR * P / nb_iso_s / 1e12, "peak": peak_dfma / 1e12,
             "unit": "T FP64-pipe thread-instructions/s", "frac": W_NB_DP_PER_PAIR * P / nb_iso_s / peak_dfma,
             "avg_launch_ms": nb_iso_s * 1e3},
        ],
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kms.items()},
        "timing_pass_ms_per_step": pass2_ms,
        "kernel_share": {k: v[0] / step_total_ms for k, v in kms.items()} if step_total_ms else None,
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "e2e": e2e,
        "next_rows": {"bond_energy": bond_energy, "interaction_lists": ilists},
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        evals = 3 if args.config <= 1 else 1
        v, dt, nn = run_cpu_oracle(args.config if args.config <= 2 else 1, evals)
        line["cpu_baseline"] = {"value": v, "unit": "atom-steps/s", "cores": 1, "kind": "oracle",
                                "sample": f"{evals} full oracle evaluation(s) of c{args.config if args.config <= 2 else 1} ({nn:,} atoms), {dt:.1f} s, 1 thread"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
