#!/usr/bin/env python
"""Benchmark of the B200 ReaxFF hot path (list build + bond orders + nonbonded).

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
One rank per GPU (torchrun for N > 1).  A step = one reax_step (lists rebuilt,
bond orders, nonbonded energies and forces) on the synthetic PETN-shaped
config C (default BASELINE.json configs[4], 16,588,000 atoms: the largest
single-GPU config; c1 is reported beside it under "c1").  N > 1 runs
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
NBR_BYTES_PER_ATOM_ALG = 900.0         # algorithmic bytes per atom of the half-list build
NBR_BYTES_PER_ATOM_FIXED = 16 + 4 + 4   # as stored here: fp32 local coords in; row length, bond-candidate count out
NBR_BYTES_PER_PAIR = 2                  # one uint16 window slot per half-list entry
NBR_BYTES_PER_BONDCAND = 4
FLUSH_BYTES = 512 << 20                 # > 126 MB L2
DEFAULT_CONFIG = 4                      # the largest single-GPU config of BASELINE.json (c4, 16.6M atoms)
ORACLE_BUDGET_S = 20.0                  # CPU seconds of the bounded oracle sample (cpu_baseline)


def config_dict(k):
    """The workload description both arms print (identical dicts)."""
    import gen
    c = gen.CONFIGS[k]
    return {"workload": workload_name(k, c), "n_atoms": c["n"], "box_A": list(c["box"]),
            "cutoffs": dict(gen.CUTOFFS), "lists": "rebuilt every step",
            "l2": "GPU arm: 512 MB written between timed steps (L2 flush)"}


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_sample(k, budget_s, threads):
    """A bounded sample of config k for the CPU oracle: a smaller periodic
    system from the same recipe (generator, density 0.0978/A^3, PETN types,
    parameters, cutoffs), sized from a calibration run so that one oracle
    evaluation takes about budget_s on `threads` threads.  c0-c2 are small
    enough to be their own sample when they fit."""
    import gen
    import oracle
    params = gen.make_params()
    c = gen.CONFIGS[k]
    cal = gen.make_system(29 * 1120, (69.3, 69.3, 69.3), gen.SEED_BASE + 1)   # c1-sized calibration
    t0 = time.perf_counter()
    oracle.evaluate_stream(cal, params, gen.CUTOFFS, threads=threads)
    per_atom = (time.perf_counter() - t0) / len(cal.pos)
    if c["n"] * per_atom <= budget_s:
        return gen.make_config(k), f"one full oracle evaluation of c{k} ({c['n']:,} atoms)"
    n = max(2088, int(round(budget_s / per_atom / 29)) * 29)
    L = (n / 0.0978) ** (1 / 3)
    s = gen.make_system(n, (L, L, L), gen.SEED_BASE + 100 + k)
    return s, (f"one full oracle evaluation (lists, bond orders, energies, forces) of a {n:,}-atom periodic "
               f"cube of {L:.2f} A from the same recipe as c{k} (generator, density 0.0978/A^3, PETN types, "
               f"parameters, 10/5 A cutoffs): a bounded sample of c{k}'s {c['n']:,} atoms")


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


def run_cpu_oracle(k, evals, threads):
    import gen
    import oracle
    params = gen.make_params()
    oracle.build()
    s, sample = oracle_sample(k, ORACLE_BUDGET_S / max(1, evals), threads)
    t0 = time.perf_counter()
    phases = {}
    for _ in range(evals):
        r = oracle.evaluate_stream(s, params, gen.CUTOFFS, threads=threads)
        for k, v in r["phase_s"].items():
            phases[k] = phases.get(k, 0.0) + v / evals
    dt = time.perf_counter() - t0
    return len(s.pos) * evals / dt, dt, sample, phases


def reference_arm(args, rank, world):
    """The tier's reference arm: the CPU oracle as it stands, on the host cores."""
    import gen
    import oracle
    if rank != 0:
        return
    params = gen.make_params()
    oracle.build()
    threads = oracle.THREADS
    # each step one oracle evaluation of a bounded sample of the config, sized
    # so that the W + K steps take about 150 s on the host cores
    budget = 150.0 / max(1, args.steps + args.warmup)
    s, sample = oracle_sample(args.config, budget, threads)
    for _ in range(args.warmup):
        oracle.evaluate_stream(s, params, gen.CUTOFFS, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.evaluate_stream(s, params, gen.CUTOFFS, threads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = len(s.pos) * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "atom-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config),
        "impl_detail": f"C oracle (oracle/oracle.c), gcc -O2 -ffp-contract=off, row-parallel on {threads} threads "
                       "(oracle.evaluate_stream)",
        "cpu_baseline": {"value": value, "unit": "atom-steps/s", "cores": threads, "cpu": cpu_model(),
                         "kind": "oracle", "sample": sample + " per step"},
        "e2e": {"value": value, "unit": "atom-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def measure_c1(rx, gen, params, dev, flush, world, steps=50):
    """Supplementary: the same step on c1 (32,480 atoms; launch- and
    tail-bound), graph-replayed, L2 flushed between steps."""
    import torch
    s = gen.make_config(1)
    n = len(s.pos)
    ctx = rx.Reax(n, s.box, params, gen.CUTOFFS, device=dev)
    pos, typ, q = (torch.from_numpy(x).to(dev) for x in (s.pos, s.type, s.q))
    F = torch.empty((n, 3), dtype=torch.float64, device=dev)
    E = torch.empty(2, dtype=torch.float64, device=dev)
    ctx.step(pos, typ, q, F, E)
    torch.cuda.synchronize()
    ctx.set_async(True)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            ctx.step(pos, typ, q, F, E)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.step(pos, typ, q, F, E)
    for _ in range(3):
        g.replay()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        flush.fill_(float(k))
        ev[k][0].record()
        g.replay()
        ev[k][1].record()
    torch.cuda.synchronize()
    ctx.check()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    ms = max_over_ranks([ms], world, dev)[0]
    return {"workload": workload_name(1, gen.CONFIGS[1]), "value": replica_throughput(n, steps, world, ms),
            "unit": "atom-steps/s", "ms_per_step": ms / steps, "steps": steps,
            "note": "supplementary (BASELINE configs[1]); the headline is the config above"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--no-c1", action="store_true", help="skip the supplementary c1 measurement")
    ap.add_argument("--no-next", action="store_true", help="skip the next_rows measurements (profiling runs)")
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

    bond_energy = ilists = species = qeq = {"skipped": "--no-next"}
    # NEXT-1 (outside `value`): reax_bond_energy on the step's bond list, K
    # calls bracketed by events on the launching stream
    try:
        if args.no_next:
            raise StopIteration
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
    except StopIteration:
        pass
    except Exception as ex:   # reported, never silently dropped
        bond_energy = {"error": str(ex)}
    # NEXT-3 (outside `value`): reax_interaction_lists (counts + lists, both
    # synchronous), K calls bracketed by events
    try:
        if args.no_next:
            raise StopIteration
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
    except StopIteration:
        pass
    except Exception as ex:   # reported, never silently dropped
        ilists = {"error": str(ex)}
    # NEXT-4 (outside `value`): reax_species on the step's bond orders
    try:
        if args.no_next:
            raise StopIteration
        one_step()
        torch.cuda.synchronize()
        ctx.species()
        sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        for k in range(3):
            flush.fill_(float(k))
            sev[k][0].record()
            _, M, comp, cnt = ctx.species()
            sev[k][1].record()
        torch.cuda.synchronize()
        species = {"row": "NEXT-4 species analysis (reax_species: union-find, renumbering, census; synchronous)",
                   "ms_per_call": sum(a.elapsed_time(b) for a, b in sev) / 3, "molecules": M, "species": len(comp),
                   "bo_threshold": 0.3}
    except StopIteration:
        pass
    except Exception as ex:   # reported, never silently dropped
        species = {"error": str(ex)}
    # NEXT-2 (outside `value`): QEq on the step's half list (H build, then the
    # dual Jacobi-PCG at the paper's tolerance 1e-6 from zero guesses), if the
    # doubly stored H fits beside the workspace
    try:
        if args.no_next:
            raise StopIteration
        qp = gen.make_qeq_params()
        free, _ = torch.cuda.mem_get_info(dev)
        need = 2 * P * 12 + n * 120
        if need > free - (4 << 30):
            qeq = {"skipped": f"H needs {need / 2**30:.1f} GiB, {free / 2**30:.1f} GiB free"}
        else:
            qeq_ms = []
            for k in range(2):
                flush.fill_(float(k))
                a, b, c_ = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record()
                ctx.qeq_build()
                b.record()
                qq, ss, tt, it = ctx.qeq_solve(qp.chi, qp.eta, tol=1e-6)
                c_.record()
                torch.cuda.synchronize()
                qeq_ms.append((a.elapsed_time(b), b.elapsed_time(c_), it))
            bms, sms, it = qeq_ms[-1]
            qeq = {"row": "NEXT-2 QEq (reax_qeq_build + reax_qeq_solve, tol 1e-6, zero guesses)", "build_ms": bms,
                   "solve_ms": sms, "iterations": it, "spmv_bytes_per_iter": 2 * P * 12 + n * 32,
                   "ms_per_iteration": sms / max(1, max(it)),
                   "achieved_gbs_per_iteration": (2 * P * 12 + n * 32) / (sms / max(1, max(it)) * 1e-3) / 1e9}
            ctx._qeq_scratch = None
            torch.cuda.empty_cache()
    except StopIteration:
        pass
    except Exception as ex:
        qeq = {"error": str(ex)}
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
    nbr_bytes = n * NBR_BYTES_PER_ATOM_ALG
    nbr_bytes_stored = n * NBR_BYTES_PER_ATOM_FIXED + P * NBR_BYTES_PER_PAIR + 2.9 * n * NBR_BYTES_PER_BONDCAND
    hbm_peak, hbm_src = None, "MEASURED_PEAKS.json hbm_gbs"
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm_peak, hbm_src = 6650.0, "B200_PROFILING.md fallback"
    traffic = nbr_traffic = dp_exec = None
    prof_src = None
    try:   # from the committed ncu --set full capture of this workload (profiles/ncu_summary.json)
        summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        prof = summ.get(f"c{args.config}", {})
        traffic = prof.get("k_nonbonded", {}).get("dram_bytes_per_launch")
        nbr_traffic = prof.get("k_nbr_build", {}).get("dram_bytes_per_launch")
        dp_exec = prof.get("k_nonbonded", {}).get("dp_thread_inst_per_pair")
        prof_src = prof.get("_source") or summ.get("_source")
    except Exception:
        pass
    c1 = None
    if not args.no_c1 and args.config != 1:
        c1 = measure_c1(rx, gen, params, dev, flush, world)
    step_total_ms = sum(v[0] for v in kms.values())
    line = {
        "metric": METRIC, "value": value, "unit": "atom-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config),
        "counts": {"half_pairs": P, "bond_entries": B, "evals_timed": args.steps,
                   "parallelism": "replicas" if world > 1 else "single GPU",
                   "launch": "direct launches" if args.no_graph else "CUDA graph replay of reax_step (async mode)"},
        "ns_per_atom_step": 1e9 / value * world if value else None,
        "roofline": {"bound": "alu", "kernel": "k_nonbonded (a7)",
                     "achieved": achieved / 1e12, "peak": peak_dfma / 1e12,
                     "unit": "T FP64-pipe thread-instructions/s", "frac": achieved / peak_dfma,
                     "traffic": traffic, "traffic_source": prof_src,
                     "work": f"{W_NB_DP_PER_PAIR:.0f} DP inst/pair x {P} pairs per launch",
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
             "bytes_per_launch": nbr_bytes, "bytes_rule": "SURVEY.md 8(d) a3: 900 B/atom (algorithmic)",
             "bytes_stored_per_launch": nbr_bytes_stored, "peak_source": hbm_src,
             "traffic": nbr_traffic, "traffic_source": prof_src},
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
        "next_rows": {"bond_energy": bond_energy, "interaction_lists": ilists, "species": species, "qeq": qeq},
        "clocks": clocks,
    }
    if c1 is not None:
        line["c1"] = c1
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = oracle.THREADS
        v, dt, sample, phases = run_cpu_oracle(args.config, 1, threads)
        line["cpu_baseline"] = {"value": v, "unit": "atom-steps/s", "cores": threads, "cpu": cpu_model(),
                                "kind": "oracle", "sample": f"{sample}; {dt:.1f} s on {threads} threads",
                                "ns_per_atom_step": 1e9 / v, "phase_s": phases}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
