"""Per-kernel timing of one library build at one config (events on the
launching stream, L2 flushed between calls): k_nbr_build through
reax_build_lists and k_nonbonded through reax_nonbonded.  Used to compare
compile-time variants (REAX_LIBRARY=path).  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import gen
    import paper_1706_07772_b200 as rx
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    dev = torch.device("cuda:0")
    s = gen.make_config(k)
    p = gen.make_params()
    n = len(s.pos)
    pos, typ, q = (torch.from_numpy(x).to(dev) for x in (s.pos, s.type, s.q))
    ctx = rx.Reax(n, s.box, p, gen.CUTOFFS, device=dev)
    ctx.build_lists(pos, typ)
    ctx.set_async(True)
    flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)
    ctx.set_timing(True)
    ctx.kernel_ms(reset=True)
    for i in range(reps):
        flush.fill_(float(i))
        ctx.build_lists(pos, typ)
    torch.cuda.synchronize()
    ctx.check()
    nbr = ctx.kernel_ms(reset=True)["nbr"][0] / reps
    ctx.bond_orders()
    ctx.kernel_ms(reset=True)
    for i in range(reps):
        flush.fill_(float(i))
        ctx.bond_orders()
    torch.cuda.synchronize()
    ctx.check()
    km = ctx.kernel_ms(reset=True)
    bonds, bo = km["bonds"][0] / reps, km["bond_orders"][0] / reps
    F = torch.empty((n, 3), dtype=torch.float64, device=dev)
    E = torch.empty(2, dtype=torch.float64, device=dev)
    ctx.nonbonded(pos, typ, q, F, E)
    ctx.kernel_ms(reset=True)
    for i in range(reps):
        flush.fill_(float(i))
        ctx.nonbonded(pos, typ, q, F, E)
    torch.cuda.synchronize()
    ctx.check()
    nb = ctx.kernel_ms(reset=True)["nonbonded"][0] / reps
    P, _ = ctx.pair_count()
    print(json.dumps({"lib": os.environ.get("REAX_LIBRARY", "default"), "config": k, "nbr_ms": nbr, "nb_ms": nb,
                      "bonds_ms": bonds, "bond_correct_ms": bo,
                      "pairs": P, "E": E.cpu().tolist()}), flush=True)


if __name__ == "__main__":
    main()
