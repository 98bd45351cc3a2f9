"""QEq on one config (H build + the dual-RHS CG at tol 1e-6 from zero
guesses), for ncu captures of k_qeq_spmv / k_qeq_hbuild.  Prints one JSON
line with the per-phase times."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import gen
    import paper_1706_07772_b200 as rx
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    dev = torch.device("cuda:0")
    s = gen.make_config(k)
    p = gen.make_params()
    qp = gen.make_qeq_params()
    ctx = rx.Reax(len(s.pos), s.box, p, gen.CUTOFFS, device=dev)
    pos, typ = (torch.from_numpy(x).to(dev) for x in (s.pos, s.type))
    ctx.build_lists(pos, typ)
    ctx.qeq_build()                       # warm-up (module load, first launches)
    ctx.qeq_solve(qp.chi, qp.eta, tol=1e-6)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    ctx.qeq_build()
    ev[1].record()
    q, _, _, it = ctx.qeq_solve(qp.chi, qp.eta, tol=1e-6)
    ev[2].record()
    torch.cuda.synchronize()
    P, _ = ctx.pair_count()
    print(json.dumps({"config": k, "build_ms": ev[0].elapsed_time(ev[1]), "solve_ms": ev[1].elapsed_time(ev[2]),
                      "iters": it, "pairs": P}), flush=True)


if __name__ == "__main__":
    main()
