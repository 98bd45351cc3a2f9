"""CTA timeline of k_nbr_build and k_nonbonded in one reax_step (measurement
only).  Build the instrumented library first:

    python paper_1706_07772_b200/build.py -DREAX_TIMELINE --out=tools/libreax_tl.so

then on the GPU box:  REAX_LIBRARY=$PWD/tools/libreax_tl.so REAX_SERIAL=1 python tools/timeline.py [config]

Prints, per kernel: CTA count, span, setup and CTA duration percentiles, the
SM-time busy fraction (union of each SM's CTA intervals over the span), and
the number of resident CTAs over ten slices of the span."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1706_07772_b200 as rx  # noqa: E402


SPANS = ("k_bond_eval", "k_scan_lookback", "k_bond_fill", "k_bond_rank", "k_bond_delta", "k_bond_correct",
         "k_finalize", "k_nb_plan")


def analyse(tl, name):
    t0, t1, t2, sm, work = tl[:, 0], tl[:, 1], tl[:, 2], tl[:, 3] & 0xFFFF, tl[:, 3] >> 16
    ok = (t0 > 0) & (t2 >= t0)
    t0, t1, t2, sm, work = t0[ok], t1[ok], t2[ok], sm[ok], work[ok]
    ph = tl[ok][:, 4:8]
    base = t0.min()
    a, b, e = (t0 - base) / 1e3, (t1 - base) / 1e3, (t2 - base) / 1e3
    span = e.max()
    busy = 0.0
    nsm = int(sm.max()) + 1
    for s in range(nsm):
        iv = sorted(zip(a[sm == s], e[sm == s]))
        cur_s, cur_e = None, None
        for x, y in iv:
            if cur_e is None or x > cur_e:
                if cur_e is not None:
                    busy += cur_e - cur_s
                cur_s, cur_e = x, y
            else:
                cur_e = max(cur_e, y)
        if cur_e is not None:
            busy += cur_e - cur_s
    pc = lambda v: "p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(v, [10, 50, 90, 100]))
    print(f"{name}: {ok.sum()} CTAs on {len(np.unique(sm))} SMs, span {span:.1f} us")
    print(f"  start   {pc(a)}")
    print(f"  setup   {pc(b - a)}")
    print(f"  cta     {pc(e - a)}")
    if ph[:, 0].max() > 0:
        print(f"  window  {pc((ph[:, 0] - t0) / 1e3)}")
        print(f"  phase1  {pc((ph[:, 1] - ph[:, 0]) / 1e3)}")
        print(f"  phase2  {pc((t1 - ph[:, 1]) / 1e3)}")
    if ph[:, 3].max() > 0:
        print(f"  rows    {pc((ph[:, 2] - t1) / 1e3)} (to first warp done)")
        print(f"  warp tail {pc((ph[:, 3] - ph[:, 2]) / 1e3)} (first to last warp done)")
        print(f"  flush   {pc((t2 - ph[:, 3]) / 1e3)}")
    if ph[:, 3].max() > 0:
        # slot-time accounting over the span (2 resident CTAs per SM = full)
        slots = 148 * max(1, int(round(np.percentile([((a <= m) & (e > m)).sum() for m in [span * 0.1, span * 0.2, span * 0.3]], 50) / 148)))
        rows_t = ((ph[:, 2] - t1) / 1e3).sum() + 0.5 * ((ph[:, 3] - ph[:, 2]) / 1e3).sum()
        setup_t = (b - a).sum()
        tail_t = 0.5 * ((ph[:, 3] - ph[:, 2]) / 1e3).sum() + ((t2 - ph[:, 3]) / 1e3).sum()
        cap = slots * span
        print(f"  slot-time ({slots} slots x span): rows {rows_t / cap:.3f}, setup {setup_t / cap:.3f}, "
              f"warp tail + flush {tail_t / cap:.3f}, empty {1 - (rows_t + setup_t + tail_t) / cap:.3f}")
    print(f"  busy SM-time fraction {busy / (148 * span):.3f}")
    edges = np.linspace(0, span, 11)
    mid = 0.5 * (edges[1:] + edges[:-1])
    res = [int(((a <= m) & (e > m)).sum()) for m in mid]
    print("  resident CTAs per tenth:", res)
    dur = e - a
    print(f"  work ({'window slots' if name == 'k_nbr_build' else 'pairs'}) {pc(work)}; corr(work, dur) %.2f"
          % np.corrcoef(work, dur)[0, 1])
    big = work >= np.percentile(work, 50)
    rate = work[big] / (e[big] - b[big])
    print(f"  upper-half CTAs: work/us after setup {pc(rate)}")
    # co-residency of the longest CTAs: overlap with other CTAs on the same SM
    for i in np.argsort(dur)[-5:]:
        same = (sm == sm[i]) & (np.arange(len(sm)) != i)
        ov = [(round(a[k], 1), round(e[k], 1), int(work[k])) for k in np.where(same)[0]]
        print(f"  long CTA: sm {sm[i]} [{a[i]:.1f}, {e[i]:.1f}] work {work[i]}; others on SM: {ov}")
    order = np.argsort(a)
    late = order[-10:]
    print("  last 10 starts (us, dur):", [(round(a[i], 1), round(e[i] - a[i], 1)) for i in late])


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    lib = rx.load_library()
    if not hasattr(lib, "reax_timeline_read"):
        raise SystemExit("REAX_LIBRARY is not a -DREAX_TIMELINE build")
    p = gen.make_params()
    s = gen.make_config(cfg)
    dev = torch.device("cuda:0")
    pos, typ, q = (torch.from_numpy(x).to(dev) for x in (s.pos, s.type, s.q))
    ctx = rx.Reax(len(s.pos), s.box, p, gen.CUTOFFS, device=dev)
    for _ in range(5):
        ctx.step(pos, typ, q)
    torch.cuda.synchronize()
    lib.reax_timeline_reset()
    ctx.step(pos, typ, q)
    torch.cuda.synchronize()
    buf = np.zeros(2 * (1 << 16) * 8 + 16, np.uint64)
    n = lib.reax_timeline_read(ctypes.c_void_p(buf.ctypes.data))
    assert n == 1 << 16
    spans = buf[2 * (1 << 16) * 8:].reshape(8, 2).astype(np.int64)
    buf = buf[:2 * (1 << 16) * 8].reshape(2, 1 << 16, 8)
    analyse(buf[0].astype(np.int64), "k_nbr_build")
    analyse(buf[1].astype(np.int64), "k_nonbonded")
    s0 = buf[0][:, 0][buf[0][:, 0] > 0].min()
    s1 = buf[1][:, 0][buf[1][:, 0] > 0].min()
    e0 = buf[0][:, 2].max()
    print("nonbonded first start - list first start %.1f us; list last end - nonbonded first start %.1f us"
          % ((s1 - s0) / 1e3, (int(e0) - int(s1)) / 1e3))
    e1 = int(buf[1][:, 2].max())
    print("nonbonded last end: %.1f us after the list start" % ((e1 - int(s0)) / 1e3))
    for i, name in enumerate(SPANS):
        a, b = spans[i]
        if b > 0:
            print(f"  {name:16s} first start {(a - int(s0)) / 1e3:7.1f}  last end {(b - int(s0)) / 1e3:7.1f} us")


if __name__ == "__main__":
    main()
