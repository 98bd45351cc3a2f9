"""NEXT-2 parity: reax_qeq_* (CUDA) against the oracle's O11 QEq
 on the same seeded inputs.
  * H x (both vectors) within 1e-12 relative of the oracle's half-stored
    SpMV (the oracle's H is pinned against a dense brute force);
  * solved tightly (tol 1e-11) both sides sit on the same exact solution:
    s, t, q within 1e-8 relative;
  * at the paper's tolerance 1e-6: the GPU's s and t have
    oracle-computed residuals below 1e-6 ||b||, sum q = 0, and the iteration
    counts are the oracle's (same algorithm, same stopping rule) within 2;
  * warm starts cut the iterations; results are bitwise
    reproducible; a new list makes an old H stale (REAX_ERR_STATE).
"""
import numpy as np
import pytest
import torch

import gen
import oracle
import paper_1706_07772_b200 as rx
from gpu_helpers import CUT, gpu_run

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def qp():
    return gen.make_qeq_params()


def _setup(system, params, ref=None):
    ref = ref if ref is not None else oracle.evaluate(system, params, CUT)
    ctx, _, _ = gpu_run(system, params)
    ctx.qeq_build()
    return ctx, ref


def _matvec_check(ctx, ref, system, params, qp, seed=0):
    n = len(system.pos)
    rng = np.random.default_rng(seed)
    xs, xt = rng.normal(size=n), rng.normal(size=n)
    hval = oracle.qeq_H(ref["pos"], system.type, system.box, params, CUT["r_nonb"], ref["hrow"], ref["hcol"])
    ea = qp.eta[system.type]
    ys_o = oracle.qeq_spmv(ea, ref["hrow"], ref["hcol"], hval, xs)
    yt_o = oracle.qeq_spmv(ea, ref["hrow"], ref["hcol"], hval, xt)
    ys, yt = ctx.qeq_matvec(qp.eta, torch.from_numpy(xs).to(DEV), torch.from_numpy(xt).to(DEV))
    scale = np.max(np.abs(ys_o))
    assert np.max(np.abs(ys.cpu().numpy() - ys_o)) <= 1e-12 * scale
    assert np.max(np.abs(yt.cpu().numpy() - yt_o)) <= 1e-12 * np.max(np.abs(yt_o))
    return hval


def _solve_check(ctx, ref, system, params, qp, hval, tight=True):
    n = len(system.pos)
    if tight:
        qo, so, to, ito = oracle.qeq(ref["pos"], system.type, system.box, params, CUT["r_nonb"], ref["hrow"],
                                     ref["hcol"], qp.chi, qp.eta, tol=1e-11)
        q, s, t, it = ctx.qeq_solve(qp.chi, qp.eta, tol=1e-11)
        for g, o in ((q, qo), (s, so), (t, to)):
            assert np.max(np.abs(g.cpu().numpy() - o)) <= 1e-8 * np.max(np.abs(o))
    # the paper's tolerance
    qo6, so6, to6, it6 = oracle.qeq(ref["pos"], system.type, system.box, params, CUT["r_nonb"], ref["hrow"],
                                    ref["hcol"], qp.chi, qp.eta, tol=1e-6)
    q, s, t, it = ctx.qeq_solve(qp.chi, qp.eta, tol=1e-6)
    s, t, q = s.cpu().numpy(), t.cpu().numpy(), q.cpu().numpy()
    ea = qp.eta[system.type]
    bs = -qp.chi[system.type]
    rs = bs - oracle.qeq_spmv(ea, ref["hrow"], ref["hcol"], hval, s)
    rt = -1.0 - oracle.qeq_spmv(ea, ref["hrow"], ref["hcol"], hval, t)
    assert np.linalg.norm(rs) <= 1.001e-6 * np.linalg.norm(bs)
    assert np.linalg.norm(rt) <= 1.001e-6 * np.sqrt(n)
    assert abs(q.sum()) <= 1e-10 * n
    assert abs(it[0] - it6[0]) <= 2 and abs(it[1] - it6[1]) <= 2, (it, it6)
    return it


def test_c0(params, c0, c0_oracle, qp):
    ctx, ref = _setup(c0, params, c0_oracle)
    hval = _matvec_check(ctx, ref, c0, params, qp)
    _solve_check(ctx, ref, c0, params, qp, hval)


def test_c1(params, qp):
    s = gen.make_config(1)
    ctx, ref = _setup(s, params)
    hval = _matvec_check(ctx, ref, s, params, qp, seed=1)
    _solve_check(ctx, ref, s, params, qp, hval)


@pytest.mark.parametrize("seed", range(3))
def test_tiny_boxes(params, qp, seed):
    rng = np.random.default_rng(400 + seed)
    s = gen.make_system(int(rng.integers(1, 300)), rng.uniform(20.05, 24.0, 3), 6100 + seed)
    ctx, ref = _setup(s, params)
    hval = _matvec_check(ctx, ref, s, params, qp, seed=seed)
    _solve_check(ctx, ref, s, params, qp, hval)


def test_warm_start_repeat_and_stale(params, c0, qp):
    ctx, ref = _setup(c0, params)
    q1, s1, t1, it1 = ctx.qeq_solve(qp.chi, qp.eta)
    q2, s2, t2, it2 = ctx.qeq_solve(qp.chi, qp.eta)           # zero guesses again: bitwise repeat
    assert torch.equal(q1, q2) and it1 == it2
    s0, t0 = s1 * (1 + 1e-4), t1 * (1 + 1e-4)
    q3, _, _, it3 = ctx.qeq_solve(qp.chi, qp.eta, s=s0, t=t0)  # warm start
    assert it3[0] < it1[0] and it3[1] < it1[1]
    assert torch.max(torch.abs(q3 - q1)) <= 1e-4 * torch.max(torch.abs(q1))
    pos = torch.from_numpy(c0.pos).to(DEV)
    ctx.build_lists(pos, torch.from_numpy(c0.type).to(DEV))   # new list: the built H is stale
    with pytest.raises(rx.ReaxError) as ei:
        ctx.qeq_solve(qp.chi, qp.eta)
    assert ei.value.code == rx.ERR_STATE


def test_maxiter_reports_nonconvergence(params, c0, qp):
    ctx, _ = _setup(c0, params)
    with pytest.raises(rx.ReaxError) as ei:
        ctx.qeq_solve(qp.chi, qp.eta, tol=1e-12, maxiter=3)
    assert ei.value.code == rx.ERR_CONVERGENCE


@pytest.mark.slow
def test_c3(params, qp):
    s = gen.make_config(3)
    ctx, ref = _setup(s, params)
    hval = _matvec_check(ctx, ref, s, params, qp, seed=3)
    _solve_check(ctx, ref, s, params, qp, hval, tight=False)   # the serial oracle's tight solve takes minutes here


def test_qeq_charges_drive_the_nonbonded_step(params, c0, c0_oracle, qp):
    """A QEq step as an MD code runs it (charges re-distributed
    every step): the GPU's QEq charges on the current lists feed
    reax_nonbonded; energies and forces match the oracle's nonbonded terms at
    the oracle's own QEq charges (both solved to 1e-11: the charges agree to
    ~1e-10, far inside the energy/force tolerances)."""
    ref = c0_oracle
    qo, _, _, _ = oracle.qeq(ref["pos"], c0.type, c0.box, params, CUT["r_nonb"], ref["hrow"], ref["hcol"], qp.chi,
                             qp.eta, tol=1e-11)
    Eo, Fo = oracle.nonbonded_rows(ref["pos"], c0.type, qo, c0.box, params, CUT["r_nonb"])
    pos = torch.from_numpy(c0.pos).to(DEV)
    typ = torch.from_numpy(c0.type).to(DEV)
    ctx = rx.Reax(len(c0.pos), c0.box, params, CUT, device=DEV)
    ctx.build_lists(pos, typ)      # the lists of this step (positions only)
    ctx.bond_orders()
    ctx.qeq_build()
    q, _, _, _ = ctx.qeq_solve(qp.chi, qp.eta, tol=1e-11)
    F, E = ctx.nonbonded(pos, typ, q)
    torch.cuda.synchronize()
    F, E = F.cpu().numpy(), E.cpu().numpy()
    assert np.all(np.abs(E - Eo) <= 1e-9 * np.abs(Eo)), (E, Eo)
    assert np.max(np.abs(F - Fo) / (1 + np.abs(Fo))) <= 1e-8
