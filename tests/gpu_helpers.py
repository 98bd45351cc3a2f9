"""Shared helpers for the -m gpu parity tests (GPU path vs the C oracle)."""
import numpy as np
import torch

import gen
import oracle
import paper_1706_07772_b200 as rx

CUT = gen.CUTOFFS
TOL_BO = 1e-12          # bond orders / Delta', absolute (north_star)
TOL_E = 1e-10           # energies, relative (north_star)
TOL_F = 1e-8            # forces: |dF| <= 1e-8 (1 + |F|) (north_star)


def gpu_run(system, params, cut=CUT, capacity=None, async_=False, pos_override=None):
    dev = torch.device("cuda:0")
    ctx = rx.Reax(len(system.pos), system.box, params, cut, capacity=capacity, device=dev)
    if async_:
        ctx.set_async(True)
    pos_np = system.pos if pos_override is None else pos_override
    pos = torch.from_numpy(np.ascontiguousarray(pos_np)).to(dev)
    typ = torch.from_numpy(system.type).to(dev)
    q = torch.from_numpy(system.q).to(dev)
    F, E = ctx.step(pos, typ, q)
    if async_:
        ctx.check()
    torch.cuda.synchronize()
    return ctx, F.cpu().numpy(), E.cpu().numpy()


def pair_keys_gpu(ctx, n):
    pi, pj = ctx.export_pairs()
    k = pi.to(torch.int64) * n + pj.to(torch.int64)
    return np.sort(k.cpu().numpy())


def pair_keys_oracle(hrow, hcol, n):
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(hrow))
    return rows * n + hcol.astype(np.int64)  # canonical: already sorted


def assert_bonds_equal(ctx, ref):
    brow, bcol, mir, bo, dl = [t.cpu().numpy() for t in ctx.export_bonds()]
    assert np.array_equal(brow, ref["brow"]), "bond row offsets differ"
    assert np.array_equal(bcol, ref["bcol"]), "bond partners differ"
    assert np.array_equal(mir, ref["mirror"]), "mirror indices differ"
    assert np.max(np.abs(bo[:, :4] - ref["raw"]), initial=0) <= TOL_BO
    assert np.max(np.abs(bo[:, 4:] - ref["corr"]), initial=0) <= TOL_BO
    assert np.max(np.abs(dl - ref["delta"]), initial=0) <= TOL_BO
    # bitwise symmetry BO_ij == BO_ji
    assert np.array_equal(bo[mir], bo)
    return bo


def assert_energy_force(E, F, Eref, Fref):
    assert np.all(np.abs(E - Eref) <= TOL_E * np.abs(Eref)), (E, Eref, (E - Eref) / Eref)
    err = np.abs(F - Fref) / (1 + np.abs(Fref))
    assert err.max(initial=0) <= TOL_F, err.max()


def full_parity(system, params, cut=CUT, **kw):
    ref = oracle.evaluate(system, params, cut)
    ctx, F, E = gpu_run(system, params, cut, **kw)
    n = len(system.pos)
    P, B = ctx.pair_count()
    assert P == len(ref["hcol"]), (P, len(ref["hcol"]))
    assert np.array_equal(pair_keys_gpu(ctx, n), pair_keys_oracle(ref["hrow"], ref["hcol"], n))
    assert B == len(ref["bcol"])
    assert_bonds_equal(ctx, ref)
    assert_energy_force(E, F, ref["E"], ref["F"])
    return ctx, ref, F, E
