"""NEXT-1 parity: reax_bond_energy (CUDA) against the oracle's O8 on the same
seeded inputs.  E_bond within 1e-10 relative, forces within 1e-8 (1 + |F|)
kcal/mol/A (north_star tolerances of the path), Newton's third law at the
larger sizes."""
import numpy as np
import pytest
import torch

import gen
import oracle
from gpu_helpers import CUT, TOL_E, TOL_F, gpu_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bparams():
    return gen.make_bond_params()


def _gpu_bond(system, params, bparams, cut=CUT, async_=False):
    ctx, _, _ = gpu_run(system, params, cut, async_=async_)
    F, E = ctx.bond_energy(bparams)
    if async_:
        ctx.check()
    torch.cuda.synchronize()
    return ctx, F.cpu().numpy(), E.cpu().numpy()[0]


def _check(system, params, bparams, cut=CUT, **kw):
    Eo, Fo, _ = oracle.evaluate_bond_energy(system, params, bparams, cut)
    _, F, E = _gpu_bond(system, params, bparams, cut, **kw)
    assert abs(E - Eo) <= TOL_E * abs(Eo), (E, Eo)
    err = np.abs(F - Fo) / (1 + np.abs(Fo))
    assert err.max(initial=0) <= TOL_F, err.max()
    return E, F


def test_c0(params, c0, bparams):
    _check(c0, params, bparams)


def test_c1(params, bparams):
    _check(gen.make_config(1), params, bparams)


def test_async_and_repeat_bitwise(params, bparams):
    """Repeated calls (synchronous, then asynchronous) give bitwise equal results."""
    s = gen.make_config(0)
    ctx, F1, E1 = _gpu_bond(s, params, bparams)
    ctx.set_async(True)
    F2, E2 = ctx.bond_energy(bparams)
    ctx.check()
    assert np.array_equal(F1, F2.cpu().numpy()) and E1 == E2.cpu().numpy()[0]


@pytest.mark.parametrize("seed", range(4))
def test_tiny_boxes_and_param_variants(params, bparams, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(40, 400))
    L = (n / 0.0978) ** (1 / 3)
    rn = min(10.0, 0.48 * 0.97 * L)
    cut = dict(r_nonb=rn, r_bond=min(5.0, rn), bo_cut=0.01)
    s = gen.make_system(n, (L, L * 1.05, L * 0.97), gen.SEED_BASE + 900 + seed)
    bp = bparams.copy()
    if seed == 1:
        bp.p_be1[:] = 0.0
    if seed == 2:
        bp.p_be2[:] = 1e-300
    _check(s, params, bp, cut)


def test_empty_and_no_bonds(params, bparams):
    s = gen.System(np.zeros((0, 3)), np.zeros(0, np.int32), np.zeros(0), np.array([25.0, 25.0, 25.0]))
    ctx, _, _ = gpu_run(s, params)
    F, E = ctx.bond_energy(bparams)
    assert E.cpu().numpy()[0] == 0.0
    # two atoms 4.9 A apart: within r_bond but BO' < bo_cut -> no bond
    s = gen.System(np.array([[1.0, 1.0, 1.0], [5.9, 1.0, 1.0]]), np.array([0, 1], np.int32), np.zeros(2),
                   np.array([25.0, 25.0, 25.0]))
    ctx, _, _ = gpu_run(s, params)
    F, E = ctx.bond_energy(bparams)
    assert E.cpu().numpy()[0] == 0.0 and torch.all(F == 0)


def test_separate_calls_match_step(params, bparams):
    import paper_1706_07772_b200 as rx
    s = gen.make_config(1)
    dev = torch.device("cuda:0")
    pos, typ, q = (torch.from_numpy(x).to(dev) for x in (s.pos, s.type, s.q))
    a = rx.Reax(len(s.pos), s.box, params, CUT, device=dev)
    a.step(pos, typ, q)
    Fa, Ea = a.bond_energy(bparams)
    b = rx.Reax(len(s.pos), s.box, params, CUT, device=dev)
    b.build_lists(pos, typ)
    b.bond_orders()
    Fb, Eb = b.bond_energy(bparams)
    torch.cuda.synchronize()
    assert torch.equal(Fa, Fb) and torch.equal(Ea, Eb)


@pytest.mark.slow
def test_c2(params, bparams):
    _check(gen.make_config(2), params, bparams)
