"""GPU parity: the CUDA path through the C ABI against the oracle, element by
element on the same seeded inputs (north_star tolerances: pair and bond sets
exact, BO 1e-12 abs, energies 1e-10 rel, forces 1e-8 (1+|F|))."""
import numpy as np
import pytest
import torch

import gen
import oracle
from gpu_helpers import (CUT, TOL_F, assert_energy_force, full_parity, gpu_run, pair_keys_gpu,
                         pair_keys_oracle)

pytestmark = pytest.mark.gpu


def test_c0_full(params, c0):
    full_parity(c0, params)


@pytest.mark.parametrize("seed", range(8))
def test_tiny_random_boxes(params, seed):
    rng = np.random.default_rng(100 + seed)
    box = rng.uniform(20.05, 26.0, 3)
    n = int(rng.integers(2, 300))
    full_parity(gen.make_system(n, box, 4000 + seed), params)


def test_ragged_sizes_and_dense_small_box(params):
    for n, box in ((1, (21, 21, 21)), (2, (20.5, 30, 22)), (33, (25, 21, 40)), (1000, (21.5, 21.5, 21.5))):
        s = gen.make_system(n, box, 77 + n)
        full_parity(s, params)


def test_exact_cutoff_pairs(params):
    # atoms placed exactly on sub-cell faces and at exactly r = R and r = r_bond
    L = 30.0
    pos = np.array([[0.0, 0.0, 0.0], [10.0, 0.0, 0.0], [20.0, 0.0, 0.0], [29.999999999999996, 1, 1],
                    [9.999999999999998, 1, 1], [5.0, 5.0, 5.0], [5.0, 15.0, 5.0], [5.0, 5.0, 15.0],
                    [1.0, 2.0, 3.0], [1.0 + 6.0, 2.0 + 8.0, 3.0], [15.0, 15.0, 15.0], [16.3, 15.0, 15.0]])
    typ = np.array([0, 1, 2, 3] * 3, np.int32)
    q = np.linspace(-0.4, 0.4, 12)
    s = gen.System(pos, typ, q - q.mean(), np.array([L, L, L]))
    ctx, ref, F, E = full_parity(s, params)
    assert len(ref["hcol"]) > 0 and len(ref["bcol"]) > 0


def test_positions_outside_box_are_wrapped(params):
    s = gen.make_system(500, (22.0, 23.0, 24.0), 9)
    k = np.random.default_rng(0).integers(-3, 4, size=s.pos.shape)
    shifted = s.pos + k * s.box
    ref = oracle.evaluate(gen.System(shifted, s.type, s.q, s.box), params, CUT)
    ctx, F, E = gpu_run(s, params, pos_override=shifted)
    n = len(s.pos)
    assert np.array_equal(pair_keys_gpu(ctx, n), pair_keys_oracle(ref["hrow"], ref["hcol"], n))
    assert_energy_force(E, F, ref["E"], ref["F"])


def test_empty_system(params):
    s = gen.System(np.zeros((0, 3)), np.zeros(0, np.int32), np.zeros(0), np.array([25.0, 25.0, 25.0]))
    ctx, F, E = gpu_run(s, params)
    assert F.shape == (0, 3) and E.tolist() == [0.0, 0.0]
    assert ctx.pair_count() == (0, 0)


def test_c1_full(params):
    full_parity(gen.make_config(1), params)


def test_async_mode_matches(params):
    s = gen.make_config(1)
    _, F1, E1 = gpu_run(s, params)
    _, F2, E2 = gpu_run(s, params, async_=True)
    assert np.array_equal(E1, E2)   # energies are reduced in a fixed order
    assert np.all(np.abs(F1 - F2) <= 1e-12 * (1 + np.abs(F1)))


def test_cuda_graph_replay_matches(params):
    import paper_1706_07772_b200 as rx
    s = gen.make_config(1)
    dev = torch.device("cuda:0")
    ctx = rx.Reax(len(s.pos), s.box, params, CUT, device=dev)
    pos = torch.from_numpy(s.pos).to(dev)
    typ = torch.from_numpy(s.type).to(dev)
    q = torch.from_numpy(s.q).to(dev)
    F0, E0 = ctx.step(pos, typ, q)
    torch.cuda.synchronize()
    F0, E0 = F0.cpu().numpy(), E0.cpu().numpy()
    ctx.set_async(True)
    F = torch.empty((len(s.pos), 3), dtype=torch.float64, device=dev)
    E = torch.empty(2, dtype=torch.float64, device=dev)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        ctx.step(pos, typ, q, F, E)  # warm-up on the capture stream
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.step(pos, typ, q, F, E)
    F.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    ctx.check()
    assert np.array_equal(E.cpu().numpy(), E0)
    assert np.array_equal(F.cpu().numpy(), F0)


def test_capacity_regrow(params):
    s = gen.make_config(0)
    ref = oracle.evaluate(s, params, CUT)
    ctx, F, E = gpu_run(s, params, capacity=dict(row_cap=64, cand_cap=2, bond_cap=100, window_cap=256))
    assert ctx.cap.row_cap >= 64 and ctx.cap.window_cap > 256
    assert_energy_force(E, F, ref["E"], ref["F"])
    n = len(s.pos)
    assert np.array_equal(pair_keys_gpu(ctx, n), pair_keys_oracle(ref["hrow"], ref["hcol"], n))


def test_repeat_steps_deterministic(params):
    import paper_1706_07772_b200 as rx
    s = gen.make_config(1)
    dev = torch.device("cuda:0")
    ctx = rx.Reax(len(s.pos), s.box, params, CUT, device=dev)
    pos = torch.from_numpy(s.pos).to(dev)
    typ = torch.from_numpy(s.type).to(dev)
    q = torch.from_numpy(s.q).to(dev)
    out = [ctx.step(pos, typ, q) for _ in range(3)]
    torch.cuda.synchronize()
    E = [o[1].cpu().numpy() for o in out]
    assert np.array_equal(E[0], E[1]) and np.array_equal(E[1], E[2])
    F = [o[0].cpu().numpy() for o in out]
    # fixed-point force accumulation: integer sums are order-free, so forces
    # are bitwise reproducible too
    assert np.array_equal(F[0], F[1]) and np.array_equal(F[1], F[2])


@pytest.mark.slow
def test_c2_full(params):
    full_parity(gen.make_config(2), params)


def test_separate_calls_match_step(params):
    """reax_build_lists + reax_bond_orders + reax_nonbonded (one stream) and
    reax_step (bond chain forked onto a side stream beside the nonbonded
    kernel) give identical lists, bond orders, forces and energies."""
    import paper_1706_07772_b200 as rx
    s = gen.make_config(1)
    dev = torch.device("cuda:0")
    n = len(s.pos)
    pos = torch.from_numpy(s.pos).to(dev)
    typ = torch.from_numpy(s.type).to(dev)
    q = torch.from_numpy(s.q).to(dev)
    a = rx.Reax(n, s.box, params, CUT, device=dev)
    Fa, Ea = a.step(pos, typ, q)
    b = rx.Reax(n, s.box, params, CUT, device=dev)
    b.build_lists(pos, typ)
    b.bond_orders()
    Fb, Eb = b.nonbonded(pos, typ, q)
    torch.cuda.synchronize()
    assert np.array_equal(pair_keys_gpu(a, n), pair_keys_gpu(b, n))
    ba = [t.cpu().numpy() for t in a.export_bonds()]
    bb = [t.cpu().numpy() for t in b.export_bonds()]
    for x, y in zip(ba, bb):
        assert np.array_equal(x, y)
    assert np.array_equal(Fa.cpu().numpy(), Fb.cpu().numpy())
    assert np.array_equal(Ea.cpu().numpy(), Eb.cpu().numpy())


def test_step_host_graph_replay(params):
    """reax_step_host replays a captured graph while its host buffers, box and
    parameters stay the same: repeated calls match the device path, new
    contents of the same buffers are picked up, new buffers are re-captured."""
    import paper_1706_07772_b200 as rx
    s = gen.make_config(0)
    n = len(s.pos)
    dev = torch.device("cuda:0")
    ctx = rx.Reax(n, s.box, params, CUT, device=dev)
    pos = torch.from_numpy(s.pos.copy()).pin_memory()
    typ = torch.from_numpy(s.type).pin_memory()
    q = torch.from_numpy(s.q).pin_memory()
    F = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    E = torch.empty(2, dtype=torch.float64).pin_memory()
    Fd, Ed = ctx.step(pos.to(dev), typ.to(dev), q.to(dev))
    Fd, Ed = Fd.cpu().numpy(), Ed.cpu().numpy()
    for _ in range(3):   # first call direct + capture, then replays
        F.zero_()
        ctx.step_host(pos, typ, q, F, E)
        assert np.array_equal(F.numpy(), Fd) and np.array_equal(E.numpy(), Ed)
    # new contents of the same pinned buffers: a translated system (same physics)
    pos.copy_(torch.from_numpy(oracle.wrap(s.pos + np.array([1.7, -2.3, 0.9]), s.box)))
    ctx.step_host(pos, typ, q, F, E)
    assert np.all(np.abs(E.numpy() - Ed) <= 1e-10 * np.abs(Ed))
    assert np.all(np.abs(F.numpy() - Fd) <= 1e-8 * (1 + np.abs(Fd)))
    # a different output buffer: re-captured, same results
    F2 = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    for _ in range(2):
        ctx.step_host(pos, typ, q, F2, E)
        assert np.array_equal(F2.numpy(), F.numpy())


def test_dense_system_regrows(params):
    """2.6x the PETN density (0.25 atoms/A^3, RSA with the 0.9 A minimum
    separation): rows of ~520 entries and windows of ~5400 atoms, beyond the
    default window capacity (it regrows; the nonbonded kernel's shared memory
    still fits) — the result is still exact against the oracle."""
    s = gen.make_system(2662, (22.0, 22.0, 22.0), gen.SEED_BASE + 321)
    ctx, _, _, _ = full_parity(s, params)
    assert ctx.cap.row_cap > 512 and ctx.cap.window_cap > 2048


def test_gpu_invariances(params):
    """GPU-only invariants at c1: a rigid translation (then
    wrap) and a relabelling of the atoms leave the pair and bond counts, the
    energies (1e-10 relative) and the forces (1e-8 (1 + |F|), permuted) as
    they were; the net force vanishes."""
    s = gen.make_config(1)
    ctx, F, E = gpu_run(s, params)
    P, B = ctx.pair_count()
    assert np.all(np.abs(F.sum(0)) <= 1e-11 * np.abs(F).sum())
    t = gen.System(oracle.wrap(s.pos + np.array([13.7, -21.1, 5.3]), s.box), s.type, s.q, s.box)
    ctx2, F2, E2 = gpu_run(t, params)
    assert ctx2.pair_count() == (P, B)
    assert np.all(np.abs(E2 - E) <= 1e-10 * np.abs(E))
    assert np.all(np.abs(F2 - F) <= 1e-8 * (1 + np.abs(F)))
    perm = np.random.default_rng(9).permutation(len(s.pos))
    r = gen.System(s.pos[perm].copy(), s.type[perm].copy(), s.q[perm].copy(), s.box)
    ctx3, F3, E3 = gpu_run(r, params)
    assert ctx3.pair_count() == (P, B)
    assert np.all(np.abs(E3 - E) <= 1e-10 * np.abs(E))
    assert np.all(np.abs(F3 - F[perm]) <= 1e-8 * (1 + np.abs(F[perm])))


def test_plan_interleaving_bitwise(params):
    """The nonbonded work plan (heavy home blocks split into units that share
    a global row counter) never changes a result: steps, separate nonbonded
    calls and steps again on one context give bitwise the forces and energies
    of a fresh context, also for a translated system (another plan)."""
    import paper_1706_07772_b200 as rx
    s = gen.make_config(1)
    dev = torch.device("cuda:0")
    pos, typ, q = (torch.from_numpy(x).to(dev) for x in (s.pos, s.type, s.q))
    ref = rx.Reax(len(s.pos), s.box, params, CUT, device=dev)
    F0, E0 = (t.clone() for t in ref.step(pos, typ, q))
    ctx = rx.Reax(len(s.pos), s.box, params, CUT, device=dev)
    for k in range(3):
        F, E = ctx.step(pos, typ, q)
        assert torch.equal(F, F0) and torch.equal(E, E0), k
        F, E = ctx.nonbonded(pos, typ, q)
        Fn, En = ctx.step(pos, typ, q)
        assert torch.equal(Fn, F0) and torch.equal(En, E0), k
    pos2 = torch.from_numpy(oracle.wrap(s.pos + np.array([3.3, -1.1, 7.7]), s.box)).to(dev)
    F1, E1 = (t.clone() for t in ref.step(pos2, typ, q))
    for k in range(3):
        F, E = ctx.step(pos2, typ, q)
        assert torch.equal(F, F1) and torch.equal(E, E1), k


def test_plan_near_limit_grid(params):
    """A 95 A box (19 sub-cells per axis: 10^3 = 1000 home blocks, just under
    the 1024-block limit of the nonbonded work plan, with partial blocks on
    three faces): full parity with the oracle through the planned grid."""
    L = 95.0
    s = gen.make_system(int(0.0978 * L ** 3), (L, L, L), gen.SEED_BASE + 1234)
    full_parity(s, params)


@pytest.mark.parametrize("seed,ntypes", [(11, 4), (12, 4), (13, 1), (14, 7), (15, 16)])
def test_parameter_draws_and_type_counts(seed, ntypes):
    """Other seeded parameter tables from the same ranges (DESIGN.md reading
    10), and other type counts (1 type; 7; the 16-type maximum,
    REAX_MAX_TYPES): types drawn uniformly; full parity on c0-sized boxes."""
    p = gen.make_params(seed=gen.SEED_BASE + seed, ntypes=ntypes)
    s = gen.make_system(1500, (25.0, 24.0, 26.5), gen.SEED_BASE + 900 + seed)
    rng = np.random.default_rng(seed)
    s = gen.System(s.pos, rng.integers(0, ntypes, len(s.pos)).astype(np.int32), s.q, s.box)
    full_parity(s, p)


def test_zero_charges_zero_coulomb(params, c0):
    """q = 0 everywhere: E_Coul is exactly 0 and the forces are
    the vdW forces alone (the oracle at q = 0)."""
    s = gen.System(c0.pos, c0.type, np.zeros_like(c0.q), c0.box)
    ctx, ref, F, E = full_parity(s, params)
    assert E[1] == 0.0
