"""Context-state and range edge cases of the C ABI:
host-graph replay after another parameter set or a re-bound workspace,
the coarsened nonbonded work plan, and REAX_ERR_RANGE."""
import ctypes
import os

import numpy as np
import pytest
import torch

import gen
import paper_1706_07772_b200 as rx
from gpu_helpers import CUT, gpu_run

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _host(s):
    return [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (s.pos, s.type, s.q)]


def test_step_host_replay_after_other_params(params):
    """reax_step_host(A) captures a graph without the parameter upload; a call
    with parameter set B on the same context uploads B; the next
    reax_step_host(A) must upload A again before replaying."""
    s = gen.make_config(0)
    n = len(s.pos)
    pB = params.copy()
    pB.eps = pB.eps * 1.7
    pB.gamma = pB.gamma * 0.8
    ctx = rx.Reax(n, s.box, params, CUT, device=DEV)
    hp, ht, hq = _host(s)
    F = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    E = torch.empty(2, dtype=torch.float64).pin_memory()
    for _ in range(2):                      # direct + capture, then a replay
        ctx.step_host(hp, ht, hq, F, E)
    FA, EA = F.numpy().copy(), E.numpy().copy()
    holderA = ctx.params
    ctx.params = rx._ParamsHolder(pB)       # same context, parameter set B
    FB, EB = ctx.step(hp.to(DEV), ht.to(DEV), hq.to(DEV))
    torch.cuda.synchronize()
    assert not np.array_equal(EB.cpu().numpy(), EA)
    ctx.params = holderA
    F.zero_()
    ctx.step_host(hp, ht, hq, F, E)         # replay path
    assert np.array_equal(E.numpy(), EA) and np.array_equal(F.numpy(), FA)


def test_rebind_same_address_drops_host_graph(params):
    """Re-binding a workspace at the same base address with another layout
    (other capacities) must not replay the graph captured for the old layout:
    the exports read the new layout and must see this step's lists."""
    s = gen.make_config(0)
    n = len(s.pos)
    ctx = rx.Reax(n, s.box, params, CUT, capacity=dict(row_cap=512, window_cap=4096, cand_cap=24), device=DEV)
    hp, ht, hq = _host(s)
    F = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    E = torch.empty(2, dtype=torch.float64).pin_memory()
    for _ in range(2):
        ctx.step_host(hp, ht, hq, F, E)
    F0, E0 = F.numpy().copy(), E.numpy().copy()
    ref = rx.Reax(n, s.box, params, CUT, device=DEV)
    ref.step(hp.to(DEV), ht.to(DEV), hq.to(DEV))
    cnt_ref, dig_ref = [t.cpu().numpy() for t in ref.export_digest()]
    # same buffer, smaller capacities: a different layout at the same base
    small = rx.Capacity(0, 0, 0, 0)
    nbytes = ctypes.c_size_t()
    resolved = rx.Capacity()
    assert ctx.lib.reax_workspace_bytes(ctx.n, ctx.box, ctypes.byref(ctx.cut), ctypes.byref(small),
                                        ctypes.byref(nbytes), ctypes.byref(resolved)) == 0
    assert nbytes.value <= ctx.workspace_bytes
    assert ctx.lib.reax_bind_workspace(ctx.ctx, ctypes.c_void_p(ctx.ws.data_ptr()), ctx.workspace_bytes, ctx.n,
                                       ctx.box, ctypes.byref(ctx.cut), ctypes.byref(resolved)) == 0
    ctx.cap = resolved
    F.zero_()
    ctx.step_host(hp, ht, hq, F, E)
    assert np.array_equal(E.numpy(), E0) and np.array_equal(F.numpy(), F0)
    cnt, dig = [t.cpu().numpy() for t in ctx.export_digest()]
    assert np.array_equal(cnt, cnt_ref) and np.array_equal(dig, dig_ref)


def test_coarsened_plan_bitwise(params):
    """REAX_NB_GRID_FRAC=0 and REAX_NB_UNIT_FRAC=0.05 (read at bind): the
    plan overflows the launched grid and k_nb_plan doubles its unit target
    over several passes; forces and energies stay bitwise those of the
    default plan."""
    s = gen.make_config(1)
    pos, typ, q = (torch.from_numpy(x).to(DEV) for x in (s.pos, s.type, s.q))
    a = rx.Reax(len(s.pos), s.box, params, CUT, device=DEV)
    Fa, Ea = (t.clone() for t in a.step(pos, typ, q))
    os.environ["REAX_NB_GRID_FRAC"] = "0"
    os.environ["REAX_NB_UNIT_FRAC"] = "0.05"
    try:
        b = rx.Reax(len(s.pos), s.box, params, CUT, device=DEV)
    finally:
        del os.environ["REAX_NB_GRID_FRAC"], os.environ["REAX_NB_UNIT_FRAC"]
    for _ in range(2):
        Fb, Eb = b.step(pos, typ, q)
        assert torch.equal(Fb, Fa) and torch.equal(Eb, Ea)


def test_err_range_close_pair(params):
    """Two atoms 0.2 A apart with a huge vdW well depth: the pair force is far
    beyond the fixed-point accumulator (2^16 kcal/mol/A): REAX_ERR_RANGE,
    reported as the documented status (not silently wrong forces)."""
    p = params.copy()
    p.eps = np.full_like(p.eps, 1.0e7)
    pos = np.array([[5.0, 5.0, 5.0], [5.2, 5.0, 5.0]])
    s = gen.System(pos, np.array([0, 0], np.int32), np.array([0.1, -0.1]), np.array([25.0, 25.0, 25.0]))
    with pytest.raises(rx.ReaxError) as ei:
        gpu_run(s, p)
    assert ei.value.code == rx.ERR_RANGE


def test_step_host_overlapped_inputs(params):
    """reax_step_host copies the inputs on its own stream (the types are first
    needed by the cell gather, the charges by the nonbonded kernel): the
    results equal the device-input step bitwise at c1, the checks that moved
    with the inputs (type range in the cell gather, non-finite charges in the
    charge gather) still report, and the context works afterwards."""
    s = gen.make_config(1)
    n = len(s.pos)
    ctx = rx.Reax(n, s.box, params, CUT, device=DEV)
    pos, typ, q = _host(s)
    F = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    E = torch.empty(2, dtype=torch.float64).pin_memory()
    Fd, Ed = ctx.step(pos.to(DEV), typ.to(DEV), q.to(DEV))
    for _ in range(3):   # direct + capture, then graph replays
        F.zero_()
        ctx.step_host(pos, typ, q, F, E)
        assert np.array_equal(F.numpy(), Fd.cpu().numpy()) and np.array_equal(E.numpy(), Ed.cpu().numpy())
    bad = typ.clone().pin_memory()
    bad[11] = params.ntypes + 2
    with pytest.raises(rx.ReaxError) as e:
        ctx.step_host(pos, bad, q, F, E)
    assert e.value.code == rx.ERR_ARG
    qn = q.clone().pin_memory()
    qn[5] = float("nan")
    with pytest.raises(rx.ReaxError) as e:
        ctx.step_host(pos, typ, qn, F, E)
    assert e.value.code == rx.ERR_NONFINITE
    ctx.step_host(pos, typ, q, F, E)
    assert np.array_equal(F.numpy(), Fd.cpu().numpy()) and np.array_equal(E.numpy(), Ed.cpu().numpy())
