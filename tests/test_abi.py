"""C-ABI boundary: the library loads and exports every symbol include/reax.h
declares; host-side validation (no GPU needed); device error paths (-m gpu)."""
import ctypes
import os
import re

import numpy as np
import pytest

import gen
import paper_1706_07772_b200 as rx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "reax.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(reax_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = rx.load_library()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(rx.EXPORTED)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rx.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    for code in range(11):
        assert len(rx.status_str(code)) > 0


def _ws(n, box, cut=(10.0, 5.0, 0.01), cap=None):
    lib = rx.load_library()
    b = (ctypes.c_double * 3)(*box)
    c = rx.Cutoffs(*cut)
    nbytes = ctypes.c_size_t()
    out = rx.Capacity()
    code = lib.reax_workspace_bytes(n, b, ctypes.byref(c), ctypes.byref(cap) if cap else None,
                                    ctypes.byref(nbytes), ctypes.byref(out))
    return code, nbytes.value, out


def test_host_validation():
    assert _ws(100, (25, 25, 25))[0] == rx.OK
    assert _ws(100, (20.0, 25, 25))[0] == rx.ERR_BOX          # needs L > 2 r_nonb
    assert _ws(100, (25, float("nan"), 25))[0] == rx.ERR_BOX
    assert _ws(100, (25, 25, 25), (10.0, 11.0, 0.01))[0] == rx.ERR_CUTOFF
    assert _ws(100, (25, 25, 25), (10.0, 5.0, 1.0))[0] == rx.ERR_CUTOFF
    assert _ws(100, (25, 25, 25), (10.0, 5.0, 0.0))[0] == rx.ERR_CUTOFF
    assert _ws(100, (25, 25, 25), (-1.0, -2.0, 0.01))[0] == rx.ERR_CUTOFF
    assert _ws(-1, (25, 25, 25))[0] == rx.ERR_ARG


def test_workspace_sizing_scales():
    c, b1, cap1 = _ws(32480, (69.3,) * 3)
    c, b2, cap2 = _ws(259840, (138.6,) * 3)
    assert b2 > 7 * b1
    assert cap1.row_cap >= 1.3 * 204.6 + 96 and cap1.window_cap == 2048 and cap1.cand_cap == 16   # rows ~170-290 at c1
    c, b4, cap4 = _ws(16588000, (553.6,) * 3)
    assert b4 < 60e9  # fits in one B200 with room to spare


@pytest.mark.gpu
def test_device_error_paths(params):
    import torch
    dev = torch.device("cuda:0")
    s = gen.make_config(0)
    n = len(s.pos)
    ctx = rx.Reax(n, s.box, params, gen.CUTOFFS, device=dev)
    pos = torch.from_numpy(s.pos).to(dev)
    typ = torch.from_numpy(s.type).to(dev)
    q = torch.from_numpy(s.q).to(dev)
    # nonbonded before any list build
    with pytest.raises(rx.ReaxError) as e:
        ctx.nonbonded(pos, typ, q)
    assert e.value.code == rx.ERR_STATE
    ctx.build_lists(pos, typ)
    # different position buffer than the one the lists were built from
    with pytest.raises(rx.ReaxError) as e:
        ctx.nonbonded(pos.clone(), typ, q)
    assert e.value.code == rx.ERR_STATE
    # type out of range
    bad = typ.clone()
    bad[7] = 9
    with pytest.raises(rx.ReaxError) as e:
        ctx.build_lists(pos, bad)
    assert e.value.code == rx.ERR_ARG
    # non-finite position / charge
    pn = pos.clone()
    pn[3, 1] = float("nan")
    with pytest.raises(rx.ReaxError) as e:
        ctx.build_lists(pn, typ)
    assert e.value.code == rx.ERR_NONFINITE
    qn = q.clone()
    qn[5] = float("inf")
    with pytest.raises(rx.ReaxError) as e:
        ctx.step(pos, typ, qn)
    assert e.value.code == rx.ERR_NONFINITE
    # bad parameter table
    p2 = params.copy()
    p2.eps[1] = float("nan")
    ctx2 = rx.Reax(n, s.box, p2, gen.CUTOFFS, device=dev)
    with pytest.raises(rx.ReaxError) as e:
        ctx2.step(pos, typ, q)
    assert e.value.code == rx.ERR_PARAM
    p3 = params.copy()
    p3.p_bo2 = p3.p_bo2.copy()
    p3.p_bo2[0, 1] += 1.0
    ctx3 = rx.Reax(n, s.box, p3, gen.CUTOFFS, device=dev)
    with pytest.raises(rx.ReaxError) as e:
        ctx3.step(pos, typ, q)
    assert e.value.code == rx.ERR_PARAM
    # wrong grid for the bound workspace
    ctx.set_box((40.0, 28.1, 26.8))
    with pytest.raises(rx.ReaxError) as e:
        ctx.step(pos, typ, q)
    assert e.value.code == rx.ERR_STATE
    # the context still works afterwards
    ctx.set_box(s.box)
    F, E = ctx.step(pos, typ, q)
    assert torch.isfinite(E).all()


@pytest.mark.gpu
def test_step_host_matches_device(params):
    import torch
    s = gen.make_config(0)
    n = len(s.pos)
    ctx = rx.Reax(n, s.box, params, gen.CUTOFFS, device=torch.device("cuda:0"))
    pos = torch.from_numpy(s.pos).pin_memory()
    typ = torch.from_numpy(s.type).pin_memory()
    q = torch.from_numpy(s.q).pin_memory()
    F = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    E = torch.empty(2, dtype=torch.float64).pin_memory()
    ctx.step_host(pos, typ, q, F, E)
    Fd, Ed = ctx.step(pos.cuda(), typ.cuda(), q.cuda())
    assert np.array_equal(E.numpy(), Ed.cpu().numpy())
    assert np.allclose(F.numpy(), Fd.cpu().numpy(), rtol=1e-12, atol=1e-12)
