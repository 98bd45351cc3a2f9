"""ctypes wrapper of the C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Never imported by the
product package paper_1706_07772_b200/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11", "-pthread"]

# Row-parallel oracle (oracle.c header): results are bitwise independent of
# the thread count; ORACLE_THREADS overrides the default of all host cores.
THREADS = int(os.environ.get("ORACLE_THREADS", "0")) or (os.cpu_count() or 1)


def _t(threads):
    return int(threads) if threads else THREADS


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        subprocess.check_call(CFLAGS + ["-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


_D = ctypes.POINTER(ctypes.c_double)


class OrcParams(ctypes.Structure):
    _fields_ = ([("ntypes", ctypes.c_int32)]
                + [(f, _D) for f in ("r_sigma", "r_pi", "r_pipi", "gamma", "r_vdw", "eps", "alpha",
                                     "gamma_w", "b131", "b132", "b133", "val", "val_boc")]
                + [(f, _D) for f in ("p_bo1", "p_bo2", "p_bo3", "p_bo4", "p_bo5", "p_bo6")]
                + [(f, ctypes.c_double) for f in ("p_boc1", "p_boc2", "p_vdw1", "coulomb_c")])


class OrcBondParams(ctypes.Structure):
    _fields_ = [(f, _D) for f in ("De_s", "De_p", "De_pp", "p_be1", "p_be2")]


class _Q:
    """Bond-energy parameters (De_s = Params.De) as the oracle's struct."""

    def __init__(self, params, bparams):
        self.keep = []
        s = OrcBondParams()
        for f, a in (("De_s", params.De), ("De_p", bparams.De_pi), ("De_pp", bparams.De_pipi),
                     ("p_be1", bparams.p_be1), ("p_be2", bparams.p_be2)):
            a = np.ascontiguousarray(a, dtype=np.float64).ravel()
            self.keep.append(a)
            setattr(s, f, a.ctypes.data_as(_D))
        self.s = s

    @property
    def ref(self):
        return ctypes.byref(self.s)


class _P:
    """Keeps the numpy buffers alive alongside the ctypes struct."""

    def __init__(self, p):
        self.keep = []
        s = OrcParams()
        s.ntypes = p.ntypes
        for f in ("r_sigma", "r_pi", "r_pipi", "gamma", "r_vdw", "eps", "alpha", "gamma_w",
                  "b131", "b132", "b133", "val", "val_boc", "p_bo1", "p_bo2", "p_bo3", "p_bo4",
                  "p_bo5", "p_bo6"):
            a = np.ascontiguousarray(getattr(p, f), dtype=np.float64).ravel()
            self.keep.append(a)
            setattr(s, f, a.ctypes.data_as(_D))
        for f in ("p_boc1", "p_boc2", "p_vdw1", "coulomb_c"):
            setattr(s, f, float(getattr(p, f)))
        self.s = s

    @property
    def ref(self):
        return ctypes.byref(self.s)


_lib = None
V, I64, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
DBL, INT = ctypes.c_double, ctypes.c_int


def _get():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        sig = {
            "orc_wrap": (None, [I64, V, V, V]),
            "orc_min_image": (DBL, [DBL, DBL]),
            "orc_half_list_brute": (I64, [I64, V, V, DBL, V, V, I64]),
            "orc_half_list_cells": (I64, [I64, V, V, DBL, V, V, I64, INT]),
            "orc_digest_cells": (None, [I64, V, V, DBL, V, V, INT]),
            "orc_digest": (None, [I64, V, V, V, V]),
            "orc_mix64_pub": (U64, [U64, U64]),
            "orc_bo_raw": (None, [DBL, INT, INT, V, V]),
            "orc_bonds": (I64, [I64, V, V, V, V, DBL, DBL, V, V, V, V, V, V, I64, INT]),
            "orc_delta": (None, [I64, V, V, V, V, V]),
            "orc_bo_corr_pair": (None, [V, DBL, DBL, DBL, DBL, INT, INT, V, V, V]),
            "orc_bo_correct": (None, [I64, V, V, V, V, V, V, V, V]),
            "orc_taper": (None, [DBL, DBL, V, V]),
            "orc_vdw": (None, [DBL, INT, INT, V, V, V]),
            "orc_coulomb_kernel": (None, [DBL, INT, INT, V, V, V]),
            "orc_pair": (None, [DBL, INT, INT, DBL, DBL, V, DBL, V, V]),
            "orc_nonbonded": (None, [I64, V, V, V, V, V, DBL, V, V, V, V]),
            "orc_nonbonded_rows": (None, [I64, V, V, V, V, V, DBL, V, V, INT]),
            "orc_atom_neighbors": (I64, [I64, I64, V, V, DBL, V, I64]),
            "orc_atom_force": (None, [I64, I64, V, V, V, V, V, DBL, V, V]),
            "orc_atom_bonds": (I64, [I64, I64, V, V, V, V, DBL, DBL, V, V, V, I64]),
            "orc_bond_energy_pair": (None, [DBL, V, DBL, DBL, DBL, DBL, INT, INT, V, V, V]),
            "orc_bond_energy": (None, [I64, V, V, V, V, V, V, V, V, V, V, V, INT]),
            "orc_angles": (I64, [I64, V, V, V, DBL, DBL, V, V, I64]),
            "orc_hbonds": (I64, [I64, V, V, V, V, DBL, ctypes.c_int32, ctypes.c_uint32, V, V, I64]),
            "orc_hbonds_cells": (I64, [I64, V, V, V, V, DBL, ctypes.c_int32, ctypes.c_uint32, V, V, I64, INT]),
            "orc_species": (I64, [I64, V, INT, V, V, V, V, V, V, V, I64, V]),
            "orc_qeq_H": (None, [I64, V, V, V, V, DBL, V, V, V]),
            "orc_qeq_spmv": (None, [I64, V, V, V, V, V, V]),
            "orc_qeq": (None, [I64, V, V, V, V, DBL, V, V, V, V, DBL, INT, V, V, V, V]),
            "orc_atom_hbonds": (I64, [I64, I64, V, V, V, INT, DBL, ctypes.c_int32, ctypes.c_uint32, V, I64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _a(x, dt):
    return np.ascontiguousarray(x, dtype=dt)


def _ptr(a):
    return a.ctypes.data


def wrap(pos, box):
    pos, box = _a(pos, np.float64), _a(box, np.float64)
    out = np.empty_like(pos)
    _get().orc_wrap(len(pos), _ptr(pos), _ptr(box), _ptr(out))
    return out


def min_image(d, L):
    return _get().orc_min_image(float(d), float(L))


def half_list(pos, box, R, mode="cells", threads=None):
    """Canonical half list (rowoff int64[n+1], col int32[P]): rows i asc, j>i asc."""
    pos, box = _a(pos, np.float64), _a(box, np.float64)
    n = len(pos)
    if mode == "cells":
        T = _t(threads)
        fn = lambda *a: _get().orc_half_list_cells(*a, T)   # noqa: E731
    else:
        fn = _get().orc_half_list_brute
    rowoff = np.empty(n + 1, np.int64)
    cap = max(1, int(n * 260))
    while True:
        col = np.empty(cap, np.int32)
        p = fn(n, _ptr(pos), _ptr(box), float(R), _ptr(rowoff), _ptr(col), cap)
        if p <= cap:
            return rowoff, col[:p].copy()
        cap = int(p)


def digest(n, rowoff, col):
    cnt = np.empty(n, np.int64)
    dig = np.empty(n, np.uint64)
    _get().orc_digest(n, _ptr(_a(rowoff, np.int64)), _ptr(_a(col, np.int32)), _ptr(cnt), _ptr(dig))
    return cnt, dig


def digest_cells(pos, box, R, threads=None):
    """Per-atom (full neighbour count, sum of mix64(min, max) mod 2^64) straight
    from the cell grid: no stored list (c3/c4)."""
    pos, box = _a(pos, np.float64), _a(box, np.float64)
    n = len(pos)
    cnt = np.empty(n, np.int64)
    dig = np.empty(n, np.uint64)
    _get().orc_digest_cells(n, _ptr(pos), _ptr(box), float(R), _ptr(cnt), _ptr(dig), _t(threads))
    return cnt, dig


def mix64(a, b):
    return _get().orc_mix64_pub(int(a), int(b))


def bo_raw(r, ti, tj, params):
    P = _P(params)
    out = np.empty(4)
    _get().orc_bo_raw(float(r), int(ti), int(tj), P.ref, _ptr(out))
    return out


def bo_corr_pair(raw, di, dboci, dj, dbocj, ti, tj, params):
    P = _P(params)
    raw = _a(raw, np.float64)
    out, f = np.empty(4), np.empty(5)
    _get().orc_bo_corr_pair(_ptr(raw), float(di), float(dboci), float(dj), float(dbocj), int(ti), int(tj),
                            P.ref, _ptr(out), _ptr(f))
    return out, f


def bonds(pos, type_, box, params, r_bond, bo_cut, hrow, hcol, threads=None):
    """Full bond CSR: brow int64[n+1], bcol int32[B] (rows sorted by j), mirror int32[B]
    (absolute entry index of the reverse bond), raw float64[B,4] (BO'sigma, BO'pi, BO'pipi, BO').
    hrow = hcol = None: candidates from the cell grid at r_bond (no stored half list)."""
    P = _P(params)
    pos, box, type_ = _a(pos, np.float64), _a(box, np.float64), _a(type_, np.int32)
    if hrow is not None:
        hrow, hcol = _a(hrow, np.int64), _a(hcol, np.int32)
    hp = _ptr(hrow) if hrow is not None else None
    hc = _ptr(hcol) if hcol is not None else None
    n = len(pos)
    brow = np.empty(n + 1, np.int64)
    cap = max(16, 8 * n)
    while True:
        bcol = np.empty(cap, np.int32)
        mir = np.empty(cap, np.int32)
        raw = np.empty((cap, 4))
        B = _get().orc_bonds(n, _ptr(pos), _ptr(type_), _ptr(box), P.ref, float(r_bond), float(bo_cut),
                             hp, hc, _ptr(brow), _ptr(bcol), _ptr(mir), _ptr(raw), cap, _t(threads))
        if B <= cap:
            return brow, bcol[:B].copy(), mir[:B].copy(), raw[:B].copy()
        cap = int(B)


def delta(type_, params, brow, raw):
    P = _P(params)
    type_ = _a(type_, np.int32)
    n = len(type_)
    out = np.empty((n, 2))
    _get().orc_delta(n, _ptr(type_), P.ref, _ptr(_a(brow, np.int64)), _ptr(_a(raw, np.float64)), _ptr(out))
    return out


def bo_correct(type_, params, brow, bcol, mirror, raw, dlt):
    P = _P(params)
    type_ = _a(type_, np.int32)
    raw = _a(raw, np.float64)
    out = np.empty_like(raw)
    _get().orc_bo_correct(len(type_), _ptr(type_), P.ref, _ptr(_a(brow, np.int64)), _ptr(_a(bcol, np.int32)),
                          _ptr(_a(mirror, np.int32)), _ptr(raw), _ptr(_a(dlt, np.float64)), _ptr(out))
    return out


def taper(r, R):
    t, d = ctypes.c_double(), ctypes.c_double()
    _get().orc_taper(float(r), float(R), ctypes.addressof(t), ctypes.addressof(d))
    return t.value, d.value


def vdw(r, ti, tj, params):
    P = _P(params)
    e, d = ctypes.c_double(), ctypes.c_double()
    _get().orc_vdw(float(r), int(ti), int(tj), P.ref, ctypes.addressof(e), ctypes.addressof(d))
    return e.value, d.value


def coulomb_kernel(r, ti, tj, params):
    P = _P(params)
    e, d = ctypes.c_double(), ctypes.c_double()
    _get().orc_coulomb_kernel(float(r), int(ti), int(tj), P.ref, ctypes.addressof(e), ctypes.addressof(d))
    return e.value, d.value


def pair(r, ti, tj, qi, qj, params, R):
    """(E_vdW_pair, E_Coul_pair), dE/dr."""
    P = _P(params)
    e = np.empty(2)
    d = ctypes.c_double()
    _get().orc_pair(float(r), int(ti), int(tj), float(qi), float(qj), P.ref, float(R), _ptr(e),
                    ctypes.addressof(d))
    return e, d.value


def nonbonded(pos, type_, q, box, params, R, hrow, hcol):
    """E = [E_vdW, E_Coul], F (n,3)."""
    P = _P(params)
    pos, type_, q, box = _a(pos, np.float64), _a(type_, np.int32), _a(q, np.float64), _a(box, np.float64)
    n = len(pos)
    E = np.empty(2)
    F = np.empty((n, 3))
    _get().orc_nonbonded(n, _ptr(pos), _ptr(type_), _ptr(q), _ptr(box), P.ref, float(R),
                         _ptr(_a(hrow, np.int64)), _ptr(_a(hcol, np.int32)), _ptr(E), _ptr(F))
    return E, F


def nonbonded_rows(pos, type_, q, box, params, R, threads=None):
    """O6 row-parallel (gather over full rows from the cell grid): E = [E_vdW, E_Coul], F (n,3)."""
    P = _P(params)
    pos, type_, q, box = _a(pos, np.float64), _a(type_, np.int32), _a(q, np.float64), _a(box, np.float64)
    n = len(pos)
    E = np.empty(2)
    F = np.empty((n, 3))
    _get().orc_nonbonded_rows(n, _ptr(pos), _ptr(type_), _ptr(q), _ptr(box), P.ref, float(R), _ptr(E), _ptr(F),
                              _t(threads))
    return E, F


def atom_neighbors(i, pos, box, R):
    pos, box = _a(pos, np.float64), _a(box, np.float64)
    out = np.empty(2048, np.int32)
    m = _get().orc_atom_neighbors(int(i), len(pos), _ptr(pos), _ptr(box), float(R), _ptr(out), 2048)
    assert m <= 2048
    return out[:m].copy()


def atom_force(i, pos, type_, q, box, params, R):
    P = _P(params)
    pos, type_, q, box = _a(pos, np.float64), _a(type_, np.int32), _a(q, np.float64), _a(box, np.float64)
    F, Eh = np.empty(3), np.empty(2)
    _get().orc_atom_force(int(i), len(pos), _ptr(pos), _ptr(type_), _ptr(q), _ptr(box), P.ref, float(R),
                          _ptr(F), _ptr(Eh))
    return F, Eh


def atom_bonds(i, pos, type_, box, params, r_bond, bo_cut):
    P = _P(params)
    pos, type_, box = _a(pos, np.float64), _a(type_, np.int32), _a(box, np.float64)
    part = np.empty(64, np.int32)
    raw = np.empty((64, 4))
    dl = np.empty(2)
    m = _get().orc_atom_bonds(int(i), len(pos), _ptr(pos), _ptr(type_), _ptr(box), P.ref, float(r_bond),
                              float(bo_cut), _ptr(part), _ptr(raw), _ptr(dl), 64)
    assert m <= 64
    return part[:m].copy(), raw[:m].copy(), dl


def evaluate(system, params, cut, mode="cells", threads=None):
    """Whole path in order: wrap -> list -> bonds -> Delta' -> corrected BO -> nonbonded."""
    pos = wrap(system.pos, system.box)
    hrow, hcol = half_list(pos, system.box, cut["r_nonb"], mode, threads)
    brow, bcol, mir, raw = bonds(pos, system.type, system.box, params, cut["r_bond"], cut["bo_cut"], hrow, hcol,
                                 threads)
    dlt = delta(system.type, params, brow, raw)
    corr = bo_correct(system.type, params, brow, bcol, mir, raw, dlt)
    E, F = nonbonded_rows(pos, system.type, system.q, system.box, params, cut["r_nonb"], threads)
    return dict(pos=pos, hrow=hrow, hcol=hcol, brow=brow, bcol=bcol, mirror=mir, raw=raw, delta=dlt,
                corr=corr, E=E, F=F)


def evaluate_stream(system, params, cut, threads=None):
    """The whole path without a stored half list (c3/c4: 3.4e9 pairs at c4):
    per-atom digests of the list, the full bond list with BO', Delta' and
    corrected BO, energies and forces — each row straight from the cell grid."""
    import time
    t = [time.perf_counter()]
    pos = wrap(system.pos, system.box)
    cnt, dig = digest_cells(pos, system.box, cut["r_nonb"], threads)
    t.append(time.perf_counter())
    brow, bcol, mir, raw = bonds(pos, system.type, system.box, params, cut["r_bond"], cut["bo_cut"], None, None,
                                 threads)
    dlt = delta(system.type, params, brow, raw)
    corr = bo_correct(system.type, params, brow, bcol, mir, raw, dlt)
    t.append(time.perf_counter())
    E, F = nonbonded_rows(pos, system.type, system.q, system.box, params, cut["r_nonb"], threads)
    t.append(time.perf_counter())
    return dict(pos=pos, cnt=cnt, dig=dig, brow=brow, bcol=bcol, mirror=mir, raw=raw, delta=dlt, corr=corr,
                E=E, F=F, phase_s={"lists (per-atom rows + digests)": t[1] - t[0], "bond orders": t[2] - t[1],
                                   "nonbonded": t[3] - t[2]})


def bond_energy_pair(r, raw, di, dboci, dj, dbocj, ti, tj, params, bparams):
    """One bond (canonical orientation): [e, de/dr|_S, de/dS_i, de/dS_j, dBO'/dr] (O8)."""
    P, Q = _P(params), _Q(params, bparams)
    raw = _a(raw, np.float64)
    out = np.empty(5)
    _get().orc_bond_energy_pair(float(r), _ptr(raw), float(di), float(dboci), float(dj), float(dbocj),
                                int(ti), int(tj), P.ref, Q.ref, _ptr(out))
    return out


def bond_energy(pos, type_, box, params, bparams, brow, bcol, raw, dlt, threads=None):
    """O8 (NEXT-1): E_bond and its forces F (n,3) at a fixed bond set."""
    P, Q = _P(params), _Q(params, bparams)
    pos, type_, box = _a(pos, np.float64), _a(type_, np.int32), _a(box, np.float64)
    n = len(pos)
    F = np.empty((n, 3))
    E = ctypes.c_double()
    _get().orc_bond_energy(n, _ptr(pos), _ptr(type_), _ptr(box), P.ref, Q.ref, _ptr(_a(brow, np.int64)),
                           _ptr(_a(bcol, np.int32)), _ptr(_a(raw, np.float64)), _ptr(_a(dlt, np.float64)),
                           _ptr(F), ctypes.addressof(E), _t(threads))
    return E.value, F


def evaluate_bond_energy(system, params, bparams, cut, ref=None):
    """Lists and bond orders (evaluate()), then O8.  Returns (E_bond, F_bond, ref)."""
    if ref is None:
        ref = evaluate(system, params, cut)
    E, F = bond_energy(ref["pos"], system.type, system.box, params, bparams, ref["brow"], ref["bcol"],
                       ref["raw"], ref["delta"])
    return E, F, ref


# NEXT-3 readings: LAMMPS-ReaxFF-style defaults
ILIST = dict(thb_cut=0.001, thb_cutsq=0.00001, r_hb=7.5, h_type=1, acc_mask=(1 << 2) | (1 << 3))


def angles(brow, bcol, corr, thb_cut, thb_cutsq):
    """O9 3-body list: (ang_off int64[B+1], ang_k int32[T]) over the full bond CSR."""
    brow, bcol, corr = _a(brow, np.int64), _a(bcol, np.int32), _a(corr, np.float64)
    n = len(brow) - 1
    off = np.empty(len(bcol) + 1, np.int64)
    cap = max(1, 8 * len(bcol))
    while True:
        k = np.empty(cap, np.int32)
        t = _get().orc_angles(n, _ptr(brow), _ptr(bcol), _ptr(corr), float(thb_cut), float(thb_cutsq), _ptr(off),
                              _ptr(k), cap)
        if t <= cap:
            return off, k[:t].copy()
        cap = int(t)


def hbonds(pos, type_, box, brow, r_hb, h_type, acc_mask, mode="brute", threads=None):
    """O9 H-bond list: (hb_off int64[n+1], hb_z int32[H]) by brute force (the
    definition) or, mode="cells", from the cell grid at r_hb (row-parallel)."""
    pos, type_, box, brow = _a(pos, np.float64), _a(type_, np.int32), _a(box, np.float64), _a(brow, np.int64)
    n = len(pos)
    off = np.empty(n + 1, np.int64)
    cap = max(1, 64 * n)
    while True:
        z = np.empty(cap, np.int32)
        if mode == "cells":
            t = _get().orc_hbonds_cells(n, _ptr(pos), _ptr(type_), _ptr(box), _ptr(brow), float(r_hb), int(h_type),
                                        int(acc_mask), _ptr(off), _ptr(z), cap, _t(threads))
        else:
            t = _get().orc_hbonds(n, _ptr(pos), _ptr(type_), _ptr(box), _ptr(brow), float(r_hb), int(h_type),
                                  int(acc_mask), _ptr(off), _ptr(z), cap)
        if t <= cap:
            return off, z[:t].copy()
        cap = int(t)


def interaction_lists(system, params, cut, ilist=None, ref=None):
    """Lists and bond orders (evaluate()), then O9.  Returns (ang_off, ang_k, hb_off, hb_z, ref)."""
    il = dict(ILIST, **(ilist or {}))
    if ref is None:
        ref = evaluate(system, params, cut)
    ao, ak = angles(ref["brow"], ref["bcol"], ref["corr"], il["thb_cut"], il["thb_cutsq"])
    ho, hz = hbonds(ref["pos"], system.type, system.box, ref["brow"], il["r_hb"], il["h_type"], il["acc_mask"])
    return ao, ak, ho, hz, ref


def atom_hbonds(i, pos, type_, box, has_bond, r_hb, h_type, acc_mask):
    """O9 H-bond list of one atom (brute force)."""
    pos, type_, box = _a(pos, np.float64), _a(type_, np.int32), _a(box, np.float64)
    out = np.empty(4096, np.int32)
    m = _get().orc_atom_hbonds(int(i), len(pos), _ptr(pos), _ptr(type_), _ptr(box), int(bool(has_bond)), float(r_hb),
                               int(h_type), int(acc_mask), _ptr(out), 4096)
    assert m <= 4096
    return out[:m].copy()


# NEXT-4: default bond-order threshold of the species analysis
SPECIES_BO_THRESH = 0.3


def species(type_, ntypes, brow, bcol, corr, thresh=SPECIES_BO_THRESH):
    """O10 species analysis: (mol_id int32[n] in 1..M, M, species_comp int32[S, ntypes]
    sorted ascending, species_count int64[S])."""
    type_, brow, bcol, corr = _a(type_, np.int32), _a(brow, np.int64), _a(bcol, np.int32), _a(corr, np.float64)
    th = np.broadcast_to(np.asarray(thresh, np.float64), (ntypes, ntypes))
    th = np.ascontiguousarray(th)
    n = len(type_)
    mol = np.empty(n, np.int32)
    cap = 1024
    while True:
        comp = np.empty((cap, ntypes), np.int32)
        cnt = np.empty(cap, np.int64)
        S = ctypes.c_int64()
        M = _get().orc_species(n, _ptr(type_), int(ntypes), _ptr(brow), _ptr(bcol), _ptr(corr), _ptr(th), _ptr(mol),
                               _ptr(comp), _ptr(cnt), cap, ctypes.addressof(S))
        if S.value <= cap:
            return mol, int(M), comp[:S.value].copy(), cnt[:S.value].copy()
        cap = S.value


# NEXT-2: QEq convergence tolerance of the paper's runs
QEQ_TOL = 1e-6


def qeq_H(pos, type_, box, params, R, hrow, hcol):
    """O11: H_ij of every canonical half-list pair (aligned with hcol)."""
    P = _P(params)
    pos, type_, box = _a(pos, np.float64), _a(type_, np.int32), _a(box, np.float64)
    hrow, hcol = _a(hrow, np.int64), _a(hcol, np.int32)
    hval = np.empty(len(hcol))
    _get().orc_qeq_H(len(pos), _ptr(pos), _ptr(type_), _ptr(box), P.ref, float(R), _ptr(hrow), _ptr(hcol), _ptr(hval))
    return hval


def qeq_spmv(eta_atom, hrow, hcol, hval, x):
    eta_atom, hrow, hcol, hval, x = (_a(eta_atom, np.float64), _a(hrow, np.int64), _a(hcol, np.int32),
                                     _a(hval, np.float64), _a(x, np.float64))
    y = np.empty_like(x)
    _get().orc_qeq_spmv(len(x), _ptr(eta_atom), _ptr(hrow), _ptr(hcol), _ptr(hval), _ptr(x), _ptr(y))
    return y


def qeq(pos, type_, box, params, R, hrow, hcol, chi, eta, tol=QEQ_TOL, maxiter=1000, s0=None, t0=None):
    """O11 QEq: (q, s, t, iters[2]) with H s = -chi, H t = -1, q = s - (sum s/sum t) t."""
    P = _P(params)
    pos, type_, box = _a(pos, np.float64), _a(type_, np.int32), _a(box, np.float64)
    hrow, hcol = _a(hrow, np.int64), _a(hcol, np.int32)
    n = len(pos)
    s = np.zeros(n) if s0 is None else np.array(s0, np.float64)
    t = np.zeros(n) if t0 is None else np.array(t0, np.float64)
    q = np.empty(n)
    it = np.zeros(2, np.int32)
    _get().orc_qeq(n, _ptr(pos), _ptr(type_), _ptr(box), P.ref, float(R), _ptr(hrow), _ptr(hcol),
                   _ptr(_a(chi, np.float64)), _ptr(_a(eta, np.float64)), float(tol), int(maxiter), _ptr(s), _ptr(t),
                   _ptr(q), _ptr(it))
    return q, s, t, it
