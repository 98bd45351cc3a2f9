"""Seeded synthetic inputs (positions, types, charges, parameter table).

INPUT ONLY: shared by the oracle (tests / bench cpu_baseline) and the CUDA
path; holds none of the method's arithmetic.  The recipe is in
``gen/reaxgen.c`` and DESIGN.md "Input recipe".  The five configs are
BASELINE.json ``configs[0..4]`` (PETN-shaped C5H8N4O12 systems standing in
for the LAMMPS PETN benchmark of PAPER.md:243, which is not available).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "reaxgen.c")
_LIB = os.path.join(_HERE, "libreaxgen.so")

SEED_BASE = 1706077720
DMIN = 0.9
NTYPES = 4
TYPE_NAMES = ("C", "H", "N", "O")
VALENCE = (4.0, 1.0, 3.0, 2.0)  # SURVEY.md §8(c) point 10
P_BOC1, P_BOC2, P_VDW1, COULOMB_C = 50.0, 9.5, 1.55, 332.0638  # §8(c) points 10-11

# (N, box) of BASELINE.json configs[0..4]; evals = repeated evaluations
CONFIGS = {
    0: dict(n=2088, box=(28.1, 28.1, 26.8), evals=1),
    1: dict(n=32480, box=(69.3, 69.3, 69.3), evals=100),
    2: dict(n=259840, box=(138.6, 138.6, 138.6), evals=50),
    3: dict(n=1039360, box=(220.0, 220.0, 220.0), evals=20),
    4: dict(n=16588000, box=(553.6, 553.6, 553.6), evals=5),
}
CUTOFFS = dict(r_nonb=10.0, r_bond=5.0, bo_cut=0.01)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def _get():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.gen_system.restype = ctypes.c_int64
        lib.gen_system.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        lib.gen_params.restype = None
        lib.gen_params.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        lib.gen_bond_params.restype = None
        lib.gen_bond_params.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        lib.gen_uniforms.restype = None
        lib.gen_uniforms.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
        _lib = lib
    return _lib


def uniforms(seed: int, k: int) -> np.ndarray:
    out = np.empty(k, np.float64)
    _get().gen_uniforms(seed, k, out.ctypes.data)
    return out


@dataclass
class System:
    pos: np.ndarray   # (N,3) float64, in [0, L)
    type: np.ndarray  # (N,) int32
    q: np.ndarray     # (N,) float64, neutral
    box: np.ndarray   # (3,) float64


def make_system(n: int, box, seed: int, dmin: float = DMIN) -> System:
    box = np.ascontiguousarray(box, dtype=np.float64)
    pos = np.empty((n, 3), np.float64)
    typ = np.empty(n, np.int32)
    q = np.empty(n, np.float64)
    tries = _get().gen_system(seed, n, box.ctypes.data, dmin, pos.ctypes.data, typ.ctypes.data,
                              q.ctypes.data, max(100 * n, 1000))
    if tries < 0:
        raise RuntimeError("generator failed (box too dense for dmin)")
    return System(pos, typ, q, box)


def make_config(k: int) -> System:
    c = CONFIGS[k]
    return make_system(c["n"], c["box"], SEED_BASE + k)


@dataclass
class Params:
    """Synthetic ReaxFF parameter table (same for all configs)."""
    ntypes: int
    r_sigma: np.ndarray
    r_pi: np.ndarray
    r_pipi: np.ndarray
    gamma: np.ndarray
    r_vdw: np.ndarray
    eps: np.ndarray
    alpha: np.ndarray
    gamma_w: np.ndarray
    b131: np.ndarray
    b132: np.ndarray
    b133: np.ndarray
    val: np.ndarray
    val_boc: np.ndarray
    p_bo1: np.ndarray  # (ntypes, ntypes) symmetric
    p_bo2: np.ndarray
    p_bo3: np.ndarray
    p_bo4: np.ndarray
    p_bo5: np.ndarray
    p_bo6: np.ndarray
    De: np.ndarray
    p_boc1: float = P_BOC1
    p_boc2: float = P_BOC2
    p_vdw1: float = P_VDW1
    coulomb_c: float = COULOMB_C

    PER_TYPE = ("r_sigma", "r_pi", "r_pipi", "gamma", "r_vdw", "eps", "alpha", "gamma_w",
                "b131", "b132", "b133", "val", "val_boc")
    PER_PAIR = ("p_bo1", "p_bo2", "p_bo3", "p_bo4", "p_bo5", "p_bo6", "De")

    def copy(self) -> "Params":
        kw = {f: (getattr(self, f).copy() if isinstance(getattr(self, f), np.ndarray) else getattr(self, f))
              for f in self.__dataclass_fields__}
        return Params(**kw)


def make_params(seed: int = SEED_BASE, ntypes: int = NTYPES) -> Params:
    pt = np.empty((ntypes, 11), np.float64)
    pp = np.empty((ntypes, ntypes, 7), np.float64)
    _get().gen_params(seed, ntypes, pt.ctypes.data, pp.ctypes.data)
    val = np.array([VALENCE[t % 4] for t in range(ntypes)], np.float64)
    cols = [np.ascontiguousarray(pt[:, k]) for k in range(11)]
    pcols = [np.ascontiguousarray(pp[:, :, k]) for k in range(7)]
    return Params(ntypes, *cols, val, val.copy(), *pcols)


BOND_SEED = SEED_BASE + 7000


@dataclass
class BondParams:
    """Bond-energy parameters per type pair (NEXT-1; reading 28).
    De_sigma is Params.De."""
    De_pi: np.ndarray     # (ntypes, ntypes) symmetric
    De_pipi: np.ndarray
    p_be1: np.ndarray
    p_be2: np.ndarray

    FIELDS = ("De_pi", "De_pipi", "p_be1", "p_be2")

    def copy(self) -> "BondParams":
        return BondParams(*(getattr(self, f).copy() for f in self.FIELDS))


def make_bond_params(seed: int = BOND_SEED, ntypes: int = NTYPES) -> BondParams:
    pp = np.empty((ntypes, ntypes, 4), np.float64)
    _get().gen_bond_params(seed, ntypes, pp.ctypes.data)
    return BondParams(*(np.ascontiguousarray(pp[:, :, k]) for k in range(4)))


QEQ_SEED = SEED_BASE + 8000


@dataclass
class QEqParams:
    """QEq parameters per type (NEXT-2; reading 33): electronegativity
    chi (kcal/mol/e) and hardness eta = H_ii (kcal/mol/e^2)."""
    chi: np.ndarray
    eta: np.ndarray

    def copy(self) -> "QEqParams":
        return QEqParams(self.chi.copy(), self.eta.copy())


def make_qeq_params(seed: int = QEQ_SEED, ntypes: int = NTYPES) -> QEqParams:
    """chi ~ U[80, 200] kcal/mol/e (3.5-8.7 eV), eta ~ U[350, 500] kcal/mol/e^2
    (ReaxFF's 2 eta of 7.6-10.8 eV): per type, chi then eta, from SplitMix64."""
    u = uniforms(seed, 2 * ntypes)
    return QEqParams(80.0 + 120.0 * u[:ntypes], 350.0 + 150.0 * u[ntypes:])
