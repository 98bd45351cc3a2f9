"""Thin Python binding of libreax (include/reax.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; there is
no CPU fallback.  If ``libreax.so`` is missing or CUDA is unavailable the
calls raise.  PyTorch provides device memory (the bound workspace, outputs)
and the stream.

Names follow the paper's kernels (arXiv:1706.07772 Table 2):
``build_lists`` (Write Lists + bond list of Init. Forces), ``bond_orders``
(Bond Orders), ``nonbonded`` (Non-Bonded Forces, Alg. 2), ``step`` (all).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("REAX_LIBRARY", os.path.join(_HERE, "libreax.so"))

(OK, ERR_ARG, ERR_BOX, ERR_CUTOFF, ERR_PARAM, ERR_CAPACITY, ERR_NONFINITE, ERR_CUDA, ERR_STATE, ERR_RANGE,
 ERR_CONVERGENCE) = range(11)
KERNEL_GROUPS = ("bin", "nbr", "bonds", "bond_orders", "nonbonded", "other", "bond_energy", "species", "qeq")
EXPORTED = ("reax_status_str", "reax_create", "reax_destroy", "reax_workspace_bytes", "reax_bind_workspace",
            "reax_required", "reax_build_lists", "reax_bond_orders", "reax_nonbonded", "reax_step",
            "reax_step_host", "reax_set_async", "reax_check", "reax_set_timing", "reax_kernel_ms",
            "reax_launches_per_step", "reax_pair_count", "reax_export_pairs", "reax_export_nbr_digest",
            "reax_export_bonds", "reax_selftest_math", "reax_last_cuda_error", "reax_bond_energy",
            "reax_interaction_counts", "reax_interaction_lists", "reax_qeq_bytes", "reax_qeq_build",
            "reax_qeq_matvec", "reax_qeq_solve", "reax_species_bytes", "reax_species")


class ReaxError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{msg} (reax_status {code})")
        self.code = code


_D = ctypes.POINTER(ctypes.c_double)


class Cutoffs(ctypes.Structure):
    _fields_ = [("r_nonb", ctypes.c_double), ("r_bond", ctypes.c_double), ("bo_cut", ctypes.c_double)]


PER_TYPE = ("r_sigma", "r_pi", "r_pipi", "gamma", "r_vdw", "eps", "alpha", "gamma_w", "b131", "b132", "b133",
            "val", "val_boc")
PER_PAIR = ("p_bo1", "p_bo2", "p_bo3", "p_bo4", "p_bo5", "p_bo6", "De")
GLOBALS = ("p_boc1", "p_boc2", "p_vdw1", "coulomb_c")


class Params(ctypes.Structure):
    _fields_ = ([("ntypes", ctypes.c_int32)] + [(f, _D) for f in PER_TYPE] + [(f, _D) for f in PER_PAIR]
                + [(f, ctypes.c_double) for f in GLOBALS])


BOND_PAIR = ("De_pi", "De_pipi", "p_be1", "p_be2")


class BondParams(ctypes.Structure):
    _fields_ = [(f, _D) for f in BOND_PAIR]


class IListParams(ctypes.Structure):
    _fields_ = [("thb_cut", ctypes.c_double), ("thb_cutsq", ctypes.c_double), ("r_hb", ctypes.c_double),
                ("h_type", ctypes.c_int32), ("acceptor_mask", ctypes.c_uint32)]


# NEXT-3 defaults (LAMMPS ReaxFF style; readings 30-31)
ILIST_DEFAULTS = dict(thb_cut=0.001, thb_cutsq=0.00001, r_hb=7.5, h_type=1, acceptor_mask=(1 << 2) | (1 << 3))


class Capacity(ctypes.Structure):
    _fields_ = [("row_cap", ctypes.c_int32), ("cand_cap", ctypes.c_int32), ("bond_cap", ctypes.c_int64),
                ("window_cap", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libreax.so (raises if absent: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libreax.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    V, I32, I64, P = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "reax_status_str": (ctypes.c_char_p, [ctypes.c_int]),
        "reax_last_cuda_error": (ctypes.c_char_p, []),
        "reax_create": (ctypes.c_int, [ctypes.POINTER(V)]),
        "reax_destroy": (ctypes.c_int, [V]),
        "reax_workspace_bytes": (ctypes.c_int, [I64, P, P, P, ctypes.POINTER(ctypes.c_size_t), P]),
        "reax_bind_workspace": (ctypes.c_int, [V, P, ctypes.c_size_t, I64, P, P, P]),
        "reax_required": (ctypes.c_int, [V, P]),
        "reax_build_lists": (ctypes.c_int, [V, I64, P, P, P, P, P, P]),
        "reax_bond_orders": (ctypes.c_int, [V, P, P, P]),
        "reax_bond_energy": (ctypes.c_int, [V, P, P, P, P, P]),
        "reax_interaction_counts": (ctypes.c_int, [V, P, ctypes.POINTER(I64), ctypes.POINTER(I64), P]),
        "reax_interaction_lists": (ctypes.c_int, [V, P, P, P, P, P, P]),
        "reax_nonbonded": (ctypes.c_int, [V, I64, P, P, P, P, P, P, P, P, P]),
        "reax_step": (ctypes.c_int, [V, I64, P, P, P, P, P, P, P, P, P]),
        "reax_step_host": (ctypes.c_int, [V, I64, P, P, P, P, P, P, P, P, P]),
        "reax_set_async": (ctypes.c_int, [V, ctypes.c_int]),
        "reax_check": (ctypes.c_int, [V, P]),
        "reax_set_timing": (ctypes.c_int, [V, ctypes.c_int]),
        "reax_kernel_ms": (ctypes.c_int, [V, P, P, ctypes.c_int]),
        "reax_launches_per_step": (I32, [V]),
        "reax_pair_count": (ctypes.c_int, [V, ctypes.POINTER(I64), ctypes.POINTER(I64), P]),
        "reax_export_pairs": (ctypes.c_int, [V, P, P, P]),
        "reax_export_nbr_digest": (ctypes.c_int, [V, P, P, P]),
        "reax_export_bonds": (ctypes.c_int, [V, P, P, P, P, P, P]),
        "reax_selftest_math": (ctypes.c_int, [V, I64, P, P, P, P, P]),
        "reax_qeq_bytes": (ctypes.c_int, [V, ctypes.POINTER(ctypes.c_size_t), P]),
        "reax_qeq_build": (ctypes.c_int, [V, P, ctypes.c_size_t, P]),
        "reax_qeq_matvec": (ctypes.c_int, [V, P, P, ctypes.c_size_t, P, P, P, P, P]),
        "reax_qeq_solve": (ctypes.c_int, [V, P, P, ctypes.c_double, I32, P, ctypes.c_size_t, P, P, P, P, P]),
        "reax_species_bytes": (ctypes.c_int, [I64, I32, ctypes.POINTER(ctypes.c_size_t)]),
        "reax_species": (ctypes.c_int, [V, P, P, ctypes.c_size_t, P, ctypes.POINTER(I64), P, P, I64,
                                        ctypes.POINTER(I64), P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def status_str(code: int) -> str:
    return load_library().reax_status_str(code).decode()


def _check(code: int, what: str):
    if code != OK:
        msg = f"{what}: {status_str(code)}"
        if code == ERR_CUDA:
            msg += " [" + _lib.reax_last_cuda_error().decode() + "]"
        raise ReaxError(code, msg)


class _ParamsHolder:
    """ctypes reax_params with its float64 buffers kept alive."""

    def __init__(self, p):
        import numpy as np
        self.keep = []
        s = Params()
        s.ntypes = int(p.ntypes)
        for f in PER_TYPE + PER_PAIR:
            a = np.ascontiguousarray(getattr(p, f), dtype=np.float64).ravel()
            self.keep.append(a)
            setattr(s, f, a.ctypes.data_as(_D))
        for f in GLOBALS:
            setattr(s, f, float(getattr(p, f)))
        self.s = s

    @property
    def ref(self):
        return ctypes.byref(self.s)


def _stream_ptr(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dptr(t: torch.Tensor, dtype, shape=None, name="tensor"):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous {dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {shape}, got {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


class Reax:
    """One libreax context with a bound workspace for a fixed (n, cell grid)."""

    def __init__(self, n: int, box, params, cutoffs=None, capacity=None, device=None):
        self.lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("libreax needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device or "cuda")
        self.n = int(n)
        self.box = (ctypes.c_double * 3)(*[float(b) for b in box])
        cut = cutoffs or dict(r_nonb=10.0, r_bond=5.0, bo_cut=0.01)
        self.cut = Cutoffs(float(cut["r_nonb"]), float(cut["r_bond"]), float(cut["bo_cut"]))
        self.params = _ParamsHolder(params)
        self.ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(self.lib.reax_create(ctypes.byref(self.ctx)), "reax_create")
        self.cap = Capacity(0, 0, 0, 0)
        if capacity:
            for k, v in capacity.items():
                setattr(self.cap, k, int(v))
        self.ws = None
        self._bind()

    def _bind(self):
        nbytes = ctypes.c_size_t()
        resolved = Capacity()
        _check(self.lib.reax_workspace_bytes(self.n, self.box, ctypes.byref(self.cut), ctypes.byref(self.cap),
                                             ctypes.byref(nbytes), ctypes.byref(resolved)), "reax_workspace_bytes")
        self.cap = resolved
        self.ws = None
        torch.cuda.synchronize(self.device)
        self.ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
        _check(self.lib.reax_bind_workspace(self.ctx, ctypes.c_void_p(self.ws.data_ptr()), nbytes.value, self.n,
                                            self.box, ctypes.byref(self.cut), ctypes.byref(self.cap)),
               "reax_bind_workspace")
        self.workspace_bytes = int(nbytes.value)

    def _grow(self):
        need = Capacity()
        _check(self.lib.reax_required(self.ctx, ctypes.byref(need)), "reax_required")
        self.cap = need
        self._bind()

    def __del__(self):
        try:
            if getattr(self, "ctx", None) and self.ctx.value:
                self.lib.reax_destroy(self.ctx)
                self.ctx = ctypes.c_void_p()
        except Exception:
            pass

    def set_box(self, box):
        self.box = (ctypes.c_double * 3)(*[float(b) for b in box])

    # ------------------------------------------------------------- compute
    def _retry(self, fn, what, retries=8):
        for _ in range(retries):
            code = fn()
            if code != ERR_CAPACITY:
                _check(code, what)
                return
            self._grow()
        _check(code, what)

    def build_lists(self, pos: torch.Tensor, type_: torch.Tensor, stream=None):
        p = _dptr(pos, torch.float64, (self.n, 3), "pos")
        t = _dptr(type_, torch.int32, (self.n,), "type")
        self._retry(lambda: self.lib.reax_build_lists(self.ctx, self.n, p, t, self.box, self.params.ref,
                                                      ctypes.byref(self.cut), _stream_ptr(stream)),
                    "reax_build_lists")

    def bond_orders(self, stream=None):
        _check(self.lib.reax_bond_orders(self.ctx, self.params.ref, ctypes.byref(self.cut), _stream_ptr(stream)),
               "reax_bond_orders")

    def nonbonded(self, pos, type_, q, force=None, energy=None, stream=None):
        force = force if force is not None else torch.empty((self.n, 3), dtype=torch.float64, device=self.device)
        energy = energy if energy is not None else torch.empty(2, dtype=torch.float64, device=self.device)
        _check(self.lib.reax_nonbonded(self.ctx, self.n, _dptr(pos, torch.float64, (self.n, 3), "pos"),
                                       _dptr(type_, torch.int32, (self.n,), "type"),
                                       _dptr(q, torch.float64, (self.n,), "q"), self.box, self.params.ref,
                                       ctypes.byref(self.cut), _dptr(force, torch.float64, (self.n, 3), "force"),
                                       _dptr(energy, torch.float64, (2,), "energy"), _stream_ptr(stream)),
               "reax_nonbonded")
        return force, energy

    def bond_energy(self, bond_params, force=None, energy=None, stream=None):
        """reax_bond_energy (NEXT-1): E_bond and its forces at the current bond list."""
        import numpy as np
        force = force if force is not None else torch.empty((self.n, 3), dtype=torch.float64, device=self.device)
        energy = energy if energy is not None else torch.empty(1, dtype=torch.float64, device=self.device)
        keep = [np.ascontiguousarray(getattr(bond_params, f), dtype=np.float64).ravel() for f in BOND_PAIR]
        bp = BondParams(*[a.ctypes.data_as(_D) for a in keep])
        _check(self.lib.reax_bond_energy(self.ctx, self.params.ref, ctypes.byref(bp),
                                         _dptr(force, torch.float64, (self.n, 3), "force"),
                                         _dptr(energy, torch.float64, (1,), "energy"), _stream_ptr(stream)),
               "reax_bond_energy")
        return force, energy

    def interaction_lists(self, stream=None, **kw):
        """reax_interaction_counts + reax_interaction_lists (NEXT-3): the
        3-body (valence-angle) and H-bond lists as CSR in input order:
        (ang_off int64[B+1], ang_k int32[T], hb_off int64[n+1], hb_z int32[H])."""
        p = dict(ILIST_DEFAULTS, **kw)
        ip = IListParams(float(p["thb_cut"]), float(p["thb_cutsq"]), float(p["r_hb"]), int(p["h_type"]),
                         int(p["acceptor_mask"]))
        na, nh = ctypes.c_int64(), ctypes.c_int64()
        _check(self.lib.reax_interaction_counts(self.ctx, ctypes.byref(ip), ctypes.byref(na), ctypes.byref(nh),
                                                _stream_ptr(stream)), "reax_interaction_counts")
        _, B = self.pair_count(stream)
        ao = torch.empty(B + 1, dtype=torch.int64, device=self.device)
        ak = torch.empty(max(na.value, 1), dtype=torch.int32, device=self.device)
        ho = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
        hz = torch.empty(max(nh.value, 1), dtype=torch.int32, device=self.device)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())
        _check(self.lib.reax_interaction_lists(self.ctx, ctypes.byref(ip), ptr(ao), ptr(ak), ptr(ho), ptr(hz),
                                               _stream_ptr(stream)), "reax_interaction_lists")
        return ao, ak[:na.value], ho, hz[:nh.value]

    # ------------------------------------------------------------ NEXT-2 QEq
    def qeq_build(self, stream=None):
        """reax_qeq_build: H of the current half list into a scratch buffer owned
        by this object (regrown when the list needs more)."""
        need = ctypes.c_size_t()
        _check(self.lib.reax_qeq_bytes(self.ctx, ctypes.byref(need), _stream_ptr(stream)), "reax_qeq_bytes")
        if getattr(self, "_qeq_scratch", None) is None or self._qeq_scratch.numel() < need.value:
            self._qeq_scratch = None
            self._qeq_scratch = torch.empty(int(need.value), dtype=torch.uint8, device=self.device)
        _check(self.lib.reax_qeq_build(self.ctx, ctypes.c_void_p(self._qeq_scratch.data_ptr()),
                                       self._qeq_scratch.numel(), _stream_ptr(stream)), "reax_qeq_build")

    def _qeq_args(self):
        return ctypes.c_void_p(self._qeq_scratch.data_ptr()), self._qeq_scratch.numel()

    def qeq_matvec(self, eta, x_s, x_t, stream=None):
        """reax_qeq_matvec: (H x_s, H x_t) with the built H (input order)."""
        import numpy as np
        e = np.ascontiguousarray(eta, np.float64)
        ys = torch.empty(self.n, dtype=torch.float64, device=self.device)
        yt = torch.empty(self.n, dtype=torch.float64, device=self.device)
        sp, nb = self._qeq_args()
        d = lambda t, nm: _dptr(t, torch.float64, (self.n,), nm)
        _check(self.lib.reax_qeq_matvec(self.ctx, e.ctypes.data, sp, nb, d(x_s, "x_s"), d(x_t, "x_t"), d(ys, "y_s"),
                                        d(yt, "y_t"), _stream_ptr(stream)), "reax_qeq_matvec")
        return ys, yt

    def qeq_solve(self, chi, eta, tol=1e-6, maxiter=1000, s=None, t=None, q=None, stream=None):
        """reax_qeq_solve: dual Jacobi-PCG from the guesses in s, t (zeros if
        None; updated in place).  Returns (q, s, t, iters[2])."""
        import numpy as np
        c = np.ascontiguousarray(chi, np.float64)
        e = np.ascontiguousarray(eta, np.float64)
        s = s if s is not None else torch.zeros(self.n, dtype=torch.float64, device=self.device)
        t = t if t is not None else torch.zeros(self.n, dtype=torch.float64, device=self.device)
        q = q if q is not None else torch.empty(self.n, dtype=torch.float64, device=self.device)
        it = (ctypes.c_int32 * 2)()
        sp, nb = self._qeq_args()
        d = lambda x, nm: _dptr(x, torch.float64, (self.n,), nm)
        _check(self.lib.reax_qeq_solve(self.ctx, c.ctypes.data, e.ctypes.data, float(tol), int(maxiter), sp, nb,
                                       d(s, "s"), d(t, "t"), d(q, "q"), it, _stream_ptr(stream)), "reax_qeq_solve")
        return q, s, t, [it[0], it[1]]

    def qeq(self, qeq_params, tol=1e-6, maxiter=1000, s=None, t=None, q=None, stream=None):
        """H of the current lists, then the solve (NEXT-2)."""
        self.qeq_build(stream)
        return self.qeq_solve(qeq_params.chi, qeq_params.eta, tol, maxiter, s, t, q, stream)

    def species(self, bo_threshold=None, mol_id=None, stream=None):
        """reax_species (NEXT-4): molecules of the current corrected bond orders
        (bonds with BO > threshold, default 0.3) and the species census.
        Returns (mol_id int32[n] on the device, 1..M, M, comp int32[S, nt]
        (numpy, sorted), count int64[S] (numpy))."""
        import numpy as np
        nt = int(self.params.s.ntypes)
        need = ctypes.c_size_t()
        _check(self.lib.reax_species_bytes(self.n, nt, ctypes.byref(need)), "reax_species_bytes")
        if getattr(self, "_sp_scratch", None) is None or self._sp_scratch.numel() < need.value:
            self._sp_scratch = torch.empty(int(need.value), dtype=torch.uint8, device=self.device)
        mol_id = mol_id if mol_id is not None else torch.empty(self.n, dtype=torch.int32, device=self.device)
        th = None
        if bo_threshold is not None:
            th = np.ascontiguousarray(np.broadcast_to(np.asarray(bo_threshold, np.float64), (nt, nt)))
        M, S = ctypes.c_int64(), ctypes.c_int64()
        cap = getattr(self, "_sp_cap", 4096)
        while True:
            comp = np.empty((cap, nt), np.int32)
            cnt = np.empty(cap, np.int64)
            code = self.lib.reax_species(self.ctx, th.ctypes.data if th is not None else None,
                                         ctypes.c_void_p(self._sp_scratch.data_ptr()), self._sp_scratch.numel(),
                                         _dptr(mol_id, torch.int32, (self.n,), "mol_id"), ctypes.byref(M),
                                         comp.ctypes.data, cnt.ctypes.data, cap, ctypes.byref(S),
                                         _stream_ptr(stream))
            if code == ERR_CAPACITY and S.value > cap:
                cap = int(S.value)
                self._sp_cap = cap
                continue
            _check(code, "reax_species")
            return mol_id, int(M.value), comp[:S.value].copy(), cnt[:S.value].copy()

    def step(self, pos, type_, q, force=None, energy=None, stream=None):
        force = force if force is not None else torch.empty((self.n, 3), dtype=torch.float64, device=self.device)
        energy = energy if energy is not None else torch.empty(2, dtype=torch.float64, device=self.device)
        args = (_dptr(pos, torch.float64, (self.n, 3), "pos"), _dptr(type_, torch.int32, (self.n,), "type"),
                _dptr(q, torch.float64, (self.n,), "q"))
        fo = _dptr(force, torch.float64, (self.n, 3), "force")
        en = _dptr(energy, torch.float64, (2,), "energy")
        self._retry(lambda: self.lib.reax_step(self.ctx, self.n, *args, self.box, self.params.ref,
                                               ctypes.byref(self.cut), fo, en, _stream_ptr(stream)), "reax_step")
        return force, energy

    def step_host(self, pos, type_, q, force, energy, stream=None):
        """reax_step_host: CPU (ideally pinned) tensors in and out; copies inside."""
        for name, t, dt in (("pos", pos, torch.float64), ("type", type_, torch.int32), ("q", q, torch.float64),
                            ("force", force, torch.float64), ("energy", energy, torch.float64)):
            if t.is_cuda or t.dtype != dt or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous host {dt} tensor")
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        self._retry(lambda: self.lib.reax_step_host(self.ctx, self.n, P(pos), P(type_), P(q), self.box,
                                                    self.params.ref, ctypes.byref(self.cut), P(force), P(energy),
                                                    _stream_ptr(stream)), "reax_step_host")
        return force, energy

    def set_async(self, enable: bool):
        _check(self.lib.reax_set_async(self.ctx, int(bool(enable))), "reax_set_async")

    def check(self, stream=None):
        _check(self.lib.reax_check(self.ctx, _stream_ptr(stream)), "reax_check")

    def set_timing(self, enable: bool):
        _check(self.lib.reax_set_timing(self.ctx, int(bool(enable))), "reax_set_timing")

    def kernel_ms(self, reset=False, peek=False):
        ms = (ctypes.c_double * len(KERNEL_GROUPS))()
        nl = (ctypes.c_int64 * len(KERNEL_GROUPS))()
        _check(self.lib.reax_kernel_ms(self.ctx, ms, nl, 2 if peek else int(reset)), "reax_kernel_ms")
        return {k: (ms[i], nl[i]) for i, k in enumerate(KERNEL_GROUPS)}

    def launches_per_step(self) -> int:
        return int(self.lib.reax_launches_per_step(self.ctx))

    def selftest_math(self, x: torch.Tensor, stream=None):
        """Device fp64 math of the nonbonded kernel on x: columns exp, ln, rsqrt, rcp, rcbrt."""
        x = x.to(self.device, torch.float64).contiguous()
        out = torch.empty((x.numel(), 5), dtype=torch.float64, device=self.device)
        _check(self.lib.reax_selftest_math(self.ctx, x.numel(), ctypes.c_void_p(x.data_ptr()),
                                           ctypes.c_void_p(out.data_ptr()), self.params.ref, ctypes.byref(self.cut),
                                           _stream_ptr(stream)), "reax_selftest_math")
        return out

    # -------------------------------------------------------------- export
    def pair_count(self, stream=None):
        p, b = ctypes.c_int64(), ctypes.c_int64()
        _check(self.lib.reax_pair_count(self.ctx, ctypes.byref(p), ctypes.byref(b), _stream_ptr(stream)),
               "reax_pair_count")
        return p.value, b.value

    def export_pairs(self, stream=None):
        P, _ = self.pair_count(stream)
        pi = torch.empty(P, dtype=torch.int32, device=self.device)
        pj = torch.empty(P, dtype=torch.int32, device=self.device)
        if P:
            _check(self.lib.reax_export_pairs(self.ctx, ctypes.c_void_p(pi.data_ptr()),
                                              ctypes.c_void_p(pj.data_ptr()), _stream_ptr(stream)),
                   "reax_export_pairs")
        return pi, pj

    def export_digest(self, stream=None):
        cnt = torch.empty(self.n, dtype=torch.int64, device=self.device)
        dig = torch.empty(self.n, dtype=torch.int64, device=self.device)
        _check(self.lib.reax_export_nbr_digest(self.ctx, ctypes.c_void_p(cnt.data_ptr()),
                                               ctypes.c_void_p(dig.data_ptr()), _stream_ptr(stream)),
               "reax_export_nbr_digest")
        return cnt, dig

    def export_bonds(self, with_bo=True, stream=None):
        _, B = self.pair_count(stream)
        brow = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
        bcol = torch.empty(max(B, 1), dtype=torch.int32, device=self.device)
        mir = torch.empty(max(B, 1), dtype=torch.int32, device=self.device)
        bo = torch.empty((max(B, 1), 8), dtype=torch.float64, device=self.device)
        dl = torch.empty((self.n, 2), dtype=torch.float64, device=self.device)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())
        _check(self.lib.reax_export_bonds(self.ctx, ptr(brow), ptr(bcol), ptr(mir), ptr(bo) if with_bo else None,
                                          ptr(dl), _stream_ptr(stream)), "reax_export_bonds")
        return brow, bcol[:B], mir[:B], bo[:B], dl
