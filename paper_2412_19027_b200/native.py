"""ctypes binding of ``lib/libcipm.so`` (C ABI: ``include/cipm.h``).

The product path has no CPU fallback: if the library is missing or a CUDA
device is absent, :func:`lib` / :class:`DeviceContext` raise immediately.
Symbolic-analysis entry points are host-only and work without a GPU (they
are exercised by the CPU test suite).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .exceptions import ConicError, raise_for_status

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CIPM_LIB") or os.path.join(PKG, "lib", "libcipm.so")   # override: debugging builds only

c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_void_p = ctypes.c_void_p
P_I64 = ctypes.POINTER(ctypes.c_int64)
P_DBL = ctypes.POINTER(ctypes.c_double)

SC = dict(TAU=0, KAPPA=1, MU=2, GTAU=3, XPX=4, QX=5, BZ=6, NRM_GX=7, NRM_ATZ=8, NRM_PX=9, NRM_XU=10,
          NRM_GZ=11, NRM_AXS=12, NRM_ZU=13, NRM_SU=14, DEN=15, DTAU_A=16, DKAPPA_A=17, DTAU_C=18,
          DKAPPA_C=19, ALPHA_A=20, SIGMA=21, ALPHA_C=22, ALPHA_FINAL=23, ALPHA_WORK=32, SZ=33, BUMPS=34,
          REFINE_STEPS=35, NB_BATCH=36, BEST_FLAG=37, REF_STEPS_A=38, REF_STEPS_C=39, STATUS=40, BEST_SCORE=41,
          BEST_VALID=42, STALL_MU=43, STALL_RP=44, STALL_RD=45, STALL_CNT=46, BEST_TAU=47, BEST_KAPPA=48,
          BEST_MU=49, BEST_GP=50, BEST_GD=51, BEST_RP=52, BEST_RD=53, BEST_R1=54, BEST_R2=55, BEST_R3=56,
          CUR_R1=57, CUR_R2=58, CUR_R3=59)
SC_COUNT = 64


class ProblemDesc(ctypes.Structure):
    _fields_ = [("n", c_i64), ("m", c_i64),
                ("p_rowptr", P_I64), ("p_colidx", P_I64),
                ("a_rowptr", P_I64), ("a_colidx", P_I64),
                ("zero_dim", c_i64), ("nonneg_dim", c_i64),
                ("n_soc", c_i64), ("soc_off", P_I64), ("soc_dim", P_I64),
                ("n_exp", c_i64), ("exp_off", P_I64),
                ("n_pow", c_i64), ("pow_off", P_I64), ("pow_alpha", P_DBL),
                ("n_psd", c_i64), ("psd_off", P_I64), ("psd_side", P_I64)]


class Settings(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int), ("delta_s", c_dbl), ("delta_d", c_dbl),
                ("beta", c_dbl), ("backtrack", c_dbl), ("step_scale", c_dbl),
                ("refine_abs", c_dbl), ("refine_rel", c_dbl), ("refine_max", ctypes.c_int),
                ("device", ctypes.c_int), ("stream", c_void_p)]


class SymInfo(ctypes.Structure):
    _fields_ = [("dim", c_i64), ("nsuper", c_i64), ("nnz_l", c_i64), ("nnz_storage", c_i64),
                ("n_updates", c_i64), ("max_width", c_i64), ("max_rows", c_i64), ("height", c_i64),
                ("flops", c_dbl), ("ordering", c_i64)]


# every exported symbol of include/cipm.h with its signature
_SIGS = {
    "cipm_version": ([], ctypes.c_int),
    "cipm_symbolic_create": ([ctypes.POINTER(ProblemDesc), ctypes.c_int, ctypes.POINTER(c_void_p)], ctypes.c_int),
    "cipm_symbolic_create_ex": ([ctypes.POINTER(ProblemDesc), ctypes.c_int, c_i64, ctypes.POINTER(c_void_p)],
                                ctypes.c_int),
    "cipm_symbolic_info_get": ([c_void_p, ctypes.POINTER(SymInfo)], ctypes.c_int),
    "cipm_symbolic_array": ([c_void_p, ctypes.c_char_p, c_void_p, P_I64], ctypes.c_int),
    "cipm_symbolic_destroy": ([c_void_p], None),
    "cipm_min_degree": ([c_i64, P_I64, P_I64, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "cipm_ctx_create": ([ctypes.POINTER(ProblemDesc), c_void_p, ctypes.POINTER(Settings),
                         ctypes.POINTER(c_void_p)], ctypes.c_int),
    "cipm_ctx_set_values": ([c_void_p, P_DBL, P_DBL, P_DBL, P_DBL, P_DBL, P_DBL, c_dbl], ctypes.c_int),
    "cipm_ctx_destroy": ([c_void_p], None),
    "cipm_ctx_set_reorder": ([c_void_p, P_I64, P_I64], ctypes.c_int),
    "cipm_ctx_set_problem": ([c_void_p, P_DBL, P_DBL, P_DBL, P_DBL, ctypes.c_int], ctypes.c_int),
    "cipm_ctx_get_equilibration": ([c_void_p, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_sync": ([c_void_p], ctypes.c_int),
    "cipm_device_bytes": ([c_void_p, P_I64], ctypes.c_int),
    "cipm_init_iterate": ([c_void_p], ctypes.c_int),
    "cipm_residuals": ([c_void_p, P_DBL], ctypes.c_int),
    "cipm_save_best": ([c_void_p], ctypes.c_int),
    "cipm_update_scaling": ([c_void_p], ctypes.c_int),
    "cipm_factor": ([c_void_p], ctypes.c_int),
    "cipm_solve_affine": ([c_void_p, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cipm_step_affine": ([c_void_p], ctypes.c_int),
    "cipm_solve_combined": ([c_void_p, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cipm_step_combined": ([c_void_p, P_DBL], ctypes.c_int),
    "cipm_take_step": ([c_void_p], ctypes.c_int),
    "cipm_read_scalars": ([c_void_p, P_DBL], ctypes.c_int),
    "cipm_get_iterate": ([c_void_p, ctypes.c_int, P_DBL, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_get_solution": ([c_void_p, ctypes.c_int, ctypes.c_int, P_DBL, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_set_iterate": ([c_void_p, P_DBL, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_kkt_solve": ([c_void_p, P_DBL, P_DBL, ctypes.POINTER(ctypes.c_int), P_DBL], ctypes.c_int),
    "cipm_apply_h": ([c_void_p, P_DBL, P_DBL], ctypes.c_int),
    "cipm_scaling_values": ([c_void_p, P_DBL, P_DBL], ctypes.c_int),
    "cipm_get_direction": ([c_void_p, ctypes.c_int, P_DBL, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_get_vector": ([c_void_p, ctypes.c_char_p, P_DBL, P_I64], ctypes.c_int),
    "cipm_kkt_set_scaling": ([c_void_p, P_DBL, P_DBL], ctypes.c_int),
    "cipm_kkt_matvec": ([c_void_p, P_DBL, P_DBL], ctypes.c_int),
    "cipm_kkt_solve_ex": ([c_void_p, P_DBL, P_DBL, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                           ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cipm_set_refinement": ([c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_int], ctypes.c_int),
    "cipm_soc_residuals": ([c_void_p, P_DBL, P_DBL], ctypes.c_int),
    "cipm_set_direction": ([c_void_p, ctypes.c_int, P_DBL, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_step_length": ([c_void_p, ctypes.c_int, P_DBL], ctypes.c_int),
    "cipm_combined_ds": ([c_void_p, P_DBL, P_DBL, c_dbl, c_dbl, P_DBL], ctypes.c_int),
    "cipm_neighborhood_ok": ([c_void_p, c_dbl, c_dbl, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cipm_membership": ([c_void_p, P_DBL, P_DBL, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
                        ctypes.c_int),
    "cipm_kkt_counters": ([c_void_p, P_I64], ctypes.c_int),
    "cipm_loop_begin": ([c_void_p, c_dbl, c_dbl, c_dbl, c_dbl, ctypes.c_int], ctypes.c_int),
    "cipm_loop_check": ([c_void_p, ctypes.c_int, P_DBL], ctypes.c_int),
    "cipm_loop_body": ([c_void_p], ctypes.c_int),
    "cipm_kernel_classes": ([c_void_p, ctypes.c_int, P_DBL], ctypes.c_int),
    "cipm_launch_count": ([c_void_p, P_I64, ctypes.c_int], ctypes.c_int),
    "cipm_io_bytes": ([c_void_p, P_I64, P_I64, ctypes.c_int], ctypes.c_int),
    "cipm_kernel_times": ([c_void_p, P_DBL, P_DBL], ctypes.c_int),
    "cipm_profile": ([c_void_p, ctypes.c_int], ctypes.c_int),
    "cipm_kernel_stats": ([c_void_p, P_DBL], ctypes.c_int),
    "cipm_timer": ([c_void_p, ctypes.c_int, P_DBL], ctypes.c_int),
    "cipm_trace": ([c_void_p, ctypes.c_int, P_I64], ctypes.c_int),
    "cipm_batch_create": ([ctypes.POINTER(ProblemDesc), ctypes.c_int, ctypes.POINTER(Settings), c_dbl, c_dbl,
                           ctypes.c_int, ctypes.POINTER(c_void_p)], ctypes.c_int),
    "cipm_batch_info": ([c_void_p, P_I64], ctypes.c_int),
    "cipm_batch_set_values": ([c_void_p, P_DBL, P_DBL, P_DBL, P_DBL, P_DBL, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_batch_solve": ([c_void_p, P_DBL], ctypes.c_int),
    "cipm_batch_set_reorder": ([c_void_p, P_I64, P_I64], ctypes.c_int),
    "cipm_batch_set_raw_values": ([c_void_p, P_DBL, P_DBL, P_DBL, ctypes.c_int], ctypes.c_int),
    "cipm_batch_results": ([c_void_p, ctypes.POINTER(ctypes.c_int32), P_DBL, P_DBL, P_DBL, P_DBL], ctypes.c_int),
    "cipm_batch_io_bytes": ([c_void_p, P_I64, P_I64, ctypes.c_int], ctypes.c_int),
    "cipm_batch_destroy": ([c_void_p], None),
}

_lib = None


def lib():
    """Load libcipm.so (fails loudly: there is no fallback implementation)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native library missing: {LIB_PATH}; run "
                               "`python -m paper_2412_19027_b200.build` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def pi64(a):
    return a.ctypes.data_as(P_I64) if a is not None and a.size else None


def pdbl(a):
    return a.ctypes.data_as(P_DBL) if a is not None and a.size else None


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Layout:
    """Family-grouped cone tables of a reordered cone list (reference ConeSet, set.py:25-83)."""

    def __init__(self, cones):
        self.zero_dim = self.nonneg_dim = 0
        soc_off, soc_dim, exp_off, pow_off, pow_alpha, psd_off, psd_side = [], [], [], [], [], [], []
        off = 0
        for c in cones:
            if c.kind == "zero":
                self.zero_dim += c.dim
            elif c.kind == "nonneg":
                self.nonneg_dim += c.dim
            elif c.kind == "soc":
                soc_off.append(off)
                soc_dim.append(c.dim)
            elif c.kind == "exp":
                exp_off.append(off)
            elif c.kind == "pow":
                pow_off.append(off)
                pow_alpha.append(c.alpha)
            elif c.kind == "psd":
                psd_off.append(off)
                psd_side.append(c.side)
            off += c.dim
        self.m = off
        self.soc_off, self.soc_dim = _i64(soc_off), _i64(soc_dim)
        self.exp_off, self.pow_off = _i64(exp_off), _i64(pow_off)
        self.pow_alpha = np.ascontiguousarray(pow_alpha, dtype=np.float64)
        self.psd_off, self.psd_side = _i64(psd_off), _i64(psd_side)

    @property
    def degree(self) -> int:
        return int(self.nonneg_dim + len(self.soc_off) + 3 * len(self.exp_off) + 3 * len(self.pow_off)
                   + int(np.sum(self.psd_side)))


def make_desc(P, A, lay: Layout):
    """ProblemDesc over the (reordered) problem patterns; keep the returned refs alive."""
    keep = dict(prp=_i64(P.rowptr), pci=_i64(P.colidx), arp=_i64(A.rowptr), aci=_i64(A.colidx))
    d = ProblemDesc()
    d.n, d.m = P.nrows, A.nrows
    d.p_rowptr, d.p_colidx = pi64(keep["prp"]) or P_I64(), pi64(keep["pci"])
    d.a_rowptr, d.a_colidx = pi64(keep["arp"]), pi64(keep["aci"])
    d.zero_dim, d.nonneg_dim = lay.zero_dim, lay.nonneg_dim
    d.n_soc, d.soc_off, d.soc_dim = len(lay.soc_off), pi64(lay.soc_off), pi64(lay.soc_dim)
    d.n_exp, d.exp_off = len(lay.exp_off), pi64(lay.exp_off)
    d.n_pow, d.pow_off, d.pow_alpha = len(lay.pow_off), pi64(lay.pow_off), pdbl(lay.pow_alpha)
    d.n_psd, d.psd_off, d.psd_side = len(lay.psd_off), pi64(lay.psd_off), pi64(lay.psd_side)
    return d, keep


class SymbolicAnalysis:
    """Host symbolic analysis handle (ordering, etree, supernodes, scatter maps)."""

    ORDERINGS = {"md": 0, "natural": 1, "nd": 2, "auto": 3, "amd": 4}

    def __init__(self, P, A, lay: Layout, ordering: int = 0, nd_leaf: int = 0):
        """ordering: 0 the reference's exact minimum degree, 1 natural, 4 approximate
        minimum degree (quotient graph), 2 nested
        dissection (parts up to nd_leaf rows ordered by MD), 3 auto (MD below 20k
        rows, else ND when its fill stays close to MD's)."""
        self._desc, self._keep = make_desc(P, A, lay)
        h = c_void_p()
        rc = lib().cipm_symbolic_create_ex(ctypes.byref(self._desc), int(ordering), int(nd_leaf), ctypes.byref(h))
        raise_for_status(rc, "symbolic analysis")
        self.handle = h

    def info(self) -> dict:
        inf = SymInfo()
        raise_for_status(lib().cipm_symbolic_info_get(self.handle, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in SymInfo._fields_}

    def array(self, name: str) -> np.ndarray:
        cnt = c_i64(0)
        raise_for_status(lib().cipm_symbolic_array(self.handle, name.encode(), None, ctypes.byref(cnt)))
        dt = np.int32 if name in ("perm", "md_perm", "sn_col", "sn_rows", "sn_parent", "upd_src", "upd_p0",
                                  "upd_p1", "order", "inbox_tgt", "level", "desc32", "tiny",
                                  "tfold_cols") else (
            np.int8 if name == "tier" else np.int64)
        out = np.empty(cnt.value, dtype=dt)
        if cnt.value:
            raise_for_status(lib().cipm_symbolic_array(self.handle, name.encode(),
                                                       out.ctypes.data_as(c_void_p), ctypes.byref(cnt)))
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib().cipm_symbolic_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def min_degree(rowptr, colidx) -> np.ndarray:
    """The reference's exact minimum-degree order of a symmetric pattern (ordering.py:15-53)."""
    rp, ci = _i64(rowptr), _i64(colidx)
    n = len(rp) - 1
    perm = np.empty(n, dtype=np.int32)
    raise_for_status(lib().cipm_min_degree(n, pi64(rp), pi64(ci) or P_I64(),
                                           perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return perm.astype(np.int64)


class DeviceContext:
    """One problem instance resident on one GPU (cipm_ctx)."""

    def __init__(self, sym: SymbolicAnalysis, settings: Settings):
        self.sym = sym
        h = c_void_p()
        rc = lib().cipm_ctx_create(ctypes.byref(sym._desc), sym.handle, ctypes.byref(settings), ctypes.byref(h))
        if rc != 0:
            raise_for_status(rc, "device context creation")
        self.handle = h
        self.n = sym._desc.n
        self.m = sym._desc.m
        self.sc = np.zeros(SC_COUNT)

    # CIPM_HOST_PROFILE=1: synchronise after every call and accumulate wall time per entry point
    host_profile = os.environ.get("CIPM_HOST_PROFILE", "0") != "0"

    def call(self, name, *args, where=None):
        if self.host_profile:
            import time
            t0 = time.perf_counter()
            rc = getattr(lib(), name)(self.handle, *args)
            lib().cipm_sync(self.handle)
            prof = self.__dict__.setdefault("profile", {})
            tot, cnt = prof.get(name, (0.0, 0))
            prof[name] = (tot + time.perf_counter() - t0, cnt + 1)
        else:
            rc = getattr(lib(), name)(self.handle, *args)
        if rc is not None and rc < 0:
            raise_for_status(rc, where or name)
        return rc

    def close(self):
        if getattr(self, "handle", None):
            lib().cipm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def require_device():
    try:
        import torch
    except Exception as e:  # pragma: no cover
        raise ConicError(f"torch unavailable: {e}") from e
    if not torch.cuda.is_available():
        raise ConicError("no CUDA device: the B200 solver path has no CPU fallback")
    return torch


def pinned_empty(shape) -> np.ndarray:
    """Page-locked float64 host array from torch's caching host allocator.  Device
    copies into / out of it are plain DMA (no driver staging through pageable
    memory), and results are handed to the caller in it without another host copy.
    The ndarray keeps its tensor (and so the pinned block) alive."""
    torch = require_device()
    return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()


def pinned_copy(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    out = pinned_empty(a.shape)
    np.copyto(out, a)
    return out
