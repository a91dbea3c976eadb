"""ctypes binding of libtmg.so (include/tmg.h).

Loads the in-tree library; there is no fallback: a missing or unloadable
library raises ``ImportError``-style ``RuntimeError`` at first use, and every
non-zero status is turned into the exception the reference raises for the
same condition (ValueError / ArithmeticError / RuntimeError).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtmg.so")

TMG_OK, TMG_EINVAL, TMG_EDEGENERATE, TMG_ECUDA = 0, 1, 2, 3
VARIANT_IDS = {"additive": 0, "additive-exp": 1, "bpx": 2, "afacc": 3, "adafac-pi": 4,
               "adafac-jac": 5, "multiplicative-v10": 6}
FLAVOR_IDS = {"geometric": 0, "boxmg": 1}
TABLE_A, TABLE_DIAG, TABLE_P, TABLE_RT, TABLE_EFFEPS = 0, 1, 2, 3, 4
PH_DOWN, PH_SMOOTH, PH_REPL, PH_UP, PH_INJECT, PH_REDUCE, PH_SMR = 0, 1, 2, 3, 4, 5, 6
F_U, F_RHO, F_SM, F_CARRY, F_G, F_PART = 0, 1, 2, 3, 4, 5

EXPORTS = ("tmg_create", "tmg_rebuild", "tmg_set_rhs", "tmg_set_u", "tmg_get_u",
           "tmg_update_fas_state", "tmg_cycle", "tmg_residual_stats", "tmg_levels",
           "tmg_level_counts", "tmg_level_tiles", "tmg_get_kinds", "tmg_get_table", "tmg_time_cycles",
           "tmg_profile_cycles", "tmg_launches_per_cycle", "tmg_destroy", "tmg_last_error",
           "tmg_device_count", "tmg3_create", "tmg3_rebuild", "tmg_dim", "tmg3_shard", "tmg3_phase", "tmg3_phase_range",
           "tmg3_field", "tmg3_stream", "tmg3_history", "tmg3_storage", "tmg3_fused", "tmg3_cycle_state")


class Config(C.Structure):
    _fields_ = [("variant", C.c_int32), ("flavor", C.c_int32), ("omega", C.c_double),
                ("omega_tilde", C.c_double), ("omega_hat", C.c_double),
                ("damping_scale", C.c_double), ("rtilde_true_operator", C.c_int32),
                ("device", C.c_int32), ("throttled", C.c_int32), ("fused_cycle", C.c_int32)]


class Tree(C.Structure):
    _fields_ = [("lmin", C.c_int32), ("lmax", C.c_int32), ("nlevels", C.c_int32),
                ("refined", C.POINTER(C.POINTER(C.c_uint8))),
                ("eps", C.POINTER(C.POINTER(C.c_double))),
                ("u", C.POINTER(C.POINTER(C.c_double)))]


class Tree3(C.Structure):
    _fields_ = [("lmin", C.c_int32), ("depth", C.c_int32), ("eps", C.POINTER(C.c_double)),
                ("u", C.POINTER(C.POINTER(C.c_double)))]


class Stats(C.Structure):
    _fields_ = [("l2h", C.c_double), ("linf", C.c_double), ("dofs", C.c_int64),
                ("updates", C.c_int64)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                           "`python -m paper_1903_10367_b200.build` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    H = C.c_void_p
    P = C.POINTER
    sig = {
        "tmg_create": ([P(Tree), P(Config), P(H)], C.c_int),
        "tmg_rebuild": ([H, P(Tree)], C.c_int),
        "tmg_set_rhs": ([H, C.c_int32, C.c_void_p], C.c_int),
        "tmg_set_u": ([H, C.c_int32, C.c_void_p], C.c_int),
        "tmg_get_u": ([H, C.c_int32, C.c_void_p], C.c_int),
        "tmg_update_fas_state": ([H], C.c_int),
        "tmg_cycle": ([H, C.c_int32, C.c_void_p], C.c_int),
        "tmg_residual_stats": ([H, P(Stats)], C.c_int),
        "tmg_levels": ([H, P(C.c_int32), P(C.c_int32)], C.c_int),
        "tmg_level_counts": ([H, C.c_int32, P(C.c_int64), P(C.c_int64), P(C.c_int64)], C.c_int),
        "tmg_level_tiles": ([H, C.c_int32, P(C.c_int64), P(C.c_int64)], C.c_int),
        "tmg_get_kinds": ([H, C.c_int32, C.c_void_p], C.c_int),
        "tmg_get_table": ([H, C.c_int32, C.c_int32, C.c_void_p], C.c_int),
        "tmg_time_cycles": ([H, C.c_int32, C.c_int64, P(C.c_float)], C.c_int),
        "tmg_profile_cycles": ([H, C.c_int32, C.c_int32, P(C.c_char_p), P(C.c_float),
                                P(C.c_int32), P(C.c_int32)], C.c_int),
        "tmg_launches_per_cycle": ([H, P(C.c_int32)], C.c_int),
        "tmg_destroy": ([H], None),
        "tmg_last_error": ([], C.c_char_p),
        "tmg_device_count": ([], C.c_int),
        "tmg3_create": ([P(Tree3), P(Config), P(H)], C.c_int),
        "tmg3_rebuild": ([H, P(Tree3)], C.c_int),
        "tmg_dim": ([H], C.c_int),
        "tmg3_shard": ([H, C.c_int32, P(C.c_int32), P(C.c_int32)], C.c_int),
        "tmg3_phase": ([H, C.c_int32, C.c_int32], C.c_int),
        "tmg3_phase_range": ([H, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32], C.c_int),
        "tmg3_field": ([H, C.c_int32, C.c_int32, P(C.c_uint64), P(C.c_int64)], C.c_int),
        "tmg3_stream": ([H, P(C.c_uint64)], C.c_int),
        "tmg3_storage": ([H, C.c_int32, P(C.c_int64)], C.c_int),
        "tmg3_fused": ([H, C.c_int32, P(C.c_int32)], C.c_int),
        "tmg3_history": ([H, C.c_int32, C.c_void_p], C.c_int),
        "tmg3_cycle_state": ([H, P(C.c_int64), P(C.c_int32), C.c_int32], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == TMG_OK:
        return
    msg = lib().tmg_last_error().decode()
    if rc == TMG_EINVAL:
        raise ValueError(msg)
    if rc == TMG_EDEGENERATE:
        raise ArithmeticError(msg)
    raise RuntimeError(f"libtmg: {msg}")


def ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class TreeArgs:
    """Keeps the contiguous copies alive while libtmg reads them."""

    def __init__(self, tree):
        lmax = tree.lmax
        nlev = len(tree.u)
        self.ref = [np.ascontiguousarray(tree.refined[l], dtype=np.uint8) for l in range(lmax)]
        self.eps = [np.ascontiguousarray(tree.eps[l], dtype=np.float64) for l in range(nlev)]
        self.u = [np.ascontiguousarray(tree.u[l], dtype=np.float64) for l in range(nlev)]
        RP = C.POINTER(C.c_uint8)
        DP = C.POINTER(C.c_double)
        self.ref_arr = (RP * max(lmax, 1))(*[r.ctypes.data_as(RP) for r in self.ref])
        self.eps_arr = (DP * nlev)(*[e.ctypes.data_as(DP) for e in self.eps])
        self.u_arr = (DP * nlev)(*[u.ctypes.data_as(DP) for u in self.u])
        self.struct = Tree(tree.lmin, lmax, nlev, self.ref_arr, self.eps_arr, self.u_arr)


class TreeArgs3:
    """3D regular tree (paper_1903_10367_b200.spacetree3d / oracle mg3d data model)."""

    def __init__(self, tree):
        L = tree.depth
        self.eps = np.ascontiguousarray(tree.eps[L], dtype=np.float64)
        self.u = [np.ascontiguousarray(tree.u[l], dtype=np.float64) for l in range(L + 1)]
        DP = C.POINTER(C.c_double)
        self.u_arr = (DP * (L + 1))(*[u.ctypes.data_as(DP) for u in self.u])
        self.struct = Tree3(tree.lmin, L, self.eps.ctypes.data_as(DP), self.u_arr)
