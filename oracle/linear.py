"""ctypes wrapper for the fp64 C oracle (oracle/linear.c).

ORACLE — test infrastructure only (see oracle/__init__.py).  Inputs are the
exact bf16 bit patterns the GPU receives (numpy uint16), widened to fp64 here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "linear.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


class _Adapter(ctypes.Structure):
    _fields_ = [("A", ctypes.c_void_p), ("B", ctypes.c_void_p),
                ("dA", ctypes.c_void_p), ("dB", ctypes.c_void_p),
                ("rank", ctypes.c_int32), ("scale", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, fp64, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        for fn in (_lib.oracle_linear_fwd, _lib.oracle_linear_bwd):
            fn.restype = ctypes.c_int
        _lib.oracle_linear_fwd.argtypes = [ctypes.c_int, P, P, ctypes.c_int, P, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int, P, P, P, ctypes.c_int64, P, P]
        _lib.oracle_linear_bwd.argtypes = [ctypes.c_int, P, P, ctypes.c_int, P, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int, P, P, P, P, ctypes.c_int64, P, P]
        _lib.oracle_num_threads.restype = ctypes.c_int
        _lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
    return _lib


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count (timing only; results are bitwise the same at any count)."""
    lib().oracle_set_num_threads(int(n))


def widen(x) -> np.ndarray:
    """bf16 bits (uint16) -> float64; float arrays are passed through as float64."""
    x = np.asarray(x)
    if x.dtype == np.uint16:
        return np.ascontiguousarray((x.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64))
    return np.ascontiguousarray(x, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _adapter_table(A_list, B_list, ranks, scales, K, N, want_grads):
    keep = []
    tab = (_Adapter * max(1, len(ranks)))()
    grads = []
    for t, r in enumerate(ranks):
        A = widen(A_list[t]).reshape(r, K) if r > 0 else np.zeros((0, K))
        B = widen(B_list[t]).reshape(N, r) if r > 0 else np.zeros((N, 0))
        keep += [A, B]
        dA = np.zeros((r, K)) if want_grads else None
        dB = np.zeros((N, r)) if want_grads else None
        grads.append((dA, dB))
        tab[t] = _Adapter(A.ctypes.data if r > 0 else None, B.ctypes.data if r > 0 else None,
                          dA.ctypes.data if (want_grads and r > 0) else None,
                          dB.ctypes.data if (want_grads and r > 0) else None,
                          int(r), float(scales[t]))
    return tab, keep, grads


def linear_fwd(seg_off, seg_task, A_list, B_list, ranks, scales, X, W, r_cap, rows=None):
    """Returns (Y, Hs).  Y is [len(rows), N] if rows is given, else [R, N]
    (rows outside every segment are NaN = not computed).  Hs is [R, r_cap]."""
    seg_off = np.ascontiguousarray(seg_off, dtype=np.int32)
    seg_task = np.ascontiguousarray(seg_task, dtype=np.int32)
    Xd, Wd = widen(X), widen(W)
    N, K = Wd.shape
    R = int(seg_off[-1])
    Xd = Xd.reshape(-1, K)
    tab, keep, _ = _adapter_table(A_list, B_list, ranks, scales, K, N, False)
    rows_a = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    nr = R if rows_a is None else len(rows_a)
    Y = np.full((nr, N), np.nan)
    Hs = np.full((max(R, 0), r_cap), np.nan)
    rc = lib().oracle_linear_fwd(len(seg_task), _ptr(seg_off), _ptr(seg_task), len(ranks), tab,
                                 K, N, r_cap, _ptr(Xd), _ptr(Wd), _ptr(rows_a), nr, _ptr(Y), _ptr(Hs))
    assert rc == 0
    return Y, Hs


def linear_bwd(seg_off, seg_task, A_list, B_list, ranks, scales, dY, X, W, r_cap, rows=None):
    """Returns (dX, Gs, [(dA_t, dB_t)])."""
    seg_off = np.ascontiguousarray(seg_off, dtype=np.int32)
    seg_task = np.ascontiguousarray(seg_task, dtype=np.int32)
    dYd, Xd, Wd = widen(dY), widen(X), widen(W)
    N, K = Wd.shape
    R = int(seg_off[-1])
    Xd = Xd.reshape(-1, K)
    dYd = dYd.reshape(-1, N)
    tab, keep, grads = _adapter_table(A_list, B_list, ranks, scales, K, N, True)
    rows_a = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    nr = R if rows_a is None else len(rows_a)
    dX = np.full((nr, K), np.nan)
    Gs = np.full((max(R, 0), r_cap), np.nan)
    rc = lib().oracle_linear_bwd(len(seg_task), _ptr(seg_off), _ptr(seg_task), len(ranks), tab,
                                 K, N, r_cap, _ptr(dYd), _ptr(Xd), _ptr(Wd), _ptr(rows_a), nr,
                                 _ptr(dX), _ptr(Gs))
    assert rc == 0
    return dX, Gs, grads


# ---------------------------------------------------------------- fused projections (column slices)
def linear_fwd_sliced(seg_off, seg_task, col_off, A, B, ranks, scales, X, W, r_cap, rows=None):
    """A fused projection = one independent LoRA linear per column slice s (include/mux.h, "Fused
    projections"; P:296 on attaching adapters to the fused qkv projection): for slice s,
    Y[:, col_off[s]:col_off[s+1]] = X W_s^T + s_{t,s} (X A_{t,s}^T) B_{t,s}^T with W_s the slice's
    rows of W.  A/B/ranks/scales are indexed [t][s].  Returns (Y, Hs) with Hs [R, S * r_cap]
    (slice s in columns [s * r_cap, (s + 1) * r_cap)) — the definition written out: one
    linear_fwd per slice, concatenated."""
    Wd = widen(W)
    S = len(col_off) - 1
    Ys, Hss = [], []
    for s in range(S):
        c0, c1 = col_off[s], col_off[s + 1]
        Y_s, Hs_s = linear_fwd(seg_off, seg_task, [a[s] for a in A], [b[s] for b in B], [r[s] for r in ranks],
                               [c[s] for c in scales], X, Wd[c0:c1], r_cap, rows=rows)
        Ys.append(Y_s)
        Hss.append(Hs_s)
    return np.concatenate(Ys, axis=1), np.concatenate(Hss, axis=1)


def linear_bwd_sliced(seg_off, seg_task, col_off, A, B, ranks, scales, dY, X, W, r_cap, rows=None):
    """Backward of linear_fwd_sliced: slice s sees dY's columns of the slice; dX is the sum over
    slices (ascending s) of each slice's dX_s = dY_s W_s + Gs_s A_{t,s} (so dX = dY W + sum_s
    Gs_s A_{t,s}).  Returns (dX, Gs [R, S * r_cap], grads[t][s] = (dA_{t,s}, dB_{t,s}))."""
    Wd = widen(W)
    dYd = widen(dY)
    N = Wd.shape[0]
    dYd = dYd.reshape(-1, N)
    S = len(col_off) - 1
    dX = None
    Gss = []
    grads = [[None] * S for _ in range(len(ranks))]
    for s in range(S):
        c0, c1 = col_off[s], col_off[s + 1]
        dX_s, Gs_s, g_s = linear_bwd(seg_off, seg_task, [a[s] for a in A], [b[s] for b in B],
                                     [r[s] for r in ranks], [c[s] for c in scales],
                                     np.ascontiguousarray(dYd[:, c0:c1]), X, Wd[c0:c1], r_cap, rows=rows)
        dX = dX_s if dX is None else dX + dX_s
        Gss.append(Gs_s)
        for t in range(len(ranks)):
            grads[t][s] = g_s[t]
    return dX, np.concatenate(Gss, axis=1), grads
