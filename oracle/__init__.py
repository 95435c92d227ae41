"""CPU oracle for Hedtke, "Methods of Matrix Multiplication" (arXiv 1106.1347).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU legs (``cpu_baseline`` and ``--impl reference``) may import
this package.  The product package ``paper_1106_1347_b200`` never imports it,
and this package imports nothing from the product.

The arithmetic lives in ``oracle.c`` (plain C99, built ``-O2 -std=c99
-ffp-contract=off``); this module only marshals numpy arrays through ctypes.
Every function cites PAPER.md lines in ``oracle.h``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]

STRASSEN_NAIV = 0
STRASSEN_WINOGRAD = 1
BASE_LITERAL = 0
BASE_FMA = 1

M_STANDARD, M_ON_ARRAY, M_KAHAN, M_UNROLL2, M_UNROLL3, M_UNROLL4, M_FMA, M_WINOGRAD, M_WINOGRAD_SCALED = range(9)
M_KAHAN_FUSED, M_WINOGRAD_FUSED, M_WINOGRAD_SCALED_FUSED = 9, 10, 11  # NEXT-3 (reading R22)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc if it is missing or older than its sources."""
    stale = force or not os.path.exists(_LIB) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB) for s in (_SRC, _HDR))
    if stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        d, i64, i32, dp, ip = (ctypes.c_double, ctypes.c_int64, ctypes.c_int32,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64))
        L.or_selfcheck.restype = ctypes.c_int
        for name in ("or_plus", "or_minus"):
            getattr(L, name).argtypes = [dp, dp, dp, i64, i64]
        L.or_scalar_mul.argtypes = [d, dp, dp, i64, i64]
        L.or_max_d.argtypes = [d, d]
        L.or_max_d.restype = d
        L.or_max_i.argtypes = [i64, i64]
        L.or_max_i.restype = i64
        L.or_norm_inf.argtypes = [dp, i64, i64]
        L.or_norm_inf.restype = d
        for name in ("or_naive_standard", "or_naive_on_array", "or_naive_kahan", "or_naive_fma",
                     "or_winograd_original", "or_naive_kahan_fused", "or_winograd_fused"):
            getattr(L, name).argtypes = [dp, dp, dp, i64, i64, i64]
            getattr(L, name).restype = ctypes.c_int
        L.or_naive_unroll.argtypes = [ctypes.c_int, dp, dp, dp, i64, i64, i64]
        L.or_naive_fma_acc.argtypes = [dp, i64, dp, i64, dp, i64, i64, i64, i64]
        L.or_naive_kahan_acc.argtypes = [dp, i64, dp, i64, dp, dp, i64, i64, i64, ctypes.c_int]
        L.or_winograd_pairs_acc.argtypes = [dp, i64, dp, i64, dp, i64, i64, i64, ctypes.c_int]
        L.or_winograd_finish.argtypes = [dp, dp, dp, dp, i64, i64]
        L.or_winograd_yz.argtypes = [dp, dp, dp, dp, i64, i64, i64]
        L.or_winograd_yz_fused.argtypes = [dp, dp, dp, dp, i64, i64, i64]
        L.or_lambda.argtypes = [d, d]
        L.or_lambda.restype = ctypes.c_int
        L.or_winograd_scaled.argtypes = [dp, dp, dp, i64, i64, i64, ctypes.POINTER(i32)]
        L.or_winograd_scaled_fused.argtypes = [dp, dp, dp, i64, i64, i64, ctypes.POINTER(i32)]
        L.or_strassen_plan_paper.argtypes = [i64, i64, i64, ctypes.POINTER(i32), ip, ip]
        L.or_strassen_plan_levels.argtypes = [i64, i64, i64, i32, i64, ip, ip, ip]
        L.or_strassen.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, dp, i64, i64, i64, i32, i64, i64, i64]
        L.or_strassen_counters.argtypes = [ip, ip]
        L.or_strassen_trace.argtypes = [dp, i64]
        L.or_strassen_trace_len.restype = i64
        L.or_int64_gemm.argtypes = [ip, ip, ip, i64, i64, i64]
        L.or_entry.argtypes = [ctypes.c_int, dp, dp, i64, i64, i64, i64, i64, i32]
        L.or_entry.restype = d
        L.or_entry_strassen.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, i64, i64, i64, i32,
                                        i64, i64, i64, i64, i64]
        L.or_entry_strassen.restype = d
        L.or_entries.argtypes = [ctypes.c_int, dp, dp, i64, i64, i64, ip, i64, i32, dp]
        L.or_entries_strassen.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, i64, i64, i64, i32, i64, i64, i64,
                                          ip, i64, dp]
        if L.or_selfcheck() != 0:
            raise RuntimeError("oracle self-check failed (contraction or Kahan pin)")
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return a


def _ab(A, B) -> Tuple[np.ndarray, np.ndarray, int, int, int]:
    A, B = _f64(A), _f64(B)
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"inner dimensions differ: {A.shape} x {B.shape}")
    return A, B, A.shape[0], A.shape[1], B.shape[1]


# ---- Section 1 -------------------------------------------------------------
def plus(X, Y):
    X, Y = _f64(X), _f64(Y)
    Z = np.empty_like(X)
    lib().or_plus(_dp(X), _dp(Y), _dp(Z), *X.shape)
    return Z


def minus(X, Y):
    X, Y = _f64(X), _f64(Y)
    Z = np.empty_like(X)
    lib().or_minus(_dp(X), _dp(Y), _dp(Z), *X.shape)
    return Z


def scalar_mul(alpha, X):
    X = _f64(X)
    Z = np.empty_like(X)
    lib().or_scalar_mul(float(alpha), _dp(X), _dp(Z), *X.shape)
    return Z


def max2(x, y):
    if isinstance(x, (int, np.integer)) and isinstance(y, (int, np.integer)):
        return int(lib().or_max_i(int(x), int(y)))
    return float(lib().or_max_d(float(x), float(y)))


def norm_inf(X) -> float:
    X = _f64(X)
    return float(lib().or_norm_inf(_dp(X), *X.shape))


# ---- Section 2.1 / 2.2 -----------------------------------------------------
def _call3(name, A, B):
    A, B, N, P, M = _ab(A, B)
    C = np.empty((N, M), dtype=np.float64)
    rc = getattr(lib(), name)(_dp(A), _dp(B), _dp(C), N, P, M)
    if rc != 0:
        raise ValueError(f"{name} failed ({rc})")
    return C


def naive_standard(A, B):
    return _call3("or_naive_standard", A, B)


def naive_on_array(A, B):
    return _call3("or_naive_on_array", A, B)


def naive_kahan(A, B):
    return _call3("or_naive_kahan", A, B)


def naive_fma(A, B):
    return _call3("or_naive_fma", A, B)


def naive_fma_acc(A, B, C):
    """C (float64 ndarray, modified in place and returned) = A B + C, continuing each entry's
    fma chain from C (reading R2; the panel step of SURVEY 8(f) NEXT-4).  A, B may be 2-D
    row-major views (unit column stride)."""
    for X in (A, B, C):
        if X.dtype != np.float64 or X.ndim != 2 or X.strides[1] != 8:
            raise ValueError("row-major float64 matrices with unit column stride required")
    N, K = A.shape
    M = B.shape[1]
    if B.shape[0] != K or C.shape != (N, M):
        raise ValueError("shape mismatch")
    rc = lib().or_naive_fma_acc(_dp(A), A.strides[0] // 8, _dp(B), B.strides[0] // 8, _dp(C), C.strides[0] // 8,
                                N, K, M)
    if rc != 0:
        raise ValueError("or_naive_fma_acc failed")
    return C


def _panel_args(A, B, *dense):
    for X in (A, B):
        if X.dtype != np.float64 or X.ndim != 2 or X.strides[1] != 8:
            raise ValueError("row-major float64 matrices with unit column stride required")
    N, K = A.shape
    M = B.shape[1]
    for X in dense:
        if X.dtype != np.float64 or X.shape != (N, M) or not X.flags.c_contiguous:
            raise ValueError("state arrays must be dense float64 N x M")
    if B.shape[0] != K:
        raise ValueError("shape mismatch")
    return N, K, M


def naive_kahan_acc(A, B, S, E, fused: bool = False):
    """NaivKahan's update resumed from the state (S = sum, E = err; modified in
    place) over a k-panel A (N x K view), B (K x M view): the NEXT-4 panel step."""
    N, K, M = _panel_args(A, B, S, E)
    if lib().or_naive_kahan_acc(_dp(A), A.strides[0] // 8, _dp(B), B.strides[0] // 8, _dp(S), _dp(E), N, K, M,
                                int(fused)) != 0:
        raise ValueError("or_naive_kahan_acc failed")
    return S, E


def winograd_pairs_acc(A, B, Acc, fused: bool = False):
    """WinogradOriginal's pair sum resumed from Acc (modified in place) over the
    K/2 pairs of a k-panel (K even)."""
    N, K, M = _panel_args(A, B, Acc)
    if lib().or_winograd_pairs_acc(_dp(A), A.strides[0] // 8, _dp(B), B.strides[0] // 8, _dp(Acc), N, K, M,
                                   int(fused)) != 0:
        raise ValueError("or_winograd_pairs_acc failed")
    return Acc


def winograd_finish(Acc, y, z):
    """The even-P epilogue C = (acc - y_i) - z_k."""
    N, M = Acc.shape
    C = np.empty((N, M), dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    if y.shape != (N,) or z.shape != (M,):
        raise ValueError("y, z must have N and M entries")
    if lib().or_winograd_finish(_dp(np.ascontiguousarray(Acc)), _dp(y), _dp(z), _dp(C), N, M) != 0:
        raise ValueError("or_winograd_finish failed")
    return C


def winograd_yz_fused(A, B):
    """y, z of P:189 accumulated by fma (NEXT-3, reading R22)."""
    A, B, N, P, M = _ab(A, B)
    y = np.empty((N,), dtype=np.float64)
    z = np.empty((M,), dtype=np.float64)
    lib().or_winograd_yz_fused(_dp(A), _dp(B), _dp(y), _dp(z), N, P, M)
    return y, z


def naive_kahan_fused(A, B):
    """NEXT-3 (reading R22): NaivKahan with err = fma(A_ik, B_kj, err)."""
    return _call3("or_naive_kahan_fused", A, B)


def winograd_fused(A, B):
    """NEXT-3 (reading R22): WinogradOriginal with y, z, acc and the odd-P term via fma."""
    return _call3("or_winograd_fused", A, B)


def winograd_scaled_fused(A, B):
    """NEXT-3: WinogradScaled on top of winograd_fused.  Returns (C, lambda)."""
    A, B, N, P, M = _ab(A, B)
    C = np.empty((N, M), dtype=np.float64)
    lam_out = ctypes.c_int32(0)
    if lib().or_winograd_scaled_fused(_dp(A), _dp(B), _dp(C), N, P, M, ctypes.byref(lam_out)) != 0:
        raise ValueError("winograd_scaled_fused failed")
    return C, int(lam_out.value)


def naive_unroll(u: int, A, B):
    A, B, N, P, M = _ab(A, B)
    C = np.empty((N, M), dtype=np.float64)
    if lib().or_naive_unroll(int(u), _dp(A), _dp(B), _dp(C), N, P, M) != 0:
        raise ValueError("bad unroll factor")
    return C


# ---- Section 2.3 -----------------------------------------------------------
def winograd_yz(A, B):
    A, B, N, P, M = _ab(A, B)
    y = np.empty((N,), dtype=np.float64)
    z = np.empty((M,), dtype=np.float64)
    lib().or_winograd_yz(_dp(A), _dp(B), _dp(y), _dp(z), N, P, M)
    return y, z


def winograd_original(A, B):
    return _call3("or_winograd_original", A, B)


def lam(nA: float, nB: float) -> int:
    return int(lib().or_lambda(float(nA), float(nB)))


def winograd_scaled(A, B):
    """Returns (C, lambda)."""
    A, B, N, P, M = _ab(A, B)
    C = np.empty((N, M), dtype=np.float64)
    lam_out = ctypes.c_int32(0)
    if lib().or_winograd_scaled(_dp(A), _dp(B), _dp(C), N, P, M, ctypes.byref(lam_out)) != 0:
        raise ValueError("winograd_scaled failed")
    return C, int(lam_out.value)


# ---- Section 2.4 -----------------------------------------------------------
def strassen_plan_paper(N: int, P: int, M: int):
    """(k, m, Y) of P:286 (k clamped at 0)."""
    k = ctypes.c_int32()
    m = ctypes.c_int64()
    Y = ctypes.c_int64()
    lib().or_strassen_plan_paper(N, P, M, ctypes.byref(k), ctypes.byref(m), ctypes.byref(Y))
    return int(k.value), int(m.value), int(Y.value)


def strassen_plan_levels(N: int, P: int, M: int, levels: int, align: int = 2):
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    lib().or_strassen_plan_levels(N, P, M, levels, align, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return int(a.value), int(b.value), int(c.value)


def _plan(N, P, M, levels, pad):
    if levels is None or levels < 0:  # the paper's square plan
        k, _m, Y = strassen_plan_paper(N, P, M)
        return k, (Y, Y, Y)
    if pad is None:
        pad = strassen_plan_levels(N, P, M, levels)
    return levels, tuple(int(x) for x in pad)


def plan(N: int, P: int, M: int, levels: int):
    """(depth, (Np, Pp, Mp)): the paper's square plan for levels < 0, else `levels` levels with
    every dimension padded to a multiple of 2^(levels+1) (reading R10).  The same plan the library
    computes (tests/test_abi_cpu.py pins the two equal); test and bench code takes it from here so
    the oracle never depends on the product."""
    return _plan(N, P, M, levels, None)


def strassen(variant: int, A, B, levels=None, pad=None, base: int = BASE_LITERAL):
    """Strassen (variant 0) or Strassen-Winograd (variant 1).

    levels=None/-1 -> the paper's plan; otherwise `levels` recursion levels
    with the padded dims `pad` = (Np, Pp, Mp) (default: strassen_plan_levels, align 2).
    """
    A, B, N, P, M = _ab(A, B)
    lv, (Np, Pp, Mp) = _plan(N, P, M, levels, pad)
    C = np.empty((N, M), dtype=np.float64)
    rc = lib().or_strassen(int(variant), int(base), _dp(A), _dp(B), _dp(C), N, P, M, lv, Np, Pp, Mp)
    if rc != 0:
        raise ValueError(f"or_strassen failed ({rc})")
    return C


def strassen_counters():
    a, b = ctypes.c_int64(), ctypes.c_int64()
    lib().or_strassen_counters(ctypes.byref(a), ctypes.byref(b))
    return int(a.value), int(b.value)


def strassen_trace(variant: int, A, B, levels: int, cap: int = 4096) -> np.ndarray:
    """Values of the 1x1 base products (H_1..H_7 per node, call order) of or_strassen."""
    buf = np.zeros(cap, dtype=np.float64)
    L = lib()
    L.or_strassen_trace(_dp(buf), cap)
    try:
        strassen(variant, A, B, levels=levels, pad=tuple(np.shape(A)[:1]) + (np.shape(A)[1], np.shape(B)[1]))
        n = int(L.or_strassen_trace_len())
    finally:
        L.or_strassen_trace(None, 0)
    return buf[:n].copy()


def int64_gemm(A, B):
    A = np.ascontiguousarray(A, dtype=np.int64)
    B = np.ascontiguousarray(B, dtype=np.int64)
    N, P = A.shape
    M = B.shape[1]
    C = np.empty((N, M), dtype=np.int64)
    ip = ctypes.POINTER(ctypes.c_int64)
    lib().or_int64_gemm(A.ctypes.data_as(ip), B.ctypes.data_as(ip), C.ctypes.data_as(ip), N, P, M)
    return C


# ---- per entry --------------------------------------------------------------
def entry(method: int, A, B, i: int, j: int, lam_: int = 0) -> float:
    A, B, N, P, M = _ab(A, B)
    return float(lib().or_entry(int(method), _dp(A), _dp(B), N, P, M, int(i), int(j), int(lam_)))


def _ij(idx) -> np.ndarray:
    ij = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1, 2))
    return ij


def entries(method: int, A, B, idx, lam_: int = 0) -> np.ndarray:
    A, B, N, P, M = _ab(A, B)
    ij = _ij(idx)
    if ij.size and (ij[:, 0].min() < 0 or ij[:, 0].max() >= N or ij[:, 1].min() < 0 or ij[:, 1].max() >= M):
        raise IndexError("entry index out of range")
    out = np.empty(ij.shape[0], dtype=np.float64)
    lib().or_entries(int(method), _dp(A), _dp(B), N, P, M, ij.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                     ij.shape[0], int(lam_), _dp(out))
    return out


def entries_strassen(variant: int, A, B, idx, levels=None, pad=None, base: int = BASE_LITERAL) -> np.ndarray:
    A, B, N, P, M = _ab(A, B)
    lv, (Np, Pp, Mp) = _plan(N, P, M, levels, pad)
    ij = _ij(idx)
    out = np.empty(ij.shape[0], dtype=np.float64)
    lib().or_entries_strassen(int(variant), int(base), _dp(A), _dp(B), N, P, M, lv, Np, Pp, Mp,
                              ij.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ij.shape[0], _dp(out))
    return out


# ---- Brent's bounds; diagnostic formulas, u = 2^-tau -----------
def brent_bound_unscaled(n: int, nA: float, nB: float, u: float = 2.0 ** -53) -> float:
    return u * (n * n + 12 * n - 8) / 4.0 * (nA + nB) ** 2


def brent_bound_scaled(n: int, nA: float, nB: float, u: float = 2.0 ** -53) -> float:
    return u * 9.0 / 8.0 * (n * n + 12 * n - 8) * nA * nB


# ---- all ten paper methods by their paper names -------------
def paper_method(name: str, A, B):
    table = {
        "NaivStandard": naive_standard,
        "NaivOnArray": naive_on_array,
        "NaivKahan": naive_kahan,
        "NaivLoopUnrollingTwo": lambda a, b: naive_unroll(2, a, b),
        "NaivLoopUnrollingThree": lambda a, b: naive_unroll(3, a, b),
        "NaivLoopUnrollingFour": lambda a, b: naive_unroll(4, a, b),
        "WinogradOriginal": winograd_original,
        "WinogradScaled": lambda a, b: winograd_scaled(a, b)[0],
        "StrassenNaiv": lambda a, b: strassen(STRASSEN_NAIV, a, b),
        "StrassenWinograd": lambda a, b: strassen(STRASSEN_WINOGRAD, a, b),
    }
    return table[name](A, B)


PAPER_METHODS = ("NaivStandard", "NaivOnArray", "NaivLoopUnrollingTwo", "NaivLoopUnrollingThree",
                 "NaivLoopUnrollingFour", "StrassenNaiv", "StrassenWinograd", "WinogradOriginal",
                 "WinogradScaled")
