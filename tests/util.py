"""Test helpers: device staging and oracle parallelism (no method arithmetic here)."""
from __future__ import annotations

import multiprocessing
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def workers() -> int:
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(16, n))


def _rows_job(args):
    import oracle

    name, A, B, lam = args
    if name == "winograd_scaled_rows":
        # the scaled method needs the global lambda: pass it in, compute row block entries
        idx = [(i, j) for i in range(A.shape[0]) for j in range(B.shape[1])]
        return oracle.entries(oracle.M_WINOGRAD_SCALED, A, B, idx, lam).reshape(A.shape[0], B.shape[1])
    f = {
        "naive_fma": oracle.naive_fma,
        "naive_standard": oracle.naive_standard,
        "naive_kahan": oracle.naive_kahan,
        "winograd_original": oracle.winograd_original,
    }[name]
    return f(A, B)


def oracle_rows(name: str, A: np.ndarray, B: np.ndarray, lam: int = 0) -> np.ndarray:
    """Row-independent oracle functions evaluated on row blocks in parallel processes.
    Each entry depends only on its row of A and its column of B, so the result is bitwise
    the full-matrix oracle's."""
    nw = workers()
    if nw == 1 or A.shape[0] < 64:
        return _rows_job((name, A, B, lam))
    blocks = np.array_split(np.arange(A.shape[0]), nw)
    # forkserver: the test process has CUDA (and its threads) initialised; forking it is unsafe
    with ProcessPoolExecutor(nw, mp_context=multiprocessing.get_context("forkserver")) as ex:
        parts = list(ex.map(_rows_job, [(name, np.ascontiguousarray(A[b]), B, lam) for b in blocks if len(b)]))
    return np.concatenate(parts, axis=0)


def norm_rows_err(C: np.ndarray, R: np.ndarray) -> float:
    """||C - R||_inf over the given rows."""
    return float(np.abs(C - R).sum(axis=1).max()) if C.size else 0.0
