"""B200-native FP64 matrix multiplication in the families of Hedtke, "Methods of Matrix
Multiplication" (arXiv 1106.1347).

Thin ctypes binding over the C ABI of ``libmm_b200.so`` (declared in ``include/mm.h``).
This module only marshals arguments: every arithmetic step runs in the sm_100a kernels of
the library.  PyTorch supplies device memory, streams and (in ``dist``) process groups.

There is no CPU fallback: if the library is missing, or the device is not a B200
(sm_100), every call raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

from . import build as _build

__all__ = [
    "MMError", "lib", "naive", "naive_on_array", "unroll2", "unroll3", "unroll4", "kahan", "winograd",
    "winograd_scaled", "strassen", "strassen_winograd", "norm_inf", "matmul", "strassen_plan",
    "workspace_size", "lambda_rule", "METHODS", "kahan_fused", "winograd_fused", "winograd_scaled_fused",
    "naive_panel", "matmul_methods", "GraphedProduct",
]

MM_NAIVE, MM_KAHAN, MM_WINOGRAD, MM_WINOGRAD_SCALED, MM_STRASSEN, MM_STRASSEN_WINOGRAD = range(6)
MM_KAHAN_FUSED, MM_WINOGRAD_FUSED, MM_WINOGRAD_SCALED_FUSED = 6, 7, 8  # NEXT-3 (R22)
METHODS = {
    "naive": MM_NAIVE,
    "kahan": MM_KAHAN,
    "winograd": MM_WINOGRAD,
    "winograd_scaled": MM_WINOGRAD_SCALED,
    "strassen": MM_STRASSEN,
    "strassen_winograd": MM_STRASSEN_WINOGRAD,
    "kahan_fused": MM_KAHAN_FUSED,
    "winograd_fused": MM_WINOGRAD_FUSED,
    "winograd_scaled_fused": MM_WINOGRAD_SCALED_FUSED,
}

# every symbol include/mm.h declares
EXPORTS = ("mm_version", "mm_status_string", "mm_naive", "mm_kahan", "mm_winograd", "mm_winograd_scaled",
           "mm_strassen", "mm_strassen_winograd", "mm_strassen_plan", "mm_workspace_size", "mm_gemm", "norm_inf",
           "mm_lambda", "mm_winograd_scaled_norms", "mm_launch_count", "mm_kahan_fused", "mm_winograd_fused",
           "mm_winograd_scaled_fused", "mm_naive_ex", "mm_dist_get_unique_id", "mm_dist_init",
           "mm_dist_workspace_size", "mm_dist_gemm", "mm_dist_finalize", "mm_kahan_ex", "mm_winograd_ex",
           "mm_winograd_yz", "mm_dist_schedule", "mm_dist_step", "mm_methods_host", "mm_methods_host_workspace_size",
           "mm_s7_schedule", "mm_s7_workspace_size", "mm_s7_step", "mm_dist_strassen7")
MM_EX_ACCUMULATE, MM_EX_KEEP_STATE, MM_EX_FUSED = 1, 2, 4


class MMError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    """Load libmm_b200.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        path = _build.LIB_PATH
        if not os.path.exists(path):
            raise MMError(f"{path} is missing: run __graft_entry__.build() (python -m paper_1106_1347_b200.build)")
        L = ctypes.CDLL(path)
        vp, i64, i32, sz, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t, ctypes.c_void_p
        L.mm_version.restype = ctypes.c_char_p
        L.mm_status_string.restype = ctypes.c_char_p
        L.mm_status_string.argtypes = [ctypes.c_int]
        for n in ("mm_naive", "mm_kahan", "mm_kahan_fused"):
            getattr(L, n).argtypes = [dp, dp, dp, i64, i64, i64, vp]
        L.mm_naive_ex.argtypes = [dp, i64, dp, i64, dp, i64, i64, i64, i64, i32, vp]
        L.mm_kahan_ex.argtypes = [dp, i64, dp, i64, dp, dp, i64, i64, i64, i32, vp]
        L.mm_winograd_ex.argtypes = [dp, i64, dp, i64, dp, dp, dp, i64, i64, i64, i32, vp]
        L.mm_winograd_yz.argtypes = [dp, dp, i64, i64, i64, dp, dp, i32, vp]
        L.mm_dist_get_unique_id.argtypes = [ctypes.c_char_p]
        L.mm_dist_init.argtypes = [i32, i32, ctypes.c_char_p, i32]
        L.mm_dist_workspace_size.argtypes = [ctypes.c_int, i64, i64, i64, i32]
        L.mm_dist_workspace_size.restype = sz
        L.mm_dist_gemm.argtypes = [ctypes.c_int, dp, dp, dp, i64, i64, i64, i32, i32, i32, vp, sz, vp]
        L.mm_dist_schedule.argtypes = [ctypes.c_int, i64, i64, i32, i32, vp, i32]
        L.mm_methods_host_workspace_size.argtypes = [vp, i32, i64, i64, i64, i32]
        L.mm_methods_host_workspace_size.restype = sz
        L.mm_methods_host.argtypes = [vp, i32, dp, dp, vp, i64, i64, i64, i32, i32, vp, sz, vp]
        L.mm_dist_step.argtypes = [ctypes.c_int, vp, dp, dp, dp, i64, i64, i64, i32, i32, vp, sz, vp]
        L.mm_s7_schedule.argtypes = [ctypes.c_int, i64, i64, i64, i32, i32, i32, i32, vp, i32]
        L.mm_s7_workspace_size.argtypes = [ctypes.c_int, i64, i64, i64, i32]
        L.mm_s7_workspace_size.restype = sz
        L.mm_s7_step.argtypes = [ctypes.c_int, vp, dp, dp, dp, i64, i64, i64, i32, vp, sz, vp]
        L.mm_dist_strassen7.argtypes = [ctypes.c_int, dp, dp, dp, i64, i64, i64, i32, i32, vp, sz, vp]
        for n in ("mm_winograd", "mm_winograd_fused"):
            getattr(L, n).argtypes = [dp, dp, dp, i64, i64, i64, vp, sz, vp]
        for n in ("mm_winograd_scaled", "mm_winograd_scaled_fused"):
            getattr(L, n).argtypes = [dp, dp, dp, i64, i64, i64, vp, sz, ctypes.POINTER(i32), vp]
        for n in ("mm_strassen", "mm_strassen_winograd"):
            getattr(L, n).argtypes = [dp, dp, dp, i64, i64, i64, i32, vp, sz, vp]
        L.mm_strassen_plan.argtypes = [i64, i64, i64, i32, ctypes.POINTER(i32), ctypes.POINTER(i64),
                                       ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.mm_workspace_size.argtypes = [ctypes.c_int, i64, i64, i64, i32]
        L.mm_workspace_size.restype = sz
        L.mm_gemm.argtypes = [ctypes.c_int, dp, dp, dp, i64, i64, i64, i32, vp, sz, ctypes.POINTER(i32), vp]
        L.norm_inf.argtypes = [dp, i64, i64, dp, vp]
        L.mm_lambda.argtypes = [ctypes.c_double, ctypes.c_double]
        L.mm_lambda.restype = i32
        L.mm_winograd_scaled_norms.argtypes = [dp, dp, dp, i64, i64, i64, dp, vp, sz, ctypes.POINTER(i32), vp]
        L.mm_launch_count.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise MMError(f"{what}: {lib().mm_status_string(rc).decode()} (status {rc})")


def _stream_handle(stream: Optional[torch.cuda.Stream], device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _operands(A: torch.Tensor, B: torch.Tensor, out: Optional[torch.Tensor]):
    if not (isinstance(A, torch.Tensor) and isinstance(B, torch.Tensor)):
        raise TypeError("A and B must be torch tensors")
    if A.dtype != torch.float64 or B.dtype != torch.float64:
        raise ValueError("A and B must be float64 (the paper's entries are of type double)")
    if A.dim() != 2 or B.dim() != 2:
        raise ValueError("A and B must be matrices")
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"inner dimensions differ: {tuple(A.shape)} x {tuple(B.shape)}")
    if not (A.is_cuda and B.is_cuda) or A.device != B.device:
        raise ValueError("A and B must be CUDA tensors on one device (use matmul() for host tensors)")
    if not (A.is_contiguous() and B.is_contiguous()):
        raise ValueError("A and B must be contiguous row-major")
    N, P = A.shape
    M = B.shape[1]
    if out is None:
        out = torch.empty((N, M), dtype=torch.float64, device=A.device)
    elif out.shape != (N, M) or out.dtype != torch.float64 or out.device != A.device or not out.is_contiguous():
        raise ValueError("out must be a contiguous float64 N x M tensor on A's device")
    return N, P, M, out


# ---- workspace: grown on demand, then reused (no allocation on later calls) ----------
_ws = {}


def _workspace(nbytes: int, device, stream=None) -> Tuple[int, int]:
    """A scratch buffer of >= nbytes for calls enqueued on `stream` (default: the current stream).
    One buffer per (device, stream): calls on different streams may run concurrently and must not
    share scratch space; the buffer is allocated on that stream, so when it is replaced by a
    larger one the caching allocator only recycles its memory in that stream's order."""
    if nbytes == 0:
        return 0, 0
    dev = torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev.index, s.cuda_stream)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        # drop the smaller buffer first: at c5 sizes the old and the new one need not fit together
        _ws.pop(key, None)
        del buf
        with torch.cuda.stream(s):
            buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        _ws[key] = buf
    return buf.data_ptr(), buf.numel()


def release_workspace():
    _ws.clear()


def workspace_size(method: str, N: int, P: int, M: int, levels: int = 0) -> int:
    return int(lib().mm_workspace_size(METHODS[method], N, P, M, levels))


def strassen_plan(N: int, P: int, M: int, levels: int):
    """(depth, Np, Pp, Mp) the library uses for this problem (levels=-1: the paper's plan)."""
    d = ctypes.c_int32()
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().mm_strassen_plan(N, P, M, levels, ctypes.byref(d), ctypes.byref(a), ctypes.byref(b),
                                  ctypes.byref(c)), "mm_strassen_plan")
    return int(d.value), int(a.value), int(b.value), int(c.value)


def lambda_rule(nA: float, nB: float) -> int:
    return int(lib().mm_lambda(float(nA), float(nB)))


def _gemm(method: int, name: str, A, B, out=None, levels: int = 0, stream=None, want_lambda=False):
    N, P, M, out = _operands(A, B, out)
    L = lib()
    ws_bytes = int(L.mm_workspace_size(method, N, P, M, levels))
    if method in (MM_STRASSEN, MM_STRASSEN_WINOGRAD) and ws_bytes == 0:
        d = strassen_plan(N, P, M, levels)[0]
        if d != 0:
            raise MMError("bad Strassen plan")
    ws_ptr, ws_len = _workspace(ws_bytes, A.device, stream)
    lam = ctypes.c_int32(0)
    st = _stream_handle(stream, A.device)
    with torch.cuda.device(A.device):  # the library launches on the current device
        rc = L.mm_gemm(method, A.data_ptr(), B.data_ptr(), out.data_ptr(), N, P, M, levels, ws_ptr, ws_len,
                       ctypes.byref(lam) if want_lambda else None, st)
    _check(rc, name)
    if want_lambda:
        return out, int(lam.value)
    return out


def naive(A, B, *, out=None, stream=None):
    """NaivStandard on the FP64 tensor cores."""
    return _gemm(MM_NAIVE, "mm_naive", A, B, out, stream=stream)


def naive_panel(A, B, C, *, accumulate: bool, stream=None):
    """C = A B (+ C) on strided 2-D views (mm_naive_ex): with accumulate=True each entry's fma
    chain continues from C, so consecutive k-panels reproduce naive() bit for bit.  A, B, C must
    be float64 CUDA tensors with unit column stride (row-major views, e.g. A[:, k0:k1])."""
    for t in (A, B, C):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.dim() == 2
                and t.stride(1) == 1):
            raise ValueError("A, B, C must be row-major float64 CUDA matrices (unit column stride)")
    N, K = A.shape
    if B.shape[0] != K or C.shape != (N, B.shape[1]):
        raise ValueError(f"shape mismatch: {tuple(A.shape)} x {tuple(B.shape)} -> {tuple(C.shape)}")
    M = B.shape[1]
    if not (A.device == B.device == C.device):
        raise ValueError("A, B, C must be on one device")
    with torch.cuda.device(A.device):
        rc = lib().mm_naive_ex(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(), C.stride(0), N,
                               K, M, 1 if accumulate else 0, _stream_handle(stream, A.device))
    _check(rc, "mm_naive_ex")
    return C


def _panel_views(A, B, C, E=None):
    for t in (A, B, C) + ((E,) if E is not None else ()):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.dim() == 2
                and t.stride(1) == 1):
            raise ValueError("operands must be row-major float64 CUDA matrices (unit column stride)")
    N, K = A.shape
    M = B.shape[1]
    if B.shape[0] != K or C.shape != (N, M) or not C.is_contiguous():
        raise ValueError(f"shape mismatch or non-dense C: {tuple(A.shape)} x {tuple(B.shape)} -> {tuple(C.shape)}")
    if E is not None and (E.shape != (N, M) or not E.is_contiguous()):
        raise ValueError("E must be a dense N x M float64 tensor")
    if not (A.device == B.device == C.device):
        raise ValueError("operands must be on one device")
    return N, K, M


def _ex_flags(accumulate, keep_state, fused):
    return (MM_EX_ACCUMULATE if accumulate else 0) | (MM_EX_KEEP_STATE if keep_state else 0) | (
        MM_EX_FUSED if fused else 0)


def kahan_panel(A, B, C, E, *, accumulate: bool, keep_state: bool, fused: bool = False, stream=None):
    """One k-panel of NaivKahan (mm_kahan_ex): A / B are panel views (A[:, k0:k1], B[k0:k1]), C and E
    dense N x M holding each entry's (sum, err); consecutive panels, the first without
    `accumulate` and all but the last with `keep_state`, reproduce kahan() bit for bit."""
    N, K, M = _panel_views(A, B, C, E)
    with torch.cuda.device(A.device):
        rc = lib().mm_kahan_ex(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(),
                               E.data_ptr() if E is not None else None, N, K, M,
                               _ex_flags(accumulate, keep_state, fused), _stream_handle(stream, A.device))
    _check(rc, "mm_kahan_ex")
    return C


def winograd_yz(A, B, y, z, *, fused: bool = False, stream=None):
    """y_i, z_k of WinogradOriginal for dense A, B into device vectors y (N), z (M)."""
    N, P = A.shape
    M = B.shape[1]
    for t, n in ((y, N), (z, M)):
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and t.numel() == n):
            raise ValueError("y, z must be contiguous float64 CUDA vectors of N and M entries")
    with torch.cuda.device(A.device):
        rc = lib().mm_winograd_yz(A.data_ptr(), B.data_ptr(), N, P, M, y.data_ptr(), z.data_ptr(),
                                  MM_EX_FUSED if fused else 0, _stream_handle(stream, A.device))
    _check(rc, "mm_winograd_yz")


def winograd_panel(A, B, C, y=None, z=None, *, accumulate: bool, keep_state: bool, fused: bool = False,
                   stream=None):
    """One k-panel (even width) of WinogradOriginal's pair sums (mm_winograd_ex); the last panel
    (keep_state=False) applies C = (acc - y_i) - z_k with y, z of the full operands."""
    N, K, M = _panel_views(A, B, C)
    with torch.cuda.device(A.device):
        rc = lib().mm_winograd_ex(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(),
                                  y.data_ptr() if y is not None else None, z.data_ptr() if z is not None else None,
                                  N, K, M, _ex_flags(accumulate, keep_state, fused), _stream_handle(stream, A.device))
    _check(rc, "mm_winograd_ex")
    return C


# NaivOnArray and the unrolled variants compute the same product; on the GPU they are the
# same DMMA kernel (their C loop shapes are prior art).
naive_on_array = naive
unroll2 = naive
unroll3 = naive
unroll4 = naive


def kahan(A, B, *, out=None, stream=None):
    """NaivKahan."""
    return _gemm(MM_KAHAN, "mm_kahan", A, B, out, stream=stream)


def winograd(A, B, *, out=None, stream=None):
    """WinogradOriginal."""
    return _gemm(MM_WINOGRAD, "mm_winograd", A, B, out, stream=stream)


def winograd_scaled(A, B, *, out=None, stream=None, return_lambda: bool = False,
                    norms: Optional[torch.Tensor] = None):
    """WinogradScaled.  return_lambda=True synchronises and returns (C, lambda).
    norms: optional 2-element float64 device tensor {||A||_inf, ||B||_inf} (e.g. the global
    norm of a row-sharded A); default: computed on the device from A and B."""
    if norms is None:
        return _gemm(MM_WINOGRAD_SCALED, "mm_winograd_scaled", A, B, out, stream=stream,
                     want_lambda=return_lambda)
    N, P, M, out = _operands(A, B, out)
    if norms.dtype != torch.float64 or norms.numel() != 2 or norms.device != A.device or not norms.is_contiguous():
        raise ValueError("norms must be a contiguous 2-element float64 tensor on A's device")
    L = lib()
    ws_ptr, ws_len = _workspace(int(L.mm_workspace_size(MM_WINOGRAD_SCALED, N, P, M, 0)), A.device, stream)
    lam = ctypes.c_int32(0)
    with torch.cuda.device(A.device):
        rc = L.mm_winograd_scaled_norms(A.data_ptr(), B.data_ptr(), out.data_ptr(), N, P, M, norms.data_ptr(), ws_ptr,
                                        ws_len, ctypes.byref(lam) if return_lambda else None,
                                        _stream_handle(stream, A.device))
    _check(rc, "mm_winograd_scaled_norms")
    return (out, int(lam.value)) if return_lambda else out


# ---- fused-multiply-add variants (reading R22).  NOT the paper's
# methods (its C99 rounds every product separately): every "s + x*y" becomes one fma(x, y, s).
def kahan_fused(A, B, *, out=None, stream=None):
    """NaivKahan with err = fma(A_ik, B_kj, err)."""
    return _gemm(MM_KAHAN_FUSED, "mm_kahan_fused", A, B, out, stream=stream)


def winograd_fused(A, B, *, out=None, stream=None):
    """WinogradOriginal with y, z, the pair sums and the odd-P term via fma."""
    return _gemm(MM_WINOGRAD_FUSED, "mm_winograd_fused", A, B, out, stream=stream)


def winograd_scaled_fused(A, B, *, out=None, stream=None, return_lambda: bool = False):
    """WinogradScaled on top of winograd_fused."""
    return _gemm(MM_WINOGRAD_SCALED_FUSED, "mm_winograd_scaled_fused", A, B, out, stream=stream,
                 want_lambda=return_lambda)


def launch_count() -> int:
    """Kernels launched by the library so far in this process."""
    return int(lib().mm_launch_count())


def strassen(A, B, *, levels: int = 2, out=None, stream=None):
    """StrassenNaiv; levels=-1 uses the paper's padding plan."""
    return _gemm(MM_STRASSEN, "mm_strassen", A, B, out, levels=levels, stream=stream)


def strassen_winograd(A, B, *, levels: int = 2, out=None, stream=None):
    """StrassenWinograd."""
    return _gemm(MM_STRASSEN_WINOGRAD, "mm_strassen_winograd", A, B, out, levels=levels, stream=stream)


def norm_inf(X: torch.Tensor, *, out=None, stream=None) -> torch.Tensor:
    """||X||_inf as a 1-element float64 device tensor."""
    if X.dtype != torch.float64 or X.dim() != 2 or not X.is_cuda or not X.is_contiguous():
        raise ValueError("X must be a contiguous float64 CUDA matrix")
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=X.device)
    with torch.cuda.device(X.device):
        rc = lib().norm_inf(X.data_ptr(), X.shape[0], X.shape[1], out.data_ptr(), _stream_handle(stream, X.device))
    _check(rc, "norm_inf")
    return out


_FUNCS = {
    "naive": naive, "kahan": kahan, "winograd": winograd, "winograd_scaled": winograd_scaled,
    "strassen": strassen, "strassen_winograd": strassen_winograd, "kahan_fused": kahan_fused,
    "winograd_fused": winograd_fused, "winograd_scaled_fused": winograd_scaled_fused,
}


# methods whose entries depend only on (row of A, column of B): a row block of C is computed
# bit-identically from the matching row block of A, so host copies can be pipelined by rows
_ROW_LOCAL = ("naive", "kahan", "winograd", "kahan_fused", "winograd_fused")
def matmul(A: torch.Tensor, B: torch.Tensor, method: str = "naive", *, levels: int = 2, device=None,
           stream=None, out: Optional[torch.Tensor] = None, row_blocks: int = 4) -> torch.Tensor:
    """The user-level call.  Device tensors run in place on their device; host tensors go through
    the C ABI's host-buffer entry point (mm_methods_host with one method): copied to `device`
    (default cuda:current), multiplied, the product copied back into `out` (or a new host tensor),
    with A's row blocks / k-panels pipelined against the kernels for page-locked tensors.  Bitwise
    the device call's result."""
    f = _FUNCS[method]
    kw = {"levels": levels} if method in ("strassen", "strassen_winograd") else {}
    if A.is_cuda and B.is_cuda:
        return f(A, B, out=out, stream=stream, **kw)
    if out is None:
        out = torch.empty((A.shape[0], B.shape[1]), dtype=torch.float64, pin_memory=A.is_pinned())
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if stream is not None:
        with torch.cuda.stream(stream):
            matmul_methods(A.contiguous(), B.contiguous(), [method], levels=levels, device=dev, outs={method: out},
                           row_blocks=row_blocks)
    else:
        matmul_methods(A.contiguous(), B.contiguous(), [method], levels=levels, device=dev, outs={method: out},
                       row_blocks=row_blocks)
    return out


def matmul_methods(A: torch.Tensor, B: torch.Tensor, methods, *, levels: int = 2, device=None,
                   outs: Optional[dict] = None, row_blocks: int = 4) -> dict:
    """The shape of the paper's test program: several methods applied to the
    SAME host operands, through the C ABI's host-buffer entry point ``mm_methods_host``: A and B
    (host float64; page-locked for the copies to overlap) are copied to the device once, every
    method's product comes back into outs[method] (page-locked host tensors, allocated if missing;
    several methods may share one) while the next method computes.  A first NaivStandard
    multiplies k-panels as they land, a first row-local method row blocks as they land, a last
    row-local method returns by row blocks of halving height.  Each product is bitwise the device
    call's.  Synchronous."""
    methods = list(methods)
    for X in (A, B):
        if X.is_cuda or X.dtype != torch.float64 or X.dim() != 2 or not X.is_contiguous():
            raise ValueError("A and B must be contiguous float64 host matrices")
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"inner dimensions differ: {tuple(A.shape)} x {tuple(B.shape)}")
    N, P = A.shape
    M = B.shape[1]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    outs = {} if outs is None else outs
    for m in methods:
        if m not in outs:
            outs[m] = torch.empty((N, M), dtype=torch.float64, pin_memory=True)
        o = outs[m]
        if o.is_cuda or o.dtype != torch.float64 or tuple(o.shape) != (N, M) or not o.is_contiguous():
            raise ValueError(f"outs[{m!r}] must be a contiguous float64 host tensor of shape {(N, M)}")
    ids = (ctypes.c_int * len(methods))(*[METHODS[m] for m in methods])
    L = lib()
    nbytes = int(L.mm_methods_host_workspace_size(ids, len(methods), N, P, M, levels))
    if nbytes == 0:
        raise MMError("mm_methods_host_workspace_size: bad arguments")
    s = torch.cuda.current_stream(dev)
    ws_ptr, ws_len = _workspace(nbytes, dev, s)
    cs = (ctypes.c_void_p * len(methods))(*[outs[m].data_ptr() for m in methods])
    with torch.cuda.device(dev):
        rc = L.mm_methods_host(ids, len(methods), A.data_ptr(), B.data_ptr(), cs, N, P, M, levels, row_blocks, ws_ptr,
                               ws_len, s.cuda_stream)
    _check(rc, "mm_methods_host")
    return outs


class GraphedProduct:
    """One product C = A B by `method`, captured once into a CUDA graph and replayed.

    For small problems a call is host/launch bound (argument checks, ctypes, up to 4d+1 launches
    for Strassen, 3 for WinogradScaled); replaying the captured launch sequence removes that
    overhead.  The graph reads A and B and writes `out` at the addresses captured, so refreshing
    the inputs in place (A.copy_(...)) and calling replay() computes the new product; the object
    owns its own workspace, so later calls of other products cannot free memory the graph uses.
    Every replay runs exactly the kernels of the direct call (bitwise the same result)."""

    def __init__(self, method: str, A: torch.Tensor, B: torch.Tensor, *, out: Optional[torch.Tensor] = None,
                 levels: int = 2):
        N, P, M, out = _operands(A, B, out)
        self.method, self.A, self.B, self.out = method, A, B, out
        mid = METHODS[method]
        L = lib()
        lv = levels if method in ("strassen", "strassen_winograd") else 0
        nbytes = int(L.mm_workspace_size(mid, N, P, M, lv))
        if method in ("strassen", "strassen_winograd") and nbytes == 0 and strassen_plan(N, P, M, lv)[0] != 0:
            raise MMError("bad Strassen plan")
        self.ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=A.device)
        ws_ptr, ws_len = (self.ws.data_ptr(), nbytes) if nbytes else (0, 0)

        def call(stream):
            _check(L.mm_gemm(mid, A.data_ptr(), B.data_ptr(), out.data_ptr(), N, P, M, lv, ws_ptr, ws_len, None,
                             stream.cuda_stream), f"mm_gemm({method})")

        with torch.cuda.device(A.device):  # the library launches on the current device
            side = torch.cuda.Stream(A.device)
            side.wait_stream(torch.cuda.current_stream(A.device))
            with torch.cuda.stream(side):
                call(side)  # warm-up outside capture: kernel attributes, occupancy queries, tensor maps
            torch.cuda.current_stream(A.device).wait_stream(side)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                call(torch.cuda.current_stream(A.device))

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.out

    __call__ = replay
