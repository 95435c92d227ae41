"""Row-block data parallelism across GPUs (one process per GPU, torch.distributed over NCCL).

C = A B is split by rows: rank r owns rows [r*ceil(N/g), min(N, (r+1)*ceil(N/g))) of A and C
(workload.shard_rows uses the same rule); B is broadcast from `root` every product -- the one
real exchange step of the path.  WinogradScaled additionally needs
the GLOBAL ||A||_inf: each rank's local norm is max-all-reduced (8 bytes), ||B||_inf is local
because B is replicated, so lambda is identical on every rank and to the 1-GPU run.

Per-entry arithmetic of every kernel depends only on (row of A, column of B, P) -- there is
no split-K and y_i / z_k are per row / column -- so the classical, Kahan, Winograd and scaled
Winograd shards are bitwise equal to the corresponding rows of the 1-GPU product.  Strassen on
a shard recurses on (N_local x P x M) and agrees within its tolerance only.

Broadcast/compute overlap, NaivStandard, NaivKahan and WinogradOriginal
(and their fused variants): with panels > 1, B is broadcast as `panels` consecutive row panels
(contiguous in memory, even boundaries), all enqueued at once on NCCL's stream; the product is
accumulated panel by panel (mm_naive_ex / mm_kahan_ex / mm_winograd_ex), each launch waiting (on
the device, not the host) for its own panel only, so the transfer of panel i+1 overlaps the work on
panel i.  Every entry's running state -- the fma chain (reading R2), Kahan's (sum, err), Winograd's
pair sum -- continues from panel to panel in k order, so the result is bitwise the one-shot product
at any panel count; Winograd's y and z are computed from the full operands before the last panel.

The compute and norm callables are injectable so that the host-side logic (sharding, the
broadcast, the max-reduction and lambda, the panel schedule) is testable with world_size 2 on
CPU (gloo).
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_rows(N: int, world: int, rank: int):
    per = (N + world - 1) // world
    lo = min(N, rank * per)
    return lo, min(N, lo + per)


def _default_compute(method: str, A, B, out, levels, norms):
    import paper_1106_1347_b200 as mm

    if method == "winograd_scaled":
        return mm.winograd_scaled(A, B, out=out, norms=norms)
    if method in ("strassen", "strassen_winograd"):
        return getattr(mm, method)(A, B, out=out, levels=levels)
    return getattr(mm, method)(A, B, out=out)


def _default_norm(X):
    import paper_1106_1347_b200 as mm

    return mm.norm_inf(X)


PANEL_METHODS = ("naive", "kahan", "kahan_fused", "winograd", "winograd_fused")


def _default_panel(method, A_panel, B_panel, out, first: bool, last: bool, ctx: dict):
    """One k-panel step on the GPU.  ctx holds the full operands ("A", "B") and the carried state
    (Kahan's err "E"; Winograd's "y", "z", computed from the full operands before the last panel)."""
    import paper_1106_1347_b200 as mm

    fused = method.endswith("_fused")
    if method == "naive":
        return mm.naive_panel(A_panel, B_panel, out, accumulate=not first)
    if method.startswith("kahan"):
        if "E" not in ctx:
            ctx["E"] = torch.empty_like(out)
        return mm.kahan_panel(A_panel, B_panel, out, ctx["E"], accumulate=not first, keep_state=not last,
                              fused=fused)
    y = z = None
    if last:
        A, B = ctx["A"], ctx["B"]
        y = torch.empty(A.shape[0], dtype=torch.float64, device=A.device)
        z = torch.empty(B.shape[1], dtype=torch.float64, device=B.device)
        mm.winograd_yz(A, B, y, z, fused=fused)
    return mm.winograd_panel(A_panel, B_panel, out, y, z, accumulate=not first, keep_state=not last, fused=fused)


def panels_supported(method: str, P: int, M: int) -> bool:
    """NaivStandard always; Kahan / Winograd need the TMA-fed panel kernels: P and M even."""
    return method == "naive" or (method in PANEL_METHODS and P % 2 == 0 and M % 2 == 0)


def panel_bounds(P: int, panels: int):
    """Consecutive k-panels [k0, k1) covering 0..P, boundaries even (16-byte aligned views)."""
    panels = max(1, min(panels, P))
    cuts = sorted({min(P, 2 * ((P * i) // (2 * panels))) for i in range(1, panels)} - {0, P})
    b = [0] + cuts + [P]
    return list(zip(b[:-1], b[1:]))


def _dist_panels(method, A_local, B, out, root, group, panels, panel_compute):
    P, M = B.shape
    bounds = panel_bounds(P, panels)
    works = [dist.broadcast(B[k0:k1], src=root, group=group, async_op=True) for k0, k1 in bounds]
    if out is None:
        out = torch.empty((A_local.shape[0], M), dtype=B.dtype, device=B.device)
    ctx = {"A": A_local, "B": B}
    for i, (k0, k1) in enumerate(bounds):
        works[i].wait()  # NCCL: the current stream waits for this panel only; gloo: the host waits
        if A_local.shape[0] > 0:
            panel_compute(method, A_local[:, k0:k1], B[k0:k1], out, i == 0, i == len(bounds) - 1, ctx)
    return out


def dist_gemm(method: str, A_local: torch.Tensor, B: torch.Tensor, *, out: Optional[torch.Tensor] = None,
              root: int = 0, group=None, levels: int = 2, compute: Optional[Callable] = None,
              norm: Optional[Callable] = None, panels: int = 1,
              panel_compute: Optional[Callable] = None) -> torch.Tensor:
    """C_local = A_local B on every rank.  B must be allocated (P x M) on every rank; its content
    on `root` is broadcast (in place) before / during the product.  A rank with no rows still
    takes part in the collectives and returns an empty (0 x M) result.  panels > 1 (NaivStandard;
    NaivKahan / WinogradOriginal and the fused variants when P and M are even): panelised broadcast
    overlapped with the accumulation (NEXT-4); panel_compute(method, A_panel, B_panel, out, first,
    last, ctx) performs one panel step."""
    compute = compute or _default_compute
    norm = norm or _default_norm
    if panels > 1 and panels_supported(method, B.shape[0], B.shape[1]):
        return _dist_panels(method, A_local, B, out, root, group, panels, panel_compute or _default_panel)
    dist.broadcast(B, src=root, group=group)
    norms = None
    if method == "winograd_scaled":
        nA = norm(A_local) if A_local.shape[0] > 0 else torch.zeros(1, dtype=torch.float64, device=B.device)
        dist.all_reduce(nA, op=dist.ReduceOp.MAX, group=group)  # ||A||_inf = max over row blocks
        norms = torch.cat([nA.reshape(1), norm(B).reshape(1)])
    if A_local.shape[0] == 0:
        return torch.empty((0, B.shape[1]), dtype=B.dtype, device=B.device)
    return compute(method, A_local, B, out, levels, norms)


class NativeComm:
    """The C ABI's own multi-GPU layer (mm_dist_*: NCCL driven from libmm_b200.so, broadcast of B
    and the panelised overlap on the library's streams).  torch.distributed only bootstraps it:
    rank 0's 128-byte NCCL id reaches the other ranks through broadcast_object_list."""

    def __init__(self, group=None):
        import ctypes
        import os

        import paper_1106_1347_b200 as mm

        if "MM_NCCL_LIBRARY" not in os.environ:
            try:  # the NCCL PyTorch ships (used when the soname is not already resident)
                import nvidia.nccl

                os.environ["MM_NCCL_LIBRARY"] = os.path.join(nvidia.nccl.__path__[0], "lib", "libnccl.so.2")
            except ImportError:
                pass
        self.mm = mm
        self.L = mm.lib()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        buf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            mm._check(self.L.mm_dist_get_unique_id(buf), "mm_dist_get_unique_id")
        obj = [buf.raw]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.device = torch.cuda.current_device()
        mm._check(self.L.mm_dist_init(self.rank, self.world, obj[0], self.device), "mm_dist_init")
        self._ws = None

    def gemm(self, method: str, A_local: torch.Tensor, B: torch.Tensor, *, out: Optional[torch.Tensor] = None,
             root: int = 0, levels: int = 2, panels: int = 1, stream=None) -> torch.Tensor:
        """C_local = A_local B through mm_dist_gemm (B: P x M on every rank, broadcast in place)."""
        mm = self.mm
        N, P = A_local.shape
        M = B.shape[1]
        for t in (A_local, B):
            if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
                raise ValueError("A_local and B must be contiguous float64 CUDA tensors")
        if B.shape[0] != P:
            raise ValueError("inner dimensions differ")
        if out is None:
            out = torch.empty((N, M), dtype=torch.float64, device=B.device)
        mid = mm.METHODS[method]
        lv = levels if method in ("strassen", "strassen_winograd") else 0
        nbytes = int(self.L.mm_dist_workspace_size(mid, N, P, M, lv))
        if nbytes and (self._ws is None or self._ws.numel() < nbytes):
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=B.device)
        ws_ptr = self._ws.data_ptr() if nbytes else None
        s = stream if stream is not None else torch.cuda.current_stream(B.device)
        mm._check(self.L.mm_dist_gemm(mid, A_local.data_ptr() if N else None, B.data_ptr(),
                                      out.data_ptr() if N else None, N, P, M, root, lv, panels, ws_ptr, nbytes,
                                      s.cuda_stream), f"mm_dist_gemm({method})")
        return out

    def close(self):
        if self.L is not None:
            self.mm._check(self.L.mm_dist_finalize(), "mm_dist_finalize")
            self.L = None
