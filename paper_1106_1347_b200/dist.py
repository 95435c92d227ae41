"""Row-block data parallelism across GPUs (one process per GPU, torch.distributed over NCCL).

C = A B is split by rows: rank r owns rows [r*ceil(N/g), min(N, (r+1)*ceil(N/g))) of A and C
(workload.shard_rows uses the same rule); B is broadcast from `root` every product -- the one
real exchange step of the path.

The schedule of one product is NOT written here: it comes from the C library
(``mm_dist_schedule``, include/mm.h), a list of communication ops (broadcasts of row ranges of B,
the max-all-reduce of WinogradScaled's norms), compute ops and record/wait events, a function of
(method, P, M, levels, panels) only.  ``dist_gemm`` executes that list over torch.distributed
(NCCL on GPUs; gloo in the CPU tests) and ``NativeComm`` has the library execute the same list
with its own NCCL communicator (``mm_dist_gemm``).  Compute ops run through ``mm_dist_step`` --
or through an injected callable, which is how the CPU tests drive the schedule with two ranks and
the oracle as the local arithmetic.

Per-entry arithmetic of every kernel depends only on (row of A, column of B, P) -- there is no
split-K and y_i / z_k are per row / column -- so the classical, Kahan, Winograd and scaled
Winograd shards are bitwise equal to the corresponding rows of the 1-GPU product (WinogradScaled
max-all-reduces {||A_r||, ||B|| of the root}, so lambda is the 1-GPU lambda).  Strassen on a
shard recurses on (N_local x P x M) and agrees within its tolerance only.  Panels are listed in
increasing k and every running state continues from panel to panel, so any panel count gives the
one-broadcast result bit for bit.
"""
from __future__ import annotations

import ctypes
from typing import Callable, List, Optional

import torch
import torch.distributed as dist

# op kinds and streams of include/mm.h
OP_BCAST, OP_ALLREDUCE_NORMS, OP_RECORD, OP_WAIT = 1, 2, 3, 4
OP_NORMS, OP_PANEL, OP_YZ, OP_SCALE_A, OP_SCALE_B = 5, 6, 7, 8, 9
OP_FORM_A, OP_FORM_B, OP_FORM_B_REST, OP_LEAF_COMBINE, OP_FULL = 10, 11, 12, 13, 14
OP_BCAST_A, OP_S7_FORM, OP_S7_PRODUCT, OP_SEND_H, OP_RECV_H, OP_S7_COMBINE = 15, 16, 17, 18, 19, 20
STREAM_COMPUTE, STREAM_COMM = 0, 1
OP_NAMES = {OP_BCAST: "bcast", OP_ALLREDUCE_NORMS: "allreduce_norms", OP_RECORD: "record", OP_WAIT: "wait",
            OP_NORMS: "norms", OP_PANEL: "panel", OP_YZ: "yz", OP_SCALE_A: "scale_a", OP_SCALE_B: "scale_b",
            OP_FORM_A: "form_a", OP_FORM_B: "form_b", OP_FORM_B_REST: "form_b_rest",
            OP_LEAF_COMBINE: "leaf_combine", OP_FULL: "full", OP_BCAST_A: "bcast_a", OP_S7_FORM: "s7_form",
            OP_S7_PRODUCT: "s7_product", OP_SEND_H: "send_h", OP_RECV_H: "recv_h", OP_S7_COMBINE: "s7_combine"}
EX_ACCUMULATE, EX_KEEP_STATE, EX_FUSED = 1, 2, 4


class DistOp(ctypes.Structure):
    """mm_dist_op of include/mm.h."""
    _fields_ = [("op", ctypes.c_int32), ("stream", ctypes.c_int32), ("index", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("lo", ctypes.c_int64), ("hi", ctypes.c_int64)]

    def __repr__(self):
        return (f"{OP_NAMES.get(self.op, self.op)}(stream={self.stream}, index={self.index}, flags={self.flags}, "
                f"[{self.lo}, {self.hi}))")


def shard_rows(N: int, world: int, rank: int):
    per = (N + world - 1) // world
    lo = min(N, rank * per)
    return lo, min(N, lo + per)


def schedule(method: str, P: int, M: int, levels: int = 2, panels: int = 1) -> List[DistOp]:
    """The op list of one distributed product (mm_dist_schedule; host only, no GPU needed)."""
    import paper_1106_1347_b200 as mm

    L = mm.lib()
    cap = 16 + 12 * max(1, panels)
    ops = (DistOp * cap)()
    n = L.mm_dist_schedule(mm.METHODS[method], P, M, levels, panels, ops, cap)
    mm._check(n if n < 0 else 0, "mm_dist_schedule")
    return [ops[i] for i in range(n)]


def panel_bounds(P: int, panels: int):
    """The k-panels [k0, k1) the schedule uses for P (those of NaivStandard's schedule)."""
    b = [(o.lo, o.hi) for o in schedule("naive", P, 2, 0, panels) if o.op == OP_PANEL]
    return b or [(0, P)]


def workspace_bytes(method: str, N_local: int, P: int, M: int, levels: int = 2) -> int:
    import paper_1106_1347_b200 as mm

    return int(mm.lib().mm_dist_workspace_size(mm.METHODS[method], N_local, P, M, levels))


def gpu_step(op: DistOp, ctx: dict) -> None:
    """Run one compute op of the schedule through mm_dist_step on the current stream."""
    import paper_1106_1347_b200 as mm

    A, B, C, ws = ctx["A"], ctx["B"], ctx["out"], ctx["ws"]
    N, P = A.shape
    M = B.shape[1]
    with torch.cuda.device(B.device):
        rc = mm.lib().mm_dist_step(mm.METHODS[ctx["method"]], ctypes.byref(op), A.data_ptr() if N else None,
                                   B.data_ptr(), C.data_ptr() if N else None, N, P, M, ctx["levels"],
                                   int(ctx["is_root"]), ws.data_ptr() if ws is not None else None,
                                   ws.numel() if ws is not None else 0,
                                   torch.cuda.current_stream(B.device).cuda_stream)
    mm._check(rc, f"mm_dist_step({OP_NAMES.get(op.op, op.op)})")


_WS = {}


def _workspace(method, N, P, M, levels, device):
    nbytes = workspace_bytes(method, N, P, M, levels)
    if nbytes == 0:
        return None
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def dist_gemm(method: str, A_local: torch.Tensor, B: torch.Tensor, *, out: Optional[torch.Tensor] = None,
              root: int = 0, group=None, levels: int = 2, panels: int = 1,
              step: Optional[Callable] = None, ctx: Optional[dict] = None) -> torch.Tensor:
    """C_local = A_local B on every rank, executing mm_dist_schedule(method, P, M, levels, panels)
    over torch.distributed.  B must be allocated (P x M) on every rank; its content on `root` is
    broadcast (in place) during the product.  A rank with no rows still takes part in the
    collectives and returns an empty (0 x M) result.

    Communication ops are issued as async collectives in list order (a collective issued after a
    compute op is ordered after it by torch -- NCCL's stream waits for the current stream at issue);
    a compute-side WAIT waits for the works recorded on that event (NCCL: the current stream waits
    on the device; gloo: the host waits).  step(op, ctx) runs a compute op (default: mm_dist_step on
    the GPU); ctx holds method, A, B, out, levels, is_root, the norms tensor the all-reduce
    reduces, and the workspace."""
    N, P = A_local.shape
    M = B.shape[1]
    if B.shape[0] != P:
        raise ValueError("inner dimensions differ")
    rank = dist.get_rank(group)
    if out is None:
        out = torch.empty((N, M), dtype=B.dtype, device=B.device)
    ctx = dict(ctx or {})
    ctx.update(method=method, A=A_local, B=B, out=out, levels=levels, is_root=rank == root)
    if step is None:
        step = gpu_step
        ctx["ws"] = _workspace(method, N, P, M, levels, B.device)
        if method.startswith("winograd_scaled"):
            ctx["norms"] = ctx["ws"][:16].view(torch.float64)  # the workspace's leading {||A||, ||B||}
    ctx.setdefault("norms", torch.zeros(2, dtype=torch.float64, device=B.device))
    pending, events = [], {}
    for op in schedule(method, P, M, levels, panels):
        if op.op == OP_BCAST:
            pending.append(dist.broadcast(B[op.lo:op.hi], src=root, group=group, async_op=True))
        elif op.op == OP_ALLREDUCE_NORMS:
            pending.append(dist.all_reduce(ctx["norms"], op=dist.ReduceOp.MAX, group=group, async_op=True))
        elif op.op == OP_RECORD:
            if op.stream == STREAM_COMM:
                events[op.index] = pending
                pending = []
            # a compute-side record needs nothing: torch orders later collectives after it
        elif op.op == OP_WAIT:
            if op.stream == STREAM_COMPUTE:
                for w in events.pop(op.index, []):
                    w.wait()
        else:
            step(op, ctx)
    for w in pending:
        w.wait()
    for ws_ in events.values():
        for w in ws_:
            w.wait()
    return out


# ---- the alternative partition (include/mm.h mm_s7_*): Strassen's seven
# top-level products H_1..H_7 (PAPER.md:270-277 / 299-306) spread over the ranks, product p on
# rank p % world; A and B broadcast from the root, every H sent to the root, which combines (level 0).
def s7_schedule(method: str, N: int, P: int, M: int, levels: int, world: int, rank: int, root: int = 0):
    """The op list of `rank` (mm_s7_schedule; host only)."""
    import paper_1106_1347_b200 as mm

    ops = (DistOp * 64)()
    n = mm.lib().mm_s7_schedule(mm.METHODS[method], N, P, M, levels, world, rank, root, ops, 64)
    mm._check(n if n < 0 else 0, "mm_s7_schedule")
    return [ops[i] for i in range(n)]


def s7_workspace_bytes(method: str, N: int, P: int, M: int, levels: int) -> int:
    import paper_1106_1347_b200 as mm

    return int(mm.lib().mm_s7_workspace_size(mm.METHODS[method], N, P, M, levels))


def s7_h_slot(ws: torch.Tensor, p: int, N: int, P: int, M: int, levels: int) -> torch.Tensor:
    """View of H slot p (dense (Np/2) x (Mp/2) float64) of an mm_s7 workspace (layout: include/mm.h)."""
    import paper_1106_1347_b200 as mm

    _, Np, _, Mp = mm.strassen_plan(N, P, M, levels)
    h = (Np // 2) * (Mp // 2)
    return ws[p * h * 8:(p + 1) * h * 8].view(torch.float64).view(Np // 2, Mp // 2)


def s7_gpu_step(op: DistOp, ctx: dict) -> None:
    """Run one compute op of an mm_s7 schedule through mm_s7_step on the current stream."""
    import paper_1106_1347_b200 as mm

    A, B, C, ws = ctx["A"], ctx["B"], ctx.get("out"), ctx["ws"]
    N, P = A.shape
    M = B.shape[1]
    with torch.cuda.device(B.device):
        rc = mm.lib().mm_s7_step(mm.METHODS[ctx["method"]], ctypes.byref(op), A.data_ptr(), B.data_ptr(),
                                 C.data_ptr() if C is not None else None, N, P, M, ctx["levels"], ws.data_ptr(),
                                 ws.numel(), torch.cuda.current_stream(B.device).cuda_stream)
    mm._check(rc, f"mm_s7_step({OP_NAMES.get(op.op, op.op)})")


def strassen7(method: str, A: torch.Tensor, B: torch.Tensor, *, out: Optional[torch.Tensor] = None, root: int = 0,
              group=None, levels: int = 2, step: Optional[Callable] = None, ctx: Optional[dict] = None,
              slot: Optional[Callable] = None) -> Optional[torch.Tensor]:
    """C = A B with Strassen's seven top-level products on the ranks, executing mm_s7_schedule over
    torch.distributed.  A (N x P) and B (P x M) allocated on every rank; the root's content is
    broadcast into them.  Returns C on the root (bitwise the one-GPU strassen / strassen_winograd
    product with the same levels), None elsewhere.  step(op, ctx) runs a compute op (default
    mm_s7_step on the GPU); slot(ctx, p) gives the tensor H slot p lives in (default: its view of
    the workspace) -- the CPU tests inject both."""
    N, P = A.shape
    M = B.shape[1]
    if B.shape[0] != P:
        raise ValueError("inner dimensions differ")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    is_root = rank == root
    if out is None and is_root:
        out = torch.empty((N, M), dtype=B.dtype, device=B.device)
    ctx = dict(ctx or {})
    ctx.update(method=method, A=A, B=B, out=out if is_root else None, levels=levels, is_root=is_root)
    if step is None:
        step = s7_gpu_step
        nbytes = s7_workspace_bytes(method, N, P, M, levels)
        if nbytes == 0:
            raise ValueError("strassen7: method must be strassen / strassen_winograd with levels >= 1")
        ctx["ws"] = torch.empty(nbytes, dtype=torch.uint8, device=B.device)
    if slot is None:
        def slot(c, p):
            return s7_h_slot(c["ws"], p, N, P, M, levels)
    pending, events = [], {}
    for op in s7_schedule(method, N, P, M, levels, world, rank, root):
        if op.op == OP_BCAST_A:
            pending.append(dist.broadcast(A[op.lo:op.hi], src=root, group=group, async_op=True))
        elif op.op == OP_BCAST:
            pending.append(dist.broadcast(B[op.lo:op.hi], src=root, group=group, async_op=True))
        elif op.op == OP_SEND_H:
            pending.append(dist.isend(slot(ctx, op.index), dst=int(op.lo), group=group))
        elif op.op == OP_RECV_H:
            pending.append(dist.irecv(slot(ctx, op.index), src=int(op.lo), group=group))
        elif op.op == OP_RECORD:
            if op.stream == STREAM_COMM:
                events[op.index] = pending
                pending = []
        elif op.op == OP_WAIT:
            if op.stream == STREAM_COMPUTE:
                for w in events.pop(op.index, []):
                    w.wait()
        else:
            step(op, ctx)
    for w in pending:
        w.wait()
    for ws_ in events.values():
        for w in ws_:
            w.wait()
    return out if is_root else None


class NativeComm:
    """The C ABI's own multi-GPU layer (mm_dist_*: NCCL driven from libmm_b200.so, the same schedule
    on the library's streams).  torch.distributed only bootstraps it: rank 0's 128-byte NCCL id
    reaches the other ranks through broadcast_object_list."""

    def __init__(self, group=None):
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
        nbytes = int(self.L.mm_dist_workspace_size(mid, N, P, M, levels))
        if nbytes and (self._ws is None or self._ws.numel() < nbytes):
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=B.device)
        ws_ptr = self._ws.data_ptr() if nbytes else None
        s = stream if stream is not None else torch.cuda.current_stream(B.device)
        mm._check(self.L.mm_dist_gemm(mid, A_local.data_ptr() if N else None, B.data_ptr(),
                                      out.data_ptr() if N else None, N, P, M, root, levels, panels, ws_ptr, nbytes,
                                      s.cuda_stream), f"mm_dist_gemm({method})")
        return out

    def strassen7(self, method: str, A: torch.Tensor, B: torch.Tensor, *, out: Optional[torch.Tensor] = None,
                  root: int = 0, levels: int = 2, stream=None) -> Optional[torch.Tensor]:
        """The alternative partition through mm_dist_strassen7 (A, B on every rank, broadcast in place);
        C on the root."""
        mm = self.mm
        N, P = A.shape
        M = B.shape[1]
        for t in (A, B):
            if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
                raise ValueError("A and B must be contiguous float64 CUDA tensors")
        if B.shape[0] != P:
            raise ValueError("inner dimensions differ")
        if out is None and self.rank == root:
            out = torch.empty((N, M), dtype=torch.float64, device=B.device)
        mid = mm.METHODS[method]
        nbytes = int(self.L.mm_s7_workspace_size(mid, N, P, M, levels))
        if nbytes == 0:
            raise ValueError("strassen7: method must be strassen / strassen_winograd with levels >= 1")
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=B.device)
        s = stream if stream is not None else torch.cuda.current_stream(B.device)
        mm._check(self.L.mm_dist_strassen7(mid, A.data_ptr(), B.data_ptr(), out.data_ptr() if out is not None else None,
                                           N, P, M, root, levels, self._ws.data_ptr(), nbytes, s.cuda_stream),
                  f"mm_dist_strassen7({method})")
        return out if self.rank == root else None

    def close(self):
        if self.L is not None:
            self.mm._check(self.L.mm_dist_finalize(), "mm_dist_finalize")
            self.L = None
