"""Every compute op of the multi-GPU schedule (mm_dist_step) on one GPU, at the shard shapes of a
g-rank run: for each rank's rows the schedule's compute ops run in order with B already complete
(the communication ops are what test_dist_cpu.py drives with two ranks), the all-reduce of the
norms replaced by the max over the ranks' NORMS results.  Each shard must be bitwise the rows of
the one-GPU product (Strassen: bitwise the one-GPU call on the same shard), for every panel count
-- this is where the panel kernels, the panelised scaling of WinogradScaled and the Strassen
formation restricted to arriving B rows are checked against the one-shot kernels."""
import numpy as np
import pytest
import torch

import workload

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_1106_1347_b200")
from paper_1106_1347_b200 import dist as d  # noqa: E402

DEV = torch.device("cuda", 0)
METHODS = ("naive", "kahan", "kahan_fused", "winograd", "winograd_fused", "winograd_scaled", "winograd_scaled_fused",
           "strassen", "strassen_winograd")


def _run_ranks(m, A, B, world, panels, levels):
    """Run the schedule's compute ops rank by rank; returns the stacked shards and the op kinds run."""
    N, P = A.shape
    M = B.shape[1]
    ops = d.schedule(m, P, M, levels, panels)
    ctxs = []
    for r in range(world):
        lo, hi = d.shard_rows(N, world, r)
        ws_bytes = d.workspace_bytes(m, hi - lo, P, M, levels)
        ws = torch.full((max(ws_bytes, 1),), 0xFF, dtype=torch.uint8, device=DEV)  # NaN-filled scratch
        ctxs.append(dict(method=m, A=A[lo:hi], B=B, out=torch.full((hi - lo, M), np.nan, dtype=torch.float64,
                                                                    device=DEV),
                         levels=levels, is_root=r == 0, ws=ws if ws_bytes else None))
    kinds = set()
    # phase 1: the NORMS of every rank, then the "all-reduce" (max over ranks) into every workspace
    for op in ops:
        if op.op == d.OP_NORMS:
            for c in ctxs:
                d.gpu_step(op, c)
            g = torch.stack([c["ws"][:16].view(torch.float64) for c in ctxs]).max(dim=0).values
            for c in ctxs:
                c["ws"][:16].view(torch.float64).copy_(g)
    for c in ctxs:
        for op in ops:
            if op.op in (d.OP_BCAST, d.OP_ALLREDUCE_NORMS, d.OP_RECORD, d.OP_WAIT, d.OP_NORMS):
                continue
            kinds.add(op.op)
            d.gpu_step(op, c)
    torch.cuda.synchronize()
    return torch.cat([c["out"] for c in ctxs]), kinds


@pytest.mark.parametrize("shape", [(700, 1024, 520), (333, 2048, 130), (64, 96, 64)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_steps_bitwise(shape, world):
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N + world)
    dA = torch.from_numpy(A * 1e4).to(DEV)  # lambda != 0
    dB = torch.from_numpy(B).to(DEV)
    for m in METHODS:
        for levels in ((1, 2, 3) if m.startswith("strassen") else (2,)):
            kw = {"levels": levels} if m.startswith("strassen") else {}
            if m.startswith("strassen"):  # recursion on each shard: the one-GPU call on that shard
                ref = torch.cat([getattr(mm, m)(dA[lo:hi], dB, **kw) for lo, hi in
                                 (d.shard_rows(N, world, r) for r in range(world)) if hi > lo])
            else:
                ref = getattr(mm, m)(dA, dB)
            for panels in (1, 2, 5):
                C, kinds = _run_ranks(m, dA, dB, world, panels, levels)
                assert torch.equal(C, ref), (m, world, panels, levels, (C - ref).abs().max().item())
                if panels > 1:
                    assert d.OP_FULL not in kinds, (m, panels, levels)


def test_scaled_panels_lambda_nonzero():
    A, B = workload.custom(256, 512, 192, seed=9)
    dA, dB = torch.from_numpy(A * 1e6).to(DEV), torch.from_numpy(B * 1e-6).to(DEV)
    C0, lam = mm.winograd_scaled(dA, dB, return_lambda=True)
    assert lam != 0
    C, _ = _run_ranks("winograd_scaled", dA, dB, 4, 4, 2)
    assert torch.equal(C, C0)


def test_odd_shapes_take_the_one_shot_path():
    # odd P (c3-like): Kahan / Winograd / scaled keep one broadcast and the one-shot kernel
    A, B = workload.custom(130, 1001, 66, seed=5)
    dA, dB = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    for m in ("kahan", "winograd", "winograd_scaled"):
        C, kinds = _run_ranks(m, dA, dB, 2, 4, 2)
        assert kinds == {d.OP_FULL}
        assert torch.equal(C, getattr(mm, m)(dA, dB)), m
    C, kinds = _run_ranks("naive", dA, dB, 2, 4, 2)  # odd P: even k-panels, odd last panel
    assert d.OP_PANEL in kinds and torch.equal(C, mm.naive(dA, dB))


def test_misaligned_shard_keeps_the_collectives():
    # a rank whose A shard is only 8-byte aligned cannot take the TMA-fed panel kernels.
    # The schedule (hence the collectives) does not depend on the shard; the rank's PANEL steps skip
    # and the one-shot kernel runs at the last one -- bitwise the same rows.
    N, P, M = 96, 256, 130
    A, B = workload.custom(N, P, M, seed=21)
    dB = torch.from_numpy(B).to(DEV)
    flat = torch.empty(N * P + 1, dtype=torch.float64, device=DEV)
    A8 = flat[1:].view(N, P)  # data_ptr % 16 == 8
    A8.copy_(torch.from_numpy(A))
    assert A8.data_ptr() % 16 == 8
    for m in ("kahan", "winograd", "kahan_fused", "winograd_fused"):
        ops = d.schedule(m, P, M, 2, 4)
        assert any(o.op == d.OP_PANEL for o in ops)
        ref = getattr(mm, m)(torch.from_numpy(A).to(DEV), dB)
        nb = d.workspace_bytes(m, N, P, M, 2)
        ctx = dict(method=m, A=A8, B=dB, out=torch.full((N, M), np.nan, dtype=torch.float64, device=DEV), levels=2,
                   is_root=True, ws=torch.empty(max(nb, 1), dtype=torch.uint8, device=DEV) if nb else None)
        for o in ops:
            if o.op not in (d.OP_BCAST, d.OP_ALLREDUCE_NORMS, d.OP_RECORD, d.OP_WAIT):
                d.gpu_step(o, ctx)
        torch.cuda.synchronize()
        assert torch.equal(ctx["out"], ref), m
