"""The alternative partition (include/mm.h mm_s7_*) on the GPU: every rank's
compute ops of mm_s7_schedule run through mm_s7_step on one GPU, each rank with its own workspace,
the broadcasts being the shared A / B and SEND_H / RECV_H a copy of the H slot from the owner's
workspace into the root's.  The root's C must be bitwise the one-GPU strassen /
strassen_winograd product with the same levels (the seven level-1 nodes are multiplied with the
one-GPU recursion, levels - 1 deep), for world sizes 1..8, any root, and padded shapes; the rank
with no product (world 8) runs no kernel.  The gloo runs of the same schedules are in
test_dist_s7_cpu.py; the NCCL executors at world 1 in test_gpu_dist_nccl.py."""
import numpy as np
import pytest
import torch

import workload

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_1106_1347_b200")
from paper_1106_1347_b200 import dist as d  # noqa: E402

DEV = torch.device("cuda", 0)


def _emulate(m, A, B, levels, world, root):
    N, P = A.shape
    M = B.shape[1]
    nbytes = d.s7_workspace_bytes(m, N, P, M, levels)
    ws = [torch.full((nbytes,), 0xFF, dtype=torch.uint8, device=DEV) for _ in range(world)]  # NaN-filled
    C = torch.full((N, M), np.nan, dtype=torch.float64, device=DEV)
    order = [r for r in range(world) if r != root] + [root]  # senders compute before the root receives
    launches = {}
    for r in order:
        ctx = dict(method=m, A=A, B=B, out=C if r == root else None, levels=levels, ws=ws[r])
        n0 = mm.launch_count()
        for op in d.s7_schedule(m, N, P, M, levels, world, r, root):
            if op.op in (d.OP_S7_FORM, d.OP_S7_PRODUCT, d.OP_S7_COMBINE):
                d.s7_gpu_step(op, ctx)
            elif op.op == d.OP_RECV_H:
                d.s7_h_slot(ws[r], op.index, N, P, M, levels).copy_(
                    d.s7_h_slot(ws[int(op.lo)], op.index, N, P, M, levels))
        launches[r] = mm.launch_count() - n0
    torch.cuda.synchronize()
    return C, launches


@pytest.mark.parametrize("shape", [(512, 512, 512), (700, 1024, 520), (333, 1001, 130), (64, 96, 64)])
def test_s7_bitwise_one_gpu(shape):
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N + P)
    dA, dB = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    for m in ("strassen", "strassen_winograd"):
        for levels in (1, 2, 3):
            ref = getattr(mm, m)(dA, dB, levels=levels)
            for world, root in ((1, 0), (2, 0), (3, 2), (7, 3), (8, 0)):
                C, launches = _emulate(m, dA, dB, levels, world, root)
                assert torch.equal(C, ref), (m, levels, world, root, (C - ref).abs().max().item())
                if world == 8:
                    assert launches[7] == 0


def test_s7_c4_levels3():
    # the bench configuration's depth: 8192^3 would need 8 x 2.4 GB of workspaces -- 2048^3 keeps
    # the same plan shape (d = 3, 256^3 leaves of the level-1 sub-products)
    A, B = workload.custom(2048, 2048, 2048, seed=11)
    dA, dB = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    for m in ("strassen", "strassen_winograd"):
        ref = getattr(mm, m)(dA, dB, levels=3)
        C, _ = _emulate(m, dA, dB, 3, 7, 0)
        assert torch.equal(C, ref), m


def test_s7_step_errors():
    A = torch.zeros(64, 64, dtype=torch.float64, device=DEV)
    op = d.DistOp(d.OP_S7_FORM, 0, 9, 0, 0, 0)  # product index out of range
    nbytes = d.s7_workspace_bytes("strassen", 64, 64, 64, 2)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    with pytest.raises(mm.MMError):
        d.s7_gpu_step(op, dict(method="strassen", A=A, B=A, out=None, levels=2, ws=ws))
    op = d.DistOp(d.OP_S7_FORM, 0, 0, 0, 0, 0)
    with pytest.raises(mm.MMError):  # workspace too small
        d.s7_gpu_step(op, dict(method="strassen", A=A, B=A, out=None, levels=2, ws=ws[:nbytes // 2]))
    op = d.DistOp(d.OP_S7_COMBINE, 0, 0, 0, 0, 0)
    with pytest.raises(mm.MMError):  # the root's C is required
        d.s7_gpu_step(op, dict(method="strassen", A=A, B=A, out=None, levels=2, ws=ws))
