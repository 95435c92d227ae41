"""The alternative partition (include/mm.h mm_s7_*): Strassen's seven
top-level products (PAPER.md:270-277 / 299-306) on the ranks.  Multi-process (gloo, CPU) runs of
the op lists mm_s7_schedule builds -- the lists mm_dist_strassen7 executes with NCCL -- driven by
paper_1106_1347_b200.dist.strassen7 with every compute op emulated by the oracle: the root's C must
be bitwise the one-process oracle Strassen / Strassen-Winograd product with the same levels, for
world sizes 1..8 (world 8: one rank without a product) and padded shapes.  Plus host-only
invariants of the schedules."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = ("strassen", "strassen_winograd")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _child(oracle, variant, side, X11, X12, X21, X22, p):
    """Operand p (H_{p+1}) of one node from its quadrants: P:271-277 (StrassenNaiv) / P:300-306
    (StrassenWinograd), restated with the oracle's elementwise Plus / Minus."""
    add, sub = oracle.plus, oracle.minus
    if variant == "strassen":
        if side == 0:
            return [add(X11, X22), add(X21, X22), X11, X22, add(X11, X12), sub(X21, X11), sub(X12, X22)][p]
        return [add(X11, X22), X11, sub(X12, X22), sub(X21, X11), X22, add(X11, X12), add(X21, X22)][p]
    if side == 0:
        A1 = sub(X11, X21)
        A2 = sub(X22, A1)
        return [X11, X12, A2, add(X21, X22), A1, sub(X12, A2), X22][p]
    B1 = sub(X22, X12)
    B2 = add(B1, X11)
    return [X11, X21, B2, sub(X12, X11), B1, X22, sub(X21, B2)][p]


def _combine(oracle, variant, H):
    """C11, C12, C21, C22 from H_1..H_7: P:279-282 / P:308-311, left to right as displayed."""
    add, sub = oracle.plus, oracle.minus
    H1, H2, H3, H4, H5, H6, H7 = H
    if variant == "strassen":
        return (add(sub(add(H1, H4), H5), H7), add(H3, H5), add(H2, H4), add(sub(add(H1, H3), H2), H6))
    H8 = add(H1, H3)
    H9 = add(H8, H4)
    return add(H1, H2), add(H9, H6), add(add(H8, H5), H7), add(H9, H5)


def _oracle_step(op, ctx):
    import oracle
    from paper_1106_1347_b200 import dist as d

    m, levels = ctx["method"], ctx["levels"]
    A, B = ctx["A"].numpy(), ctx["B"].numpy()
    N, P = A.shape
    M = B.shape[1]
    _, (Np, Pp, Mp) = oracle.plan(N, P, M, levels)
    h, k, w = Np // 2, Pp // 2, Mp // 2
    ctx["trace"].append((op.op, op.index))
    if op.op == d.OP_S7_FORM:
        assert np.array_equal(A, ctx["A_true"]) and np.array_equal(B, ctx["B_true"]), "A / B not arrived"
        Ae = np.zeros((Np, Pp))
        Ae[:N, :P] = A
        Be = np.zeros((Pp, Mp))
        Be[:P, :M] = B
        ctx["L"] = _child(oracle, m, 0, Ae[:h, :k], Ae[:h, k:], Ae[h:, :k], Ae[h:, k:], op.index)
        ctx["R"] = _child(oracle, m, 1, Be[:k, :w], Be[:k, w:], Be[k:, :w], Be[k:, w:], op.index)
    elif op.op == d.OP_S7_PRODUCT:
        H = oracle.strassen(0 if m == "strassen" else 1, ctx["L"], ctx["R"], levels=levels - 1, pad=(h, k, w),
                            base=oracle.BASE_FMA)
        ctx["slots"][op.index][...] = torch.from_numpy(H)
    elif op.op == d.OP_S7_COMBINE:
        H = [ctx["slots"][p].numpy() for p in range(7)]
        assert all(np.isfinite(x).all() for x in H), "combination before every H arrived"
        Cq = _combine(oracle, m, H)
        C = np.block([[Cq[0], Cq[1]], [Cq[2], Cq[3]]])
        ctx["out"].numpy()[...] = C[:N, :M]
    else:
        raise AssertionError(f"unexpected compute op {op!r}")


CASES = [(9, 13, 7, 1), (9, 13, 7, 2), (16, 8, 16, 3), (20, 12, 10, 2), (1, 1, 1, 1)]


def _worker(rank, world, port, seed, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import workload
        from paper_1106_1347_b200.dist import strassen7

        out = {}
        root = world - 1 if world > 2 else 0  # a root other than rank 0 too
        for N, P, M, levels in CASES:
            A, B = workload.custom(N, P, M, seed=seed + N + P + M)
            _, (Np, Pp, Mp) = oracle.plan(N, P, M, levels)
            for m in VARIANTS:
                At = torch.from_numpy(A.copy()) if rank == root else torch.full((N, P), np.nan, dtype=torch.float64)
                Bt = torch.from_numpy(B.copy()) if rank == root else torch.full((P, M), np.nan, dtype=torch.float64)
                slots = [torch.full((Np // 2, Mp // 2), np.nan, dtype=torch.float64) for _ in range(7)]
                ctx = {"A_true": A, "B_true": B, "trace": [], "slots": slots}
                C = strassen7(m, At, Bt, root=root, levels=levels, step=_oracle_step, ctx=ctx,
                              slot=lambda c, p: c["slots"][p])
                assert np.array_equal(At.numpy(), A) and np.array_equal(Bt.numpy(), B)
                if rank == root:
                    out[(m, N, P, M, levels)] = C.numpy().copy()
                else:
                    assert C is None
                from paper_1106_1347_b200 import dist as d

                own = sorted(i for k, i in ctx["trace"] if k in (d.OP_S7_FORM, d.OP_S7_PRODUCT))
                assert own == sorted([p for p in range(7) if p % world == rank] * 2), (rank, ctx["trace"])
                assert ((d.OP_S7_COMBINE, 0) in ctx["trace"]) == (rank == root)
        q.put((rank, root, out))
    except BaseException as e:
        import traceback

        q.put((rank, "error", traceback.format_exc()))
        raise e
    finally:
        dist.destroy_process_group()


def _run(world, seed=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in procs:
            r = q.get(timeout=300)
            assert r[1] != "error", r[2]
            res.append(r)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    return res


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_s7_bitwise_one_process_strassen(world):
    import oracle
    import workload

    res = _run(world)
    roots = {r[1] for r in res}
    assert len(roots) == 1
    root = roots.pop()
    out = next(r[2] for r in res if r[0] == root)
    assert len(out) == len(CASES) * len(VARIANTS)
    for N, P, M, levels in CASES:
        A, B = workload.custom(N, P, M, seed=3 + N + P + M)
        lv, pad = oracle.plan(N, P, M, levels)
        for m in VARIANTS:
            ref = oracle.strassen(0 if m == "strassen" else 1, A, B, levels=lv, pad=pad, base=oracle.BASE_FMA)
            assert np.array_equal(out[(m, N, P, M, levels)], ref), (world, m, N, P, M, levels)


def test_s7_schedule_invariants():
    """Every product formed and multiplied exactly once over the ranks, on its owner p % world;
    every non-root owner sends its H to the root once, after computing it, and the root receives
    exactly the H's it does not compute, before combining; every rank takes part in both
    broadcasts (A and B, all rows) before any compute op."""
    from paper_1106_1347_b200 import dist as d

    for m in VARIANTS:
        for world in range(1, 10):
            for root in sorted({0, world - 1, world // 2}):
                made, sent, recv = [], [], []
                for rank in range(world):
                    ops = d.s7_schedule(m, 100, 37, 55, 2, world, rank, root)
                    kinds = [o.op for o in ops]
                    assert kinds[:2] == [d.OP_BCAST_A, d.OP_BCAST]
                    assert (ops[0].lo, ops[0].hi, ops[1].lo, ops[1].hi) == (0, 100, 0, 37)
                    ready = set()
                    for i, o in enumerate(ops):
                        if o.op == d.OP_S7_FORM:
                            assert o.index % world == rank and ops[i + 1].op == d.OP_S7_PRODUCT
                            assert ops[i + 1].index == o.index
                            assert any(x.op == d.OP_WAIT and x.index == 0 and x.stream == d.STREAM_COMPUTE
                                       for x in ops[:i])
                            made.append(o.index)
                        elif o.op == d.OP_S7_PRODUCT:
                            ready.add(o.index)
                        elif o.op == d.OP_SEND_H:
                            assert rank != root and o.lo == root and o.index in ready
                            sent.append(o.index)
                        elif o.op == d.OP_RECV_H:
                            assert rank == root and o.lo == o.index % world != root
                            recv.append(o.index)
                        elif o.op == d.OP_S7_COMBINE:
                            assert rank == root and i == len(ops) - 1
                            assert sorted(recv + list(ready)) == list(range(7))
                    if rank != root:
                        assert d.OP_S7_COMBINE not in kinds and d.OP_RECV_H not in kinds
                assert sorted(made) == list(range(7)), (m, world, root)
                assert sorted(sent) == sorted(recv) == sorted(p for p in range(7) if p % world != root)


def test_s7_rejects():
    import paper_1106_1347_b200 as mm
    from paper_1106_1347_b200 import dist as d

    with pytest.raises(mm.MMError):
        d.s7_schedule("naive", 16, 16, 16, 2, 2, 0)
    with pytest.raises(mm.MMError):
        d.s7_schedule("strassen", 16, 16, 16, 0, 2, 0)  # levels >= 1
    with pytest.raises(mm.MMError):
        d.s7_schedule("strassen", 16, 16, 16, 2, 2, 2)  # rank out of range
    assert d.s7_workspace_bytes("strassen", 16, 16, 16, 0) == 0
    assert d.s7_workspace_bytes("kahan", 16, 16, 16, 2) == 0
    # 7 H slots of (Np/2)(Mp/2) doubles, the two level-1 operands, the levels-1 sub-product's arena
    ws = d.s7_workspace_bytes("strassen", 64, 64, 64, 1)
    assert ws >= 7 * 32 * 32 * 8 + 2 * 32 * 32 * 8
