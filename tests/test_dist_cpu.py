"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU schedule: the op list the C library
builds (mm_dist_schedule -- the same list mm_dist_gemm executes with NCCL) executed by
paper_1106_1347_b200.dist over gloo, with every compute op emulated by the oracle.  This covers
sharding, the panelised broadcast of B, the max-all-reduce of {||A_r||, ||B||} and lambda, and the
order of every compute op against the arrival of the B rows it reads (B is NaN on non-root ranks
until its rows land), for every method, several panel counts and Strassen depths; the per-rank
results must be bitwise the rows of the 1-process oracle product."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


FIRST_SPAN = {1: 1, 2: 2, 3: 3, 4: 2, 5: 3}  # levels of the first formation pass


def _oracle_step(op, ctx):
    """Emulates one compute op of the schedule with the oracle (the arithmetic the GPU kernels are
    checked against bitwise elsewhere) and checks that every B row the op reads has arrived."""
    import oracle
    from paper_1106_1347_b200 import dist as d

    m, levels = ctx["method"], ctx["levels"]
    A, B, C = ctx["A"].numpy(), ctx["B"].numpy(), ctx["out"].numpy()
    N, P = A.shape
    M = B.shape[1]
    Bt = ctx["B_true"]
    fused = m.endswith("_fused")
    ctx["trace"].append(op.op)

    def arrived(lo, hi):
        assert np.array_equal(B[lo:hi], Bt[lo:hi]), (repr(op), "reads B rows that have not arrived")

    if op.op == d.OP_NORMS:
        ctx["norms"][0] = oracle.norm_inf(A) if N else 0.0
        ctx["norms"][1] = oracle.norm_inf(B) if ctx["is_root"] else 0.0
        return
    if N == 0:
        return
    lam = oracle.lam(float(ctx["norms"][0]), float(ctx["norms"][1])) if m.startswith("winograd_scaled") else 0
    if op.op == d.OP_PANEL:
        arrived(op.lo, op.hi)
        first, last = not op.flags & d.EX_ACCUMULATE, not op.flags & d.EX_KEEP_STATE
        assert bool(op.flags & d.EX_FUSED) == fused
        if first:
            C[...] = 0.0
        k0, k1 = op.lo, op.hi
        if m == "naive":
            oracle.naive_fma_acc(A[:, k0:k1], B[k0:k1], C)
        elif m.startswith("kahan"):
            if first:
                ctx["E"] = np.zeros_like(C)
            oracle.naive_kahan_acc(A[:, k0:k1], B[k0:k1], C, ctx["E"], fused)
        elif m.startswith("winograd_scaled"):
            oracle.winograd_pairs_acc(ctx["As"][:, k0:k1], ctx["Bs"][k0:k1], C, fused)
            if last:
                arrived(0, P)
                yz = oracle.winograd_yz_fused if fused else oracle.winograd_yz
                C[...] = oracle.winograd_finish(C, *yz(ctx["As"], ctx["Bs"]))
        else:
            oracle.winograd_pairs_acc(A[:, k0:k1], B[k0:k1], C, fused)
            if last:
                C[...] = oracle.winograd_finish(C, *ctx["yz"])
    elif op.op == d.OP_YZ:
        arrived(0, P)
        ctx["yz"] = (oracle.winograd_yz_fused if fused else oracle.winograd_yz)(A, B)
    elif op.op == d.OP_SCALE_A:
        ctx["As"] = oracle.scalar_mul(2.0 ** lam, A)
        ctx["Bs"] = np.full((P, M), np.nan)
    elif op.op == d.OP_SCALE_B:
        arrived(op.lo, op.hi)
        ctx["Bs"][op.lo:op.hi] = oracle.scalar_mul(2.0 ** -lam, B[op.lo:op.hi])
    elif op.op in (d.OP_FORM_A, d.OP_FORM_B, d.OP_FORM_B_REST):
        span, h = _first_pass_units(P, levels)
        if op.op == d.OP_FORM_B:  # quadrant rows [lo, hi) read B rows u + r h, r < 2^span
            for r in range(1 << span):
                arrived(min(P, r * h + op.lo), min(P, r * h + op.hi))
            ctx.setdefault("formed", set()).update(range(op.lo, op.hi))
        elif op.op == d.OP_FORM_B_REST:
            assert ctx.get("formed") == set(range(h)), "B-side formation of every unit before the rest"
    elif op.op == d.OP_LEAF_COMBINE:
        arrived(0, P)
        assert ctx.get("formed", set(range(_first_pass_units(P, levels)[1]))) == set(
            range(_first_pass_units(P, levels)[1]))
        C[...] = _oracle_full(m, A, B, levels, lam)
    elif op.op == d.OP_FULL:
        arrived(0, P)
        C[...] = _oracle_full(m, A, B, levels, lam)
    else:
        raise AssertionError(f"unexpected compute op {op!r}")


def _first_pass_units(P, levels):
    # reading R10: P padded to a multiple of 2^(levels+1); the first pass spans FIRST_SPAN levels
    q = 2 << levels
    span = FIRST_SPAN[levels]
    return span, (-(-P // q) * q) >> span


def _oracle_full(m, A, B, levels, lam):
    import oracle

    N, P, M = A.shape[0], A.shape[1], B.shape[1]
    if m in ("strassen", "strassen_winograd"):
        lv, pad = oracle.plan(N, P, M, levels)
        return oracle.strassen(0 if m == "strassen" else 1, A, B, levels=lv, pad=pad, base=oracle.BASE_FMA)
    if m.startswith("winograd_scaled"):
        code = oracle.M_WINOGRAD_SCALED_FUSED if m.endswith("_fused") else oracle.M_WINOGRAD_SCALED
        idx = [(i, j) for i in range(N) for j in range(M)]
        return oracle.entries(code, A, B, idx, lam).reshape(N, M)
    return {"naive": oracle.naive_fma, "kahan": oracle.naive_kahan, "kahan_fused": oracle.naive_kahan_fused,
            "winograd": oracle.winograd_original, "winograd_fused": oracle.winograd_fused}[m](A, B)


METHODS = ("naive", "kahan", "kahan_fused", "winograd", "winograd_fused", "winograd_scaled",
           "winograd_scaled_fused", "strassen", "strassen_winograd")


def _worker(rank, world, port, N, P, M, seed, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workload
        from paper_1106_1347_b200.dist import dist_gemm, shard_rows

        A, B = workload.custom(N, P, M, seed=seed)
        A = A * 1e5  # make lambda non-zero
        lo, hi = shard_rows(N, world, rank)
        assert (lo, hi) == workload.shard_rows(N, world, rank)
        A_loc = torch.from_numpy(np.ascontiguousarray(A[lo:hi]))
        out, traces = {}, {}
        for panels in (1, 2, 3, 5):
            for m in METHODS:
                for levels in ((1, 2, 3) if m.startswith("strassen") else (2,)):
                    # B re-broadcast from scratch: NaN everywhere but on the root
                    Bp = torch.from_numpy(B.copy()) if rank == 0 else torch.full((P, M), np.nan, dtype=torch.float64)
                    ctx = {"B_true": B, "trace": []}
                    C = dist_gemm(m, A_loc, Bp, panels=panels, levels=levels, step=_oracle_step, ctx=ctx)
                    assert np.array_equal(Bp.numpy(), B)  # the broadcast delivered all of B
                    out[(m, panels, levels)] = C.numpy().copy()
                    traces[(m, panels, levels)] = ctx["trace"]
        q.put((rank, lo, hi, out, traces))
    except BaseException as e:  # report instead of leaving the parent waiting on the queue
        import traceback

        q.put((rank, "error", traceback.format_exc(), None, None))
        raise e
    finally:
        dist.destroy_process_group()


def test_schedule_panel_bounds():
    # the k-panels of the C schedule: consecutive, even boundaries, at most `panels` of them
    from paper_1106_1347_b200 import dist as d

    for P in (2, 16, 1000, 8192):
        for n in (2, 3, 8, 64):
            b = [(o.lo, o.hi) for o in d.schedule("naive", P, 64, 2, n) if o.op == d.OP_PANEL]
            assert b[0][0] == 0 and b[-1][1] == P
            assert all(k0 < k1 for k0, k1 in b) and all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
            assert all(k0 % 2 == 0 for k0, _ in b)
            assert len(b) <= n


def test_schedule_covers_b_once():
    # every row of B is broadcast exactly once, whatever the method, levels and panel count
    from paper_1106_1347_b200 import dist as d

    for m in METHODS:
        for P, M in ((8192, 8192), (1001, 3000), (20, 10), (13, 7)):
            for lv in (-1, 0, 1, 2, 3, 4, 5):
                for n in (1, 2, 5, 64):
                    rows = np.zeros(P, dtype=np.int64)
                    for o in d.schedule(m, P, M, lv, n):
                        if o.op == d.OP_BCAST:
                            rows[o.lo:o.hi] += 1
                    assert (rows == 1).all(), (m, P, M, lv, n)


def _run(world, N, P, M, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, P, M, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in procs:
            r = q.get(timeout=240)
            assert r[1] != "error", r[2]
            res.append(r)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        for p in procs:  # a rank left waiting in a collective by a failed peer
            if p.is_alive():
                p.kill()
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("world,shape", [(2, (9, 13, 7)), (2, (1, 5, 3)), (2, (16, 8, 16)), (2, (7, 20, 10)),
                                         (2, (12, 32, 6)), (3, (2, 6, 5)), (4, (11, 10, 9))])
def test_row_sharded_bitwise(world, shape):
    """world 3 with N = 2 leaves rank 2 without rows (it still takes part in every collective);
    world 4 with N = 11 gives shards of 3, 3, 3, 2 rows."""
    import oracle
    import workload

    N, P, M = shape
    res = _run(world, N, P, M, seed=N + P + M)
    A, B = workload.custom(N, P, M, seed=N + P + M)
    A = A * 1e5
    full = {m: _oracle_full(m, A, B, 0, 0) for m in METHODS if not m.startswith(("winograd_scaled", "strassen"))}
    C, lam = oracle.winograd_scaled(A, B)
    assert lam != 0
    full["winograd_scaled"] = C
    full["winograd_scaled_fused"] = oracle.winograd_scaled_fused(A, B)[0]
    for rank, lo, hi, out, traces in res:
        for (m, panels, levels), Cr in out.items():
            assert Cr.shape == (hi - lo, M)
            if hi == lo:
                continue
            if m.startswith("strassen"):  # recursion on the shard: the oracle on the same shard
                assert np.array_equal(Cr, _oracle_full(m, A[lo:hi], B, levels, 0)), (rank, m, panels, levels)
            else:
                assert np.array_equal(Cr, full[m][lo:hi]), (rank, m, panels)
    assert sum(hi - lo for _, lo, hi, _, _ in res) == N
    # the panel paths really ran where the schedule allows them
    _, _, _, _, traces = res[0]
    from paper_1106_1347_b200 import dist as d

    assert d.OP_PANEL in traces[("naive", 3, 2)]
    assert (d.OP_PANEL in traces[("winograd_scaled", 3, 2)]) == (P % 2 == 0 and M % 2 == 0)
    assert d.OP_FORM_B in traces[("strassen_winograd", 2, 2)]


def test_schedule_invariants_random():
    """Properties of mm_dist_schedule over random (method, P, M, levels, panels), checked by
    simulating which rows of B have arrived at every compute op: each row is broadcast exactly once;
    a compute op only reads rows whose broadcast it has waited for (PANEL / SCALE_B: its k-range;
    FORM_B: its units' 2^span row ranges; YZ / FULL / LEAF_COMBINE / FORM_B_REST: all of B); every
    RECORD precedes its WAIT; the norms are all-reduced before anything reads lambda; PANEL k-ranges
    tile [0, P) in increasing order with the accumulate / keep-state flags of a first / last panel."""
    import random

    from paper_1106_1347_b200 import dist as d

    rng = random.Random(11061347)
    for _ in range(400):
        m = rng.choice(METHODS)
        P, M = rng.randint(1, 5000), rng.randint(1, 300)
        lv = rng.choice((-1, 0, 1, 2, 3, 4, 5))
        n = rng.choice((1, 2, 3, 4, 7, 8, 16, 64))
        ops = d.schedule(m, P, M, lv, n)
        sent = np.zeros(P, dtype=np.int64)
        pending, recorded, waited = [], {}, set()
        arrived = np.zeros(P, dtype=bool)
        reduced = False
        norms_done = False
        panels = []
        for o in ops:
            if o.op == d.OP_BCAST:
                sent[o.lo:o.hi] += 1
                pending.append((o.lo, o.hi))
            elif o.op == d.OP_ALLREDUCE_NORMS:
                assert norms_done, "all-reduce before the local norms"
                pending.append("norms")
            elif o.op == d.OP_RECORD:
                if o.stream == d.STREAM_COMM:
                    recorded[o.index] = pending
                    pending = []
                else:
                    recorded[o.index] = ["compute"]
            elif o.op == d.OP_WAIT:
                assert o.index in recorded, "wait before record"
                if o.stream == d.STREAM_COMPUTE:
                    for item in recorded[o.index]:
                        if item == "norms":
                            reduced = True
                        elif item != "compute":
                            arrived[item[0]:item[1]] = True
                waited.add(o.index)
            else:
                if o.op == d.OP_NORMS:
                    norms_done = True
                    continue
                if o.op in (d.OP_SCALE_A, d.OP_SCALE_B, d.OP_FULL) and m.startswith("winograd_scaled"):
                    assert reduced, "lambda read before the norms were all-reduced"
                if o.op in (d.OP_PANEL, d.OP_SCALE_B):
                    assert arrived[o.lo:o.hi].all(), (m, o)
                    if o.op == d.OP_PANEL:
                        panels.append(o)
                elif o.op == d.OP_FORM_B:
                    span = FIRST_SPAN[lv]
                    q = 2 << lv
                    h = (-(-P // q) * q) >> span
                    for r in range(1 << span):
                        a, b = min(P, r * h + o.lo), min(P, r * h + o.hi)
                        assert arrived[a:b].all(), (m, o)
                elif o.op in (d.OP_YZ, d.OP_FULL, d.OP_LEAF_COMBINE, d.OP_FORM_B_REST):
                    assert arrived.all(), (m, o)
        assert (sent == 1).all(), (m, P, M, lv, n)
        if panels:
            assert panels[0].lo == 0 and panels[-1].hi == P
            assert all(a.hi == b.lo for a, b in zip(panels, panels[1:]))
            assert not panels[0].flags & d.EX_ACCUMULATE and all(p.flags & d.EX_ACCUMULATE for p in panels[1:])
            assert not panels[-1].flags & d.EX_KEEP_STATE
            assert all(p.flags & d.EX_KEEP_STATE for p in panels[:-1]) or m == "naive"
            assert all(bool(p.flags & d.EX_FUSED) == m.endswith("_fused") for p in panels)
