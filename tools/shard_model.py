"""Per-rank timing of the multi-GPU schedule on ONE GPU, and the modelled scaling it implies.

Only one GPU is reachable from this sandbox, so the g-GPU run is measured rank by rank: for each
method of bench.py's step and g in (1, 2, 4, 8), the compute ops of rank 0's schedule
(mm_dist_schedule -- the list mm_dist_gemm and dist.dist_gemm execute) run on rank 0's shard
(ceil(N/g) rows) with B already resident, each op timed with CUDA events.  The broadcast is then
modelled: the communication ops run back to back on their own stream at `--link-gbs` (default
770 GB/s), panel i landing at sum_{j <= i} bytes_j / bw, and a compute op that
waits for panel i starts at max(end of the previous op, arrival of panel i).  T_g is the modelled
end of the last op; E_g = T_1 / (g T_g) with T_1 the one-GPU call of the whole problem.

    python tools/shard_model.py [--config c4] [--methods ...] [--levels 3] [--panels 8] [--out f.jsonl]

--s7 models the alternative partition instead (include/mm.h mm_s7_*: Strassen's seven top-level
products on the ranks): every product's S7_FORM + S7_PRODUCT and the root's S7_COMBINE timed on
one GPU; A and B broadcast at the link rate before any compute, each non-root H (8 (Np/2)(Mp/2)
bytes) sent once its product ends, the root's inbound link receiving them one after another, the
combination after the last one.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1106_1347_b200 as mm  # noqa: E402
import workload  # noqa: E402
from paper_1106_1347_b200 import dist as d  # noqa: E402

COMM = (d.OP_BCAST, d.OP_ALLREDUCE_NORMS, d.OP_RECORD, d.OP_WAIT)


def time_ops(m, A, B, ops, levels, reps):
    """Median time (ms) of every compute op of `ops` on this shard (B complete, norms = the
    shard's own: the all-reduce is a max of 8 bytes and does not change the work)."""
    N, P = A.shape
    M = B.shape[1]
    nb = d.workspace_bytes(m, N, P, M, levels)
    ctx = dict(method=m, A=A, B=B, out=torch.empty((N, M), dtype=torch.float64, device=B.device), levels=levels,
               is_root=True, ws=torch.zeros(max(nb, 1), dtype=torch.uint8, device=B.device) if nb else None)
    compute = [o for o in ops if o.op not in COMM]
    samples = [[] for _ in compute]
    for r in range(reps + 1):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in compute]
        for (e0, e1), o in zip(evs, compute):
            e0.record()
            d.gpu_step(o, ctx)
            e1.record()
        torch.cuda.synchronize()
        if r:
            for s, (e0, e1) in zip(samples, evs):
                s.append(e0.elapsed_time(e1))
    return [statistics.median(s) for s in samples], ctx["out"]


def model(ops, op_ms, M, link_gbs, allreduce_us=25.0):
    """Modelled end time (ms) of the schedule: comm ops serial at link_gbs, compute ops serial,
    joined by the schedule's record / wait events."""
    t_comm = t_comp = 0.0
    ev = {}
    it = iter(op_ms)
    bcast_ms = 0.0
    for o in ops:
        if o.op == d.OP_BCAST:
            dt = 8.0 * (o.hi - o.lo) * M / (link_gbs * 1e9) * 1e3
            t_comm += dt
            bcast_ms += dt
        elif o.op == d.OP_ALLREDUCE_NORMS:
            t_comm += allreduce_us / 1e3
        elif o.op == d.OP_RECORD:
            ev[o.index] = t_comm if o.stream == d.STREAM_COMM else t_comp
        elif o.op == d.OP_WAIT:
            if o.stream == d.STREAM_COMM:
                t_comm = max(t_comm, ev.get(o.index, 0.0))
            else:
                t_comp = max(t_comp, ev.get(o.index, 0.0))
        else:
            t_comp += next(it)
    return max(t_comp, t_comm), bcast_ms


def s7_rows(a, cfg, A, B, T1):
    """Modelled T_g of the seven-products partition for the Strassen methods (see the docstring)."""
    N, P, M = cfg.N, cfg.P, cfg.M
    rows = []
    for m in (x for x in a.methods.split(",") if x.startswith("strassen")):
        nb = d.s7_workspace_bytes(m, N, P, M, a.levels)
        ws = torch.zeros(nb, dtype=torch.uint8, device=B.device)
        C = torch.empty((N, M), dtype=torch.float64, device=B.device)
        ctx = dict(method=m, A=A, B=B, out=C, levels=a.levels, ws=ws)
        form, prod = [0.0] * 7, [0.0] * 7
        comb = 0.0
        for r in range(a.reps + 1):
            evs = []
            for p in range(7):
                for kind in (d.OP_S7_FORM, d.OP_S7_PRODUCT):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    d.s7_gpu_step(d.DistOp(kind, 0, p, 0, 0, 0), ctx)
                    e1.record()
                    evs.append((kind, p, e0, e1))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            d.s7_gpu_step(d.DistOp(d.OP_S7_COMBINE, 0, 0, 0, 0, 0), ctx)
            e1.record()
            torch.cuda.synchronize()
            if r:  # mean over the timed repetitions
                for kind, p, x0, x1 in evs:
                    (form if kind == d.OP_S7_FORM else prod)[p] += x0.elapsed_time(x1) / a.reps
                comb += e0.elapsed_time(e1) / a.reps
        ref = getattr(mm, m)(A, B, levels=a.levels)
        torch.cuda.synchronize()
        assert torch.equal(C, ref), m  # all seven products on one rank: the one-GPU product
        _, Np, _, Mp = mm.strassen_plan(N, P, M, a.levels)
        bw = a.link_gbs * 1e9
        h_ms = 8.0 * (Np // 2) * (Mp // 2) / bw * 1e3
        in_ms = 8.0 * (N * P + P * M) / bw * 1e3
        for g in [int(x) for x in a.gpus.split(",")] + [7]:
            done = {}
            in_g = in_ms if g > 1 else 0.0  # one GPU: nothing to broadcast
            for r in range(g):
                t = in_g
                for p in range(7):
                    if p % g == r:
                        t += form[p] + prod[p]
                        done[p] = t
            root_compute = max([done[p] for p in range(7) if p % g == 0] + [in_g])
            link = 0.0
            for p in sorted((p for p in range(7) if p % g != 0), key=lambda p: done[p]):
                link = max(link, done[p]) + h_ms
            t = max(root_compute, link) + comb
            rows.append({"config": a.config, "method": m, "partition": "s7", "g": g, "levels": a.levels,
                         "inputs_bcast_ms": round(in_ms, 3), "h_send_ms": round(h_ms, 3),
                         "form_ms": [round(x, 4) for x in form], "product_ms": [round(x, 3) for x in prod],
                         "combine_ms": round(comb, 4), "modelled_T_g_ms": round(t, 3), "T_1_ms": round(T1[m], 3),
                         "E_g": round(T1[m] / (g * t), 4), "link_gbs": a.link_gbs})
            print(json.dumps(rows[-1]), flush=True)
        del ws, C
        torch.cuda.empty_cache()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--methods", default=",".join(bench.METHODS))
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--panels", type=int, default=8)
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--link-gbs", type=float, default=770.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--s7", action="store_true", help="model the seven-products partition of the Strassen methods")
    a = ap.parse_args()
    cfg = workload.CONFIGS[a.config]
    N, P, M = cfg.N, cfg.P, cfg.M
    dev = torch.device("cuda", 0)
    A = torch.from_numpy(workload.matrix(cfg, 0)).to(dev)
    B = torch.from_numpy(workload.matrix(cfg, 1)).to(dev)
    methods = a.methods.split(",")
    gs = [int(x) for x in a.gpus.split(",")]
    if a.s7:
        T1 = {}
        for m in (x for x in methods if x.startswith("strassen")):
            out = torch.empty((N, M), dtype=torch.float64, device=dev)
            getattr(mm, m)(A, B, out=out, levels=a.levels)
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                getattr(mm, m)(A, B, out=out, levels=a.levels)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            T1[m] = statistics.median(ts)
            del out
        mm.release_workspace()
        rows = s7_rows(a, cfg, A, B, T1)
        if a.out:
            with open(a.out, "w") as fh:
                for r in rows:
                    fh.write(json.dumps(r) + "\n")
        return
    rows, T1, Tg = [], {}, {g: 0.0 for g in gs}
    for m in methods:
        kw = {"levels": a.levels} if m.startswith("strassen") else {}
        f = getattr(mm, m)
        out = torch.empty((N, M), dtype=torch.float64, device=dev)
        f(A, B, out=out, **kw)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f(A, B, out=out, **kw)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        T1[m] = statistics.median(ts)
        ref = out
        pn = bench.panels_for_method(argparse.Namespace(panels=a.panels), m)
        for g in gs:
            lo, hi = d.shard_rows(N, g, 0)
            ops = d.schedule(m, P, M, a.levels, pn if g > 1 else 1)
            op_ms, C = time_ops(m, A[lo:hi], B, ops, a.levels, a.reps)
            if not m.startswith(("strassen", "winograd_scaled")):  # (scaled: lambda from the shard's norm here)
                assert torch.equal(C, ref[lo:hi]), (m, g)
            t, bms = model(ops, op_ms, M, a.link_gbs) if g > 1 else (sum(op_ms), 0.0)
            # the one-shot method on the same shard (what the panels cost over it)
            full_ms, _ = time_ops(m, A[lo:hi], B, d.schedule(m, P, M, a.levels, 1), a.levels, a.reps)
            Tg[g] += t
            row = {"config": a.config, "method": m, "g": g, "shard_rows": hi - lo, "panels": pn if g > 1 else 1,
                   "compute_ms": round(sum(op_ms), 3), "one_shot_shard_ms": round(sum(full_ms), 3),
                   "bcast_ms_at_link": round(bms, 3),
                   "modelled_T_g_ms": round(t, 3), "T_1_ms": round(T1[m], 3),
                   "E_g": round(T1[m] / (g * t), 4), "link_gbs": a.link_gbs,
                   "ops": [f"{d.OP_NAMES[o.op]}[{o.lo},{o.hi})" for o in ops if o.op not in COMM],
                   "op_ms": [round(x, 4) for x in op_ms]}
            rows.append(row)
            print(json.dumps({k: v for k, v in row.items() if k not in ("ops", "op_ms")}), flush=True)
        del out
        mm.release_workspace()
        d._WS.clear()
        torch.cuda.empty_cache()
    step1 = sum(T1.values())
    for g in gs:
        rows.append({"config": a.config, "method": "step", "g": g, "modelled_T_g_ms": round(Tg[g], 3),
                     "T_1_ms": round(step1, 3), "E_g": round(step1 / (g * Tg[g]), 4), "link_gbs": a.link_gbs})
        print(json.dumps(rows[-1]), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
