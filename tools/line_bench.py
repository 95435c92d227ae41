"""Timing of the line kernels (lines.cuh) at full-problem and shard shapes: norm_inf, Winograd's
y/z pass, and the multi-GPU WinogradScaled steps (norms, scale_a, scale_b panels), each by CUDA
events (median of --reps).  GB/s counts the bytes each pass must move (reads + copy writes).

    python tools/line_bench.py [--rows 8192,1024] [--P 8192] [--M 8192] [--reps 5]
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

import paper_1106_1347_b200 as mm  # noqa: E402
from paper_1106_1347_b200 import dist as d  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="8192,1024")
    ap.add_argument("--P", type=int, default=8192)
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    P, M = a.P, a.M
    dev = torch.device("cuda", 0)
    B = torch.randn((P, M), dtype=torch.float64, device=dev)
    tag = os.environ.get("MM_LN_MAX_STAGES", "default")
    for N in map(int, a.rows.split(",")):
        A = torch.randn((N, P), dtype=torch.float64, device=dev)
        y = torch.empty(N, dtype=torch.float64, device=dev)
        z = torch.empty(M, dtype=torch.float64, device=dev)
        out = {"rows": N, "P": P, "M": M, "ln_max_stages": tag}
        t = timed(lambda: mm.norm_inf(A), a.reps)
        out["norm_inf_A_ms"], out["norm_inf_A_gbs"] = round(t, 4), round(8 * N * P / t / 1e6, 1)
        t = timed(lambda: mm.winograd_yz(A, B, y, z), a.reps)
        out["yz_ms"], out["yz_gbs"] = round(t, 4), round(8 * (N * P + P * M) / t / 1e6, 1)
        ops = d.schedule("winograd_scaled", P, M, 2, 4)
        nb = d.workspace_bytes("winograd_scaled", N, P, M, 2)
        ctx = dict(method="winograd_scaled", A=A, B=B, out=torch.empty((N, M), dtype=torch.float64, device=dev),
                   levels=2, is_root=True, ws=torch.zeros(nb, dtype=torch.uint8, device=dev))
        for o in ops:
            if o.op == d.OP_NORMS:
                t = timed(lambda: d.gpu_step(o, ctx), a.reps)
                out["norms_AB_ms"], out["norms_AB_gbs"] = round(t, 4), round(8 * (N * P + P * M) / t / 1e6, 1)
            elif o.op == d.OP_SCALE_A:
                t = timed(lambda: d.gpu_step(o, ctx), a.reps)
                out["scale_a_ms"], out["scale_a_gbs"] = round(t, 4), round(16 * N * P / t / 1e6, 1)
            elif o.op == d.OP_SCALE_B and o.index == 0:
                t = timed(lambda: d.gpu_step(o, ctx), a.reps)
                out["scale_b_panel_ms"] = round(t, 4)
                out["scale_b_panel_gbs"] = round(16 * (o.hi - o.lo) * M / t / 1e6, 1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
