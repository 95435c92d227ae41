"""Per-config, per-method device timings on one B200.

For each BASELINE.json config that fits one GPU (c1-c4) and each method: median of R timed
calls (CUDA events, inputs resident), GFLOP/s as 2NPM/t, fraction of the 37.22 TF FP64
peak, the error against NaivKahan on the device as ||C - N||_inf / (||A|| ||B||)
(the paper's stability column), and the error against the product itself on two
seeded rows -- sum_j |C_ij - (AB)_ij| / (||A|| ||B||), (AB)_ij by bench.exact_rows (Dot2, twice
double precision) -- Brent's E.  Writes JSON lines to stdout.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench  # noqa: E402  (exact_rows: the reference of the error column)
import paper_1106_1347_b200 as mm
import workload

PEAK = 37.22


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    methods = [("naive", None), ("kahan", None), ("winograd", None), ("winograd_scaled", None),
               ("strassen", 1), ("strassen", 2), ("strassen", 3), ("strassen_winograd", 1),
               ("strassen_winograd", 2), ("strassen_winograd", 3), ("strassen_winograd", -1),
               ("kahan_fused", None), ("winograd_fused", None), ("winograd_scaled_fused", None)]
    for key in a.configs.split(","):
        cfg = workload.CONFIGS[key]
        A_h, B_h = workload.operands(key)
        A = torch.from_numpy(A_h).cuda()
        B = torch.from_numpy(B_h).cuda()
        del A_h, B_h
        nA, nB = mm.norm_inf(A).item(), mm.norm_inf(B).item()
        rows = sorted({int(i) for i in workload.sample_positions(cfg.cfg_id, cfg.N, cfg.M, 2, shard=7)[:, 0]})
        X = torch.from_numpy(bench.exact_rows(A[rows].cpu().numpy(), B.cpu().numpy())).cuda()
        K = mm.kahan(A, B)
        C = torch.empty_like(K)
        for name, lv in methods:
            if lv == -1 and cfg.N > 2048:
                continue  # the paper's plan recurses to order-17 bases: only for small sizes
            f = getattr(mm, name)
            kw = {"levels": lv} if lv is not None else {}
            f(A, B, out=C, **kw)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                f(A, B, out=C, **kw)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            # back to back: R calls between one event pair (the host enqueue overlaps the GPU work)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                f(A, B, out=C, **kw)
            e1.record()
            torch.cuda.synchronize()
            ms_b2b = e0.elapsed_time(e1) / a.reps
            ms_graph = None
            if cfg.N <= 2048 and lv != -1:  # launch-bound sizes: replay the captured launch sequence
                gp = mm.GraphedProduct(name, A, B, out=C, **kw)
                gp.replay()
                e0.record()
                for _ in range(a.reps):
                    gp.replay()
                e1.record()
                torch.cuda.synchronize()
                ms_graph = round(e0.elapsed_time(e1) / a.reps, 4)
                del gp
            err = (C - K).abs().sum(dim=1).max().item() / (nA * nB) if name != "kahan" else 0.0
            err_x = (C[rows] - X).abs().sum(dim=1).max().item() / (nA * nB)
            g = 2.0 * cfg.N * cfg.P * cfg.M / ms / 1e6
            print(json.dumps({"config": key, "N": cfg.N, "P": cfg.P, "M": cfg.M, "method": name, "levels": lv,
                              "ms": round(ms, 4), "ms_back_to_back": round(ms_b2b, 4), "ms_graph": ms_graph,
                              "gflops": round(g, 1),
                              "frac_fp64_peak": round(g / 1e3 / PEAK, 4),
                              "rel_err_vs_kahan": err, "rel_err_vs_exact": err_x, "exact_rows": rows}),
                  flush=True)
        mm.release_workspace()
        del A, B, C, K
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
