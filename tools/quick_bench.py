"""Quick per-method device timing (development aid; bench.py is the contract)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1106_1347_b200 as mm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs=3, default=[8192, 8192, 8192])
    ap.add_argument("--methods", default="naive,kahan,winograd,winograd_scaled,strassen,strassen_winograd,kahan_fused,winograd_fused")
    ap.add_argument("--levels", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    N, P, M = a.n
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(N, P, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(P, M, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(N, M, dtype=torch.float64, device="cuda")
    for name in a.methods.split(","):
        f = getattr(mm, name)
        kw = {"levels": a.levels} if name.startswith("strassen") else {}
        f(A, B, out=C, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            f(A, B, out=C, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(json.dumps({"method": name, "shape": [N, P, M], "ms": round(ms, 3),
                          "gflops": round(2.0 * N * P * M / ms / 1e6, 1), **kw}), flush=True)


if __name__ == "__main__":
    main()
