"""The paper's section-3 experiment on B200 -- SURVEY.md 8(f) NEXT-2.

Protocol: A is an n x n random matrix (U[0,1), reading R13), B = 8A
(MultiplyWithScalar), N := NaivKahan(A, B) is the reference; every method runs
-R times and the table reports its time and NormInf(N - C).  Here every product runs on the GPU
through the C ABI; the unrolled / on-array variants are the DMMA kernel (reading R18), Strassen
runs both the paper's padding plan (levels = -1) and the GPU plan (explicit levels).
Times are per product (reading R14): the median of R CUDA-event-timed calls after one warm-up.
The paper's printed values (tests/golden/paper_table.txt, a text fixture) are shown beside ours
as context; its machine is unknown and its code unoptimised.

    python tools/paper_experiment.py [--sizes 200,800] [--repeats 10] [--json out.jsonl]
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
import workload  # noqa: E402

# (row label as printed in the paper, library call, kwargs)
ROWS = [
    ("NaivStandard", "naive", {}),
    ("NaivOnArray", "naive_on_array", {}),
    ("NaivLoopUnrollingTwo", "unroll2", {}),
    ("NaivLoopUnrollingThree", "unroll3", {}),
    ("NaivLoopUnrollingFour", "unroll4", {}),
    ("StrassenNaiv", "strassen", {"levels": -1}),
    ("StrassenWinograd", "strassen_winograd", {"levels": -1}),
    ("WinogradOriginal", "winograd", {}),
    ("WinogradScaled", "winograd_scaled", {}),
]
EXTRA = [
    ("StrassenNaiv (GPU plan, 2 levels)", "strassen", {"levels": 2}),
    ("StrassenWinograd (GPU plan, 2 levels)", "strassen_winograd", {"levels": 2}),
    # the fused-FMA variants (not the paper's methods; reading R22)
    ("NaivKahan (fused FMA)", "kahan_fused", {}),
    ("WinogradOriginal (fused FMA)", "winograd_fused", {}),
    ("WinogradScaled (fused FMA)", "winograd_scaled_fused", {}),
]


def printed_values(fname):
    out = {}
    path = os.path.join(ROOT, "tests", "golden", fname)
    with open(path) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            n, name, val, ln = line.split()
            out[(int(n), name)] = (float(val), int(ln))
    return out


def time_call(fn, repeats):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(ts)


def run(n, repeats, seed=42):
    A_h, B_h = workload.paper_protocol(n, seed)
    A = torch.from_numpy(A_h).cuda()
    B = torch.from_numpy(B_h).cuda()
    out = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ref = mm.kahan(A, B)  # N := NaivKahan
    t_ref = time_call(lambda: mm.kahan(A, B, out=out), repeats)
    res = [{"n": n, "method": "NaivKahan", "seconds": t_ref, "deviation": None}]
    for label, fn_name, kw in ROWS + EXTRA:
        f = getattr(mm, fn_name)
        if kw.get("levels") == -1 and n.bit_length() - 5 > 7:
            continue  # the paper's plan recurses k = floor(log2 n) - 4 levels to 7^k bases of order
            # 17..32: beyond k = 7 (n >= 4096) its arena and launch grid are impractical
        C = f(A, B, **kw)
        dev = float(mm.norm_inf(ref - C).item())  # NormInf(Minus(N, C))
        t = time_call(lambda: f(A, B, out=out, **kw), repeats)
        res.append({"n": n, "method": label, "seconds": t, "deviation": dev})
    mm.release_workspace()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="200,400,800,1600,3200")
    ap.add_argument("--repeats", type=int, default=10)  # the paper's -R default
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    printed = printed_values("paper_table.txt")
    ptimes = printed_values("paper_times.txt")
    lines = []
    for n in map(int, a.sizes.split(",")):
        rows = run(n, a.repeats)
        lines += rows
        print(f"\n-O {n} -R {a.repeats}   (B200, FP64; paper values: PAPER.md section 3, unknown CPU, -O0)")
        print(f"{'method':42s} {'time (s)':>12s} {'NormInf(N-C)':>14s} {'paper time':>11s} {'paper dev':>13s}")
        for r in rows:
            p, pt = printed.get((n, r["method"])), ptimes.get((n, r["method"]))
            pdev = f"{p[0]:.10f}" if p else ""
            ptim = f"{pt[0]:.6f}" if pt else ""
            dev = "" if r["deviation"] is None else f"{r['deviation']:.10f}"
            print(f"{r['method']:42s} {r['seconds']:12.6f} {dev:>14s} {ptim:>11s} {pdev:>13s}")
    if a.json:
        with open(a.json, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
