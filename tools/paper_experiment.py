"""The paper's section-3 experiment on B200 -- SURVEY.md 8(f) NEXT-2.

Protocol: A is an n x n random matrix (U[0,1), reading R13), B = 8A
(MultiplyWithScalar), N := NaivKahan(A, B) is the reference; every method runs
-R times and the table reports its time and NormInf(N - C).  Here every product runs on the GPU
through the C ABI; the unrolled / on-array variants are the DMMA kernel (reading R18: their rows
are marked as aliases), Strassen runs the paper's padding plan (levels = -1) and, with
--extra, the GPU plan (explicit levels) and the NEXT-3 fused variants.  Times are per product
(reading R14): the mean of R CUDA-event-timed calls after one warm-up; the deviation is from the
last call.  With the table format the paper's printed values (tests/golden/paper_table.txt,
paper_times.txt) are shown beside ours as context; its machine is unknown and its code
unoptimised.

    python tools/paper_experiment.py [-O 400] [-R 10] [--seed 42] [--methods NaivStandard,...]
                                     [--format table|csv|json] [--sizes 200,800] [--extra]

-O / -R default to the paper's standards (400, 10); --sizes runs several orders.
CSV: header `method,seconds,deviation` (empty deviation for the reference row); JSON: {order,
repeats, seed, results: [{method, seconds, deviation|null}], aliases}.  Bad arguments exit with a
usage message and status 2.
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


PAPER_NAMES = ["NaivKahan"] + [r[0] for r in ROWS]
ALIASES = {"NaivOnArray": "NaivStandard", "NaivLoopUnrollingTwo": "NaivStandard",
           "NaivLoopUnrollingThree": "NaivStandard", "NaivLoopUnrollingFour": "NaivStandard"}


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
    return statistics.mean(ts)


def run(n, repeats, seed=42, methods=None, extra=False):
    A_h, B_h = workload.paper_protocol(n, seed)
    A = torch.from_numpy(A_h).cuda()
    B = torch.from_numpy(B_h).cuda()
    out = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ref = mm.kahan(A, B)  # N := NaivKahan, always run first as the reference
    t_ref = time_call(lambda: mm.kahan(A, B, out=out), repeats)
    res = [{"n": n, "method": "NaivKahan", "seconds": t_ref, "deviation": None}]
    for label, fn_name, kw in ROWS + (EXTRA if extra else []):
        if methods is not None and label not in methods:
            continue
        f = getattr(mm, fn_name)
        if kw.get("levels") == -1 and n.bit_length() - 5 > 7:
            continue  # the paper's plan recurses k = floor(log2 n) - 4 levels to 7^k bases of order
            # 17..32: beyond k = 7 (n >= 4096) its arena and launch grid are impractical
        t = time_call(lambda: f(A, B, out=out, **kw), repeats)
        dev = float(mm.norm_inf(ref - out).item())  # NormInf(Minus(N, C)) of the last call
        res.append({"n": n, "method": label, "seconds": t, "deviation": dev})
    mm.release_workspace()
    return res


def render_table(rows, n, repeats, printed, ptimes):
    lines = [f"TIME TEST FOR METHODS OF MATRIX MULTIPLICATION: C = A*(8A), where A is a random {n} x {n} matrix",
             f"-O {n} -R {repeats}   (B200, FP64; paper values: PAPER.md section 3, unknown CPU, -O0)",
             f"{'method':42s} {'time (sec)':>12s} {'NormInf( N-C )':>14s} {'paper time':>11s} {'paper dev':>13s}"]
    for r in rows:
        p, pt = printed.get((n, r["method"])), ptimes.get((n, r["method"]))
        pdev = f"{p[0]:.10f}" if p else ""
        ptim = f"{pt[0]:.6f}" if pt else ""
        dev = "" if r["deviation"] is None else f"{r['deviation']:.10f}"
        name = "N := NaivKahan" if r["method"] == "NaivKahan" else r["method"]
        if r["method"] in ALIASES:
            name += " *"
        lines.append(f"{name:42s} {r['seconds']:12.6f} {dev:>14s} {ptim:>11s} {pdev:>13s}")
    lines.append("* the same DMMA kernel as NaivStandard on the GPU (DESIGN.md reading R18); the oracle implements "
                 "each loop shape literally")
    return "\n".join(lines)


def render_csv(rows):
    out = ["method,seconds,deviation"]
    for r in rows:
        out.append(f"{r['method']},{r['seconds']!r},{'' if r['deviation'] is None else repr(r['deviation'])}")
    return "\n".join(out)


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description="PAPER.md section 3 on B200: time and NormInf(N - C) per method")
    ap.add_argument("-O", dest="order", type=int, default=400, help="matrix size n (paper standard: 400)")
    ap.add_argument("-R", dest="repeats", type=int, default=10, help="repeats (paper standard: 10); mean time")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--methods", default=None, help="comma-separated paper method names (default: all)")
    ap.add_argument("--format", choices=("table", "csv", "json"), default="table")
    ap.add_argument("--sizes", default=None, help="several orders, e.g. 200,400,800 (overrides -O)")
    ap.add_argument("--extra", action="store_true", help="also the GPU Strassen plan and the fused variants")
    ap.add_argument("--json", default=None, help="also write every row as JSON lines to this file")
    a = ap.parse_args(argv)
    if a.order < 1 or a.repeats < 1:
        ap.error("-O and -R must be positive")
    if a.methods is not None:
        a.methods = [x for x in a.methods.split(",") if x]
        bad = [x for x in a.methods if x not in PAPER_NAMES]
        if bad or not a.methods:
            ap.error(f"unknown method(s) {bad}; valid: {', '.join(PAPER_NAMES)}")
    try:
        a.sizes = [int(x) for x in a.sizes.split(",")] if a.sizes else [a.order]
    except ValueError:
        ap.error("--sizes takes comma-separated positive integers")
    if any(n < 1 for n in a.sizes):
        ap.error("sizes must be positive")
    return a


def main(argv=None):
    a = parse_args(argv)
    printed = printed_values("paper_table.txt")
    ptimes = printed_values("paper_times.txt")
    lines = []
    for n in a.sizes:
        rows = run(n, a.repeats, a.seed, a.methods, a.extra)
        lines += rows
        if a.format == "table":
            print(render_table(rows, n, a.repeats, printed, ptimes) + "\n")
        elif a.format == "csv":
            print(render_csv(rows))
        else:
            print(json.dumps({"order": n, "repeats": a.repeats, "seed": a.seed,
                              "results": [{k: r[k] for k in ("method", "seconds", "deviation")} for r in rows],
                              "aliases": {k: v for k, v in ALIASES.items() if any(r["method"] == k for r in rows)}}))
    if a.json:
        with open(a.json, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
