"""CPU-oracle timings for BASELINE.md section 4 (BASELINE.md section 3's plan), on the host this
runs on (run it on the GPU box's host, where bench.py's cpu_baseline is measured).

  * single thread: full products for c1 (128^3, all methods) and c2 (1024^3, the classical,
    Kahan and Winograd families); sampled output entries for c3 / c4, reported as GFLOP/s =
    2 P samples / t and an extrapolated full-product time (labelled "extrapolated");
  * all cores: the same untouched per-entry oracle routine (bitwise the single-thread result)
    driven by a process pool over row blocks, for c2 NaivStandard.

Test infrastructure (it calls oracle/): never on the product path.
    python tools/oracle_timing.py > profiles/r01/oracle_timing.jsonl
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workload  # noqa: E402

FULL = {
    "naive_standard": lambda A, B: oracle.naive_standard(A, B),
    "naive_on_array": lambda A, B: oracle.naive_on_array(A, B),
    "naive_kahan": lambda A, B: oracle.naive_kahan(A, B),
    "unroll2": lambda A, B: oracle.naive_unroll(2, A, B),
    "unroll3": lambda A, B: oracle.naive_unroll(3, A, B),
    "unroll4": lambda A, B: oracle.naive_unroll(4, A, B),
    "winograd_original": lambda A, B: oracle.winograd_original(A, B),
    "winograd_scaled": lambda A, B: oracle.winograd_scaled(A, B)[0],
    "strassen_paper_plan": lambda A, B: oracle.strassen(0, A, B),
    "strassen_winograd_paper_plan": lambda A, B: oracle.strassen(1, A, B),
}


def emit(**kw):
    print(json.dumps(kw), flush=True)


def _rows(args):
    lo, hi, key = args
    A, B = workload.operands(key)
    idx = [(i, j) for i in range(lo, hi) for j in range(B.shape[1])]
    return lo, oracle.entries(oracle.M_STANDARD, A, B, idx).reshape(hi - lo, B.shape[1])


def main():
    cores = len(os.sched_getaffinity(0))
    emit(host_cpus=os.cpu_count(), affinity=cores)
    for key, names in (("c1", list(FULL)), ("c2", ["naive_standard", "naive_kahan", "winograd_original",
                                                   "winograd_scaled"])):
        A, B = workload.operands(key)
        N, P, M = A.shape[0], A.shape[1], B.shape[1]
        for name in names:
            t0 = time.perf_counter()
            FULL[name](A, B)
            t = time.perf_counter() - t0
            emit(config=key, method=name, mode="full product, 1 thread", seconds=round(t, 4),
                 gflops=round(2.0 * N * P * M / t / 1e9, 4))
    # all cores, c2 NaivStandard: row blocks of the per-entry routine in a process pool
    A, B = workload.operands("c2")
    ref = oracle.naive_standard(A, B)
    N = A.shape[0]
    blocks = [(i, min(N, i + 32), "c2") for i in range(0, N, 32)]
    with mp.get_context("fork").Pool(cores) as pool:
        t0 = time.perf_counter()
        parts = pool.map(_rows, blocks)
        t = time.perf_counter() - t0
    C = np.empty_like(ref)
    for lo, block in parts:
        C[lo:lo + block.shape[0]] = block
    emit(config="c2", method="naive_standard", mode=f"full product, {cores} processes (per-entry routine)",
         seconds=round(t, 4), gflops=round(2.0 * N ** 3 / t / 1e9, 4), bitwise_equal_single_thread=bool(
             np.array_equal(C, ref)))
    # sampled entries for the large configs
    for key in ("c3", "c4"):
        A, B = workload.operands(key)
        N, P, M = A.shape[0], A.shape[1], B.shape[1]
        idx = [tuple(map(int, x)) for x in workload.sample_positions(int(key[1]), N, M, 512, 77)]
        for name, m in (("naive_standard", oracle.M_STANDARD), ("naive_kahan", oracle.M_KAHAN),
                        ("winograd_original", oracle.M_WINOGRAD)):
            t0 = time.perf_counter()
            oracle.entries(m, A, B, idx)
            t = time.perf_counter() - t0
            g = 2.0 * P * len(idx) / t / 1e9
            emit(config=key, method=name, mode=f"{len(idx)} sampled entries, 1 thread", seconds=round(t, 4),
                 gflops=round(g, 4), extrapolated_full_product_s=round(2.0 * N * P * M / (g * 1e9), 1))


if __name__ == "__main__":
    main()
