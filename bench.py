#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the B200 FP64 matmul library.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference] [--config c4]

One STEP = one pass of the whole hot path over the workload: every
method of the C ABI -- mm_naive, mm_kahan, mm_winograd, mm_winograd_scaled (which includes
norm_inf and lambda), mm_strassen and mm_strassen_winograd -- once each on the same
synthetic A, B.  Metric (BASELINE.json): FP64 GFLOP/s counted as 2NPM per method call, so
`value` = 6 * 2NPM / (time per step).  Per-method GFLOP/s and fractions of the FP64 peak are
in "methods".

N > 1 (torchrun, one process per GPU, NCCL): C is split by row blocks of A and B is broadcast
from rank 0 inside every product, following the library's multi-GPU schedule (mm_dist_schedule:
B in row panels that the product consumes as they land) executed over torch.distributed
(paper_1106_1347_b200.dist.dist_gemm -- the executor the two-rank CPU tests drive) or, with
--dist-impl native, by the library's own NCCL layer (mm_dist_gemm).  The global problem is fixed,
so scaling is "strong"; ms_per_step is the max over ranks.

BASELINE.json's scaling config (c5, 32768^3, classical + Strassen-Winograd at 1/2/4/8 GPUs):
    python bench.py --config c5 --methods naive,strassen_winograd --levels 2 [--gpus N]

--impl reference times the CPU oracle (oracle/, the plain C99 implementation the parity tests
use) on a bounded sample of entries of the same workload: this task has no runnable
reference implementation (/root/reference holds only the paper), so the oracle is the
reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METHODS = ("naive", "kahan", "winograd", "winograd_scaled", "strassen", "strassen_winograd")
METRIC = "FP64 GFLOP/s (2NPM/t) per method vs FP64 peak at 1/2/4/8 B200; ‖E‖∞ rel err"

# FP64 peaks on B200: MEASURED_PEAKS.json has no FP64 entry, so the
# denominators are derived from the unit counts and the max SM clock (MEASURED_PEAKS.json
# sm_max_mhz = 1965; FP64 load holds that clock, profiles/r01_probe/clocks.csv):
#   DMMA / DFMA: 148 SMs x 64 FMA/clk x 2 flop = 37.22 TFLOP/s (probe P2 measured DMMA 37.0)
#   DADD / DMUL (one flop per lane-op):          18.61 TFLOP/s (probe P2 DFMA issue: 17.0 T op/s)
SMS = 148


def fp64_peaks(sm_mhz: float = 1965.0):
    f = SMS * 64 * sm_mhz * 1e6
    return {"dmma_tflops": 2 * f / 1e12, "simt_op_tflops": f / 1e12}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("mine", "reference"), default="mine")
    ap.add_argument("--config", default="c4")
    ap.add_argument("--levels", type=int, default=3, help="Strassen recursion levels (c4: 3 levels, 1024^3 leaves, is fastest: profiles/r01/table_v2.jsonl)")
    ap.add_argument("--methods", default=",".join(METHODS))
    ap.add_argument("--panels", type=int, default=8,
                    help="N>1: B broadcast in this many row panels overlapped with NaivStandard's accumulation "
                         "(the other methods: half as many; their per-panel cost is higher, "
                         "profiles/r01/panel_bench.jsonl)")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"),
                    help="N > 1 collectives (gloo only to exercise the multi-rank path on fewer GPUs)")
    ap.add_argument("--dist-impl", default="torch", choices=("torch", "native"),
                    help="N > 1 executor of the schedule: torch.distributed (dist.dist_gemm) or the library's "
                         "own NCCL layer (mm_dist_gemm)")
    ap.add_argument("--err-rows", type=int, default=2,
                    help="rows of C checked against the exactly rounded product (abs_err column); 0 = off")
    ap.add_argument("--e2e-blocks", type=int, default=8,
                    help="e2e: k-panels / row blocks the host<->device copies are pipelined in")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline sample")
    return ap.parse_args()


# ---------------------------------------------------------------------------- helpers
def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, pw, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


def load_traffic():
    p = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------- CPU oracle legs
def oracle_sample(cfg, A, B, levels, budget_s: float, methods, lam=None, counts=None):
    """Time the oracle's per-entry functions on seeded sample entries of the workload.
    Returns (flops, seconds, counts): flops counted like the GPU metric, 2P per entry."""
    import numpy as np

    import oracle
    import workload

    N, P, M = A.shape[0], A.shape[1], B.shape[1]
    if lam is None and "winograd_scaled" in methods:
        lam = oracle.lam(oracle.norm_inf(A), oracle.norm_inf(B))
    d, (Np, Pp, Mp) = oracle.plan(N, P, M, levels)
    pos = workload.sample_positions(cfg.cfg_id, N, M, 200000, shard=42)
    total_t, total_f, used = 0.0, 0.0, {}
    per_method = budget_s / len(methods)
    for m in methods:
        target = None if counts is None else counts[m]
        n_done, t_m, i0 = 0, 0.0, 0
        chunk = 64
        while True:
            sel = np.arange(i0, i0 + chunk) % len(pos)  # cycle through the seeded positions
            idx = pos[sel]
            i0 += chunk
            t0 = time.perf_counter()
            if m in ("strassen", "strassen_winograd"):
                oracle.entries_strassen(0 if m == "strassen" else 1, A, B, idx, levels=d, pad=(Np, Pp, Mp),
                                        base=oracle.BASE_FMA)
            else:
                code = {"naive": oracle.M_FMA, "kahan": oracle.M_KAHAN, "winograd": oracle.M_WINOGRAD,
                        "winograd_scaled": oracle.M_WINOGRAD_SCALED}[m]
                oracle.entries(code, A, B, idx, lam or 0)
            t_m += time.perf_counter() - t0
            n_done += len(idx)
            if target is not None:
                if n_done >= target:
                    break
            elif t_m >= per_method:
                break
        used[m] = n_done
        total_t += t_m
        total_f += 2.0 * P * n_done
    return total_f, total_t, used


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import workload

    cfg = workload.CONFIGS[args.config]
    methods = tuple(args.methods.split(","))
    A, B = workload.operands(args.config, 0)
    # calibrate the per-step sample so the whole run stays within a few minutes
    _, t_cal, used = oracle_sample(cfg, A, B, args.levels, 1.2, methods)
    per_step_budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    counts = {m: max(16, int(used[m] * per_step_budget / max(t_cal, 1e-3))) for m in methods}
    for _ in range(args.warmup):
        oracle_sample(cfg, A, B, args.levels, 0, methods, counts={m: 16 for m in methods})
    flops = secs = 0.0
    for _ in range(args.steps):
        f, t, used = oracle_sample(cfg, A, B, args.levels, 0, methods, counts=counts)
        flops += f
        secs += t
    v = flops / secs / 1e9
    sample = (f"{sum(used.values())} seeded entries per step of {args.config} ({', '.join(f'{m}:{used[m]}' for m in methods)}),"
              f" single-thread C99 oracle per-entry functions")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(secs / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, cfg, world),
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def panels_for_method(args, m):
    return args.panels if m == "naive" else max(1, args.panels // 2)


def exact_rows(A_rows, B):
    """Rows of the product AB to about twice double precision, as the reference of the
    error column: Ogita-Rump-Oishi Dot2 -- every product split exactly into p + e (Dekker's
    TwoProduct, 2^27 + 1 splitting), the p summed with TwoSum and every rounding error and e carried
    in a second accumulator -- vectorised over the columns.  Its error is below u |(AB)_ij| +
    (P u)^2 sum_k |A_ik B_kj| (u = 2^-53), orders of magnitude under any method's, so this stands
    for the exact product of Brent's ||E||.  Diagnostic, outside the timed
    region."""
    import numpy as np

    split = 134217729.0

    def halves(x):
        t = split * x
        hi = t - (t - x)
        return hi, x - hi

    bh, bl = halves(B)
    out = np.empty((A_rows.shape[0], B.shape[1]))
    for r in range(A_rows.shape[0]):
        s = np.zeros(B.shape[1])
        c = np.zeros(B.shape[1])
        for k in range(B.shape[0]):
            a = float(A_rows[r, k])
            p = a * B[k]
            ah, al = halves(a)
            e = ((ah * bh[k] - p) + ah * bl[k] + al * bh[k]) + al * bl[k]  # a B[k] = p + e exactly
            t = s + p
            z = t - s
            c += ((s - (t - z)) + (p - z)) + e  # TwoSum error of s + p, plus e
            s = t
        out[r] = s + c
    return out


def config_dict(args, cfg, world):
    return {
        "workload": f"{cfg.key}: A {cfg.N}x{cfg.P}, B {cfg.P}x{cfg.M} float64 ({cfg.dist}), one call of each of "
                    f"{args.methods.replace(',', ', ')} per step",
        "N": cfg.N, "P": cfg.P, "M": cfg.M, "strassen_levels": args.levels,
        "parallelism": (f"row-block dp{world} (B broadcast via {args.dist_backend}, schedule executed by "
                        f"{'mm_dist_gemm' if args.dist_impl == 'native' else 'dist.dist_gemm'}; row panels "
                        f"overlapped: naive {args.panels}, others {max(1, args.panels // 2)})"
                        if world > 1 else "1 GPU"),
        "l2": (f"inputs larger than L2 (A, B, C = {8 * cfg.N * cfg.P / 1e6:.0f} MB each vs 126 MB L2)"
               if cfg.N >= 4096 else "inputs smaller than L2 (not flushed)"),
    }


# ---------------------------------------------------------------------------- GPU arm
def run_mine(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1106_1347_b200 as mm
    import workload
    from paper_1106_1347_b200 import dist as mmdist

    rank, world, local = env_rank()
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # host-staged collectives: lets the N > 1 code path run with several ranks on one GPU (tests)
            dist.init_process_group(args.dist_backend)
    cfg = workload.CONFIGS[args.config]
    methods = tuple(args.methods.split(","))
    N, P, M = cfg.N, cfg.P, cfg.M
    lo, hi = workload.shard_rows(N, world, rank)
    n_loc = hi - lo

    A_h = workload.matrix(cfg, 0, 0, lo, hi)
    B_h = workload.matrix(cfg, 1, 0) if rank == 0 else np.zeros((P, M))
    A = torch.from_numpy(A_h).to(dev)
    B = torch.from_numpy(B_h).to(dev)
    outs = {m: torch.empty((n_loc, M), dtype=torch.float64, device=dev) for m in methods}
    stream = torch.cuda.current_stream(dev)

    # N > 1: the library's schedule, executed over torch.distributed (default) or by the library's
    # own NCCL layer (--dist-impl native)
    native = mmdist.NativeComm() if world > 1 and args.dist_impl == "native" and args.dist_backend == "nccl" else None

    def panels_for(m):
        return panels_for_method(args, m)

    def one_method(m):
        if native is not None:
            return native.gemm(m, A, B, out=outs[m], levels=args.levels, panels=panels_for(m))
        if world > 1:
            return mmdist.dist_gemm(m, A, B, out=outs[m], levels=args.levels, panels=panels_for(m))
        if m == "winograd_scaled":
            return mm.winograd_scaled(A, B, out=outs[m])
        if m in ("strassen", "strassen_winograd"):
            return getattr(mm, m)(A, B, out=outs[m], levels=args.levels)
        return getattr(mm, m)(A, B, out=outs[m])

    def step(ev=None):
        for m in methods:
            if ev is not None:
                ev[m][0].record(stream)
            one_method(m)
            if ev is not None:
                ev[m][1].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    gpu_uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    sampler = ClockSampler(gpu_uuid)
    evs = [{m: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for m in methods}
           for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    n0 = mm.launch_count()
    t0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = mm.launch_count() - n0
    clocks = sampler.stop()
    ms = t0.elapsed_time(t1) / args.steps
    per_m = {m: statistics.mean(e[m][0].elapsed_time(e[m][1]) for e in evs) for m in methods}
    if world > 1:
        t = torch.tensor([ms] + [per_m[m] for m in methods], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        per_m = {m: float(t[i + 1]) for i, m in enumerate(methods)}

    flop = 2.0 * N * P * M
    value = flop * len(methods) / (ms / 1e3) / 1e9
    peaks = fp64_peaks()

    # per-method results; error of each method against NaivKahan (the paper's "N")
    # as ||N - C||_inf / (||A|| ||B||) on this rank's rows (diagnostic, outside the timed region)
    ref = outs.get("kahan")
    nA = float(mm.norm_inf(A).item()) if n_loc else 0.0
    nB = float(mm.norm_inf(B).item())
    if world > 1:
        tt = torch.tensor([nA], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nA = float(tt[0])
    res = {}
    for m in methods:
        g = flop / (per_m[m] / 1e3) / 1e9
        entry = {"ms": round(per_m[m], 3), "gflops": round(g, 1), "frac_fp64_peak": round(g / 1e3 / peaks["dmma_tflops"], 4)}
        if ref is not None and m != "kahan" and n_loc:
            e = float((outs[m] - ref).abs().sum(dim=1).max().item())
            if world > 1:
                tt = torch.tensor([e], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                e = float(tt[0])
            entry["rel_err_vs_kahan"] = e / (nA * nB) if nA * nB > 0 else 0.0
        res[m] = entry

    # ||E||_inf against the exactly rounded product on a few seeded rows of this rank's shard
    # (Brent's E), as sum_j |C_ij - (AB)_ij| / (||A|| ||B||)
    if args.err_rows > 0 and rank == 0 and n_loc > 0:
        rows = sorted({int(i) for i in workload.sample_positions(cfg.cfg_id, n_loc, M, 64, shard=7)[:, 0]})
        rows = rows[:args.err_rows]
        cols = np.arange(M) if M <= 8192 else np.sort(workload.sample_positions(cfg.cfg_id, 1, M, 4096, 8)[:, 1])
        X = exact_rows(A_h[rows], B_h[:, cols])
        ii = torch.tensor(rows, device=dev)
        jj = torch.from_numpy(cols).to(dev)
        for m in methods:
            Cm = outs[m][ii][:, jj].cpu().numpy()
            res[m]["rel_err_vs_exact"] = float(np.abs(Cm - X).sum(axis=1).max()) / (nA * nB) if nA * nB > 0 else 0.0
        err_note = (f"rows {rows} of rank 0's shard, {'all' if M <= 8192 else len(cols)} columns, "
                    f"against the product to twice double precision (Dot2: TwoProduct + TwoSum)")
    else:
        err_note = None

    # roofline of the dominant kernel (largest share of the step)
    # (the DRAM bytes per launch were captured at c4's full size: reported for that workload only)
    traffic = load_traffic() if (args.config == "c4" and world == 1) else {}
    n_eff = n_loc
    kernels = {
        "naive": ("tensor", 2.0 * n_eff * P * M, peaks["dmma_tflops"], "dgemm_tma_kernel"),
        "kahan": ("alu", 5.0 * n_eff * P * M, peaks["simt_op_tflops"],
                  "kahan_tma_kernel" if P % 2 == 0 and M % 2 == 0 else "kahan_gemm_kernel"),
        "winograd": ("alu", 4.0 * n_eff * M * (P // 2), peaks["simt_op_tflops"],
                     "winograd_tma_kernel" if P % 2 == 0 and M % 2 == 0 else "winograd_kernel"),
    }
    roof_all = {}
    for m, (bound, fl, pk, kname) in kernels.items():
        if m in per_m:
            ach = fl / (per_m[m] / 1e3) / 1e12
            roof_all[m] = {"bound": bound, "achieved": round(ach, 3), "peak": round(pk, 3), "unit": "TFLOP/s",
                           "frac": round(ach / pk, 4), "traffic": traffic.get(kname), "kernel": kname}
    dom = max(per_m, key=per_m.get)
    roofline = dict(roof_all.get(dom) or {"bound": "mixed", "achieved": None, "peak": None, "unit": "TFLOP/s",
                                          "frac": None, "traffic": None, "kernel": dom})
    roofline["share_of_step"] = round(per_m[dom] / ms, 4)
    roofline["peak_source"] = ("derived: 148 SMs x 64 FP64 lanes x 1.965 GHz (MEASURED_PEAKS.json has no FP64 "
                               "entry; probes measured DMMA 37.0 TF and DADD 18.48 / DMUL 18.44 T op/s, "
                               "profiles/r01_probe)")

    # ---- e2e: the user-level call on pinned host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, methods, A_h, B_h if rank == 0 else None, dev, world, rank, n_loc, P, M, native)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64, workload/)",
        "config": config_dict(args, cfg, world), "methods": res, "roofline": roofline,
        "roofline_by_kernel": roof_all, "gpu_launches": int(launches), "clocks": clocks, "e2e": e2e,
    }
    if err_note:
        line["err_sample"] = err_note
    if rank == 0 and world == 1 and not args.no_cpu:
        f, t, used = oracle_sample(cfg, A_h, B_h, args.levels, args.cpu_seconds, methods)
        line["cpu_baseline"] = {
            "value": round(f / t / 1e9, 4), "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
            "sample": f"{sum(used.values())} seeded entries of {cfg.key} ({', '.join(f'{m}:{used[m]}' for m in methods)}) "
                      f"through the oracle's per-entry functions, single thread, {t:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if native is not None:
        native.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, methods, A_h, B_h, dev, world, rank, n_loc, P, M, native=None):
    import torch
    import torch.distributed as dist

    import paper_1106_1347_b200 as mm
    from paper_1106_1347_b200 import dist as mmdist

    hA = torch.from_numpy(A_h).pin_memory()
    hB = torch.from_numpy(B_h).pin_memory() if B_h is not None else None
    hC = torch.empty((n_loc, M), dtype=torch.float64).pin_memory()
    stream = torch.cuda.current_stream(dev)
    dB = torch.empty((P, M), dtype=torch.float64, device=dev)

    # world 1: the paper's test-program call -- every method on the same host
    # operands: H2D A, B once per step, each product D2H'd while the next computes.  The order puts
    # a row-local method first (its row blocks start as A lands) and one last (its C streams back
    # by row blocks); the per-step work is the same six products as the device-timed step.
    order = sorted(methods, key=lambda m: {"naive": 0, "kahan": 9}.get(m, 5))
    houts = None
    if world == 1:
        # one pinned host C per method; above 16 GB of them (c5) the methods share one (the copies are
        # ordered on one copy stream, so each product still crosses PCIe in full every step)
        if 8.0 * n_loc * M * len(methods) <= 16e9:
            houts = {m: torch.empty((n_loc, M), dtype=torch.float64).pin_memory() for m in methods}
        else:
            shared = torch.empty((n_loc, M), dtype=torch.float64).pin_memory()
            houts = {m: shared for m in methods}

    def step():
        if world == 1:
            mm.matmul_methods(hA, hB, order, levels=args.levels, outs=houts, row_blocks=args.e2e_blocks)
            return
        # N > 1: each rank's rows of A (and B on the root) copied once per step; every product
        # broadcasts B inside dist_gemm and its C rows come back to the host
        dA = hA.to(dev, non_blocking=True)
        if rank == 0:
            dB.copy_(hB, non_blocking=True)
        for m in methods:
            pn = panels_for_method(args, m)
            if native is not None:
                C = native.gemm(m, dA, dB, levels=args.levels, panels=pn)
            else:
                C = mmdist.dist_gemm(m, dA, dB, levels=args.levels, panels=pn)
            hC.copy_(C, non_blocking=True)
        stream.synchronize()

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(1, args.steps)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0])
    from workload import CONFIGS

    cfgN = CONFIGS[args.config].N
    flop = 2.0 * cfgN * P * M * len(methods)
    h2d = 8 * (n_loc * P + (P * M if rank == 0 else 0))  # A (this rank's rows) and B (root) once per step
    d2h = len(methods) * 8 * n_loc * M
    return {"value": round(flop / (ms / 1e3) / 1e9, 1), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3), "steps": steps,
            "path": "C ABI mm_methods_host (via paper_1106_1347_b200.matmul_methods) on pinned host buffers: per step "
                    "H2D of A and B once, in k-panels that NaivStandard consumes as they land; every method's C D2H, "
                    "overlapped with the next method"
            if world == 1 else "dist_gemm: per step H2D of each rank's A rows (+ B on the root) once, every method's "
                               "C rows D2H"}


def main():
    args = parse_args()
    rank, world, _ = env_rank()
    if args.gpus > 1 and world == 1 and "WORLD_SIZE" not in os.environ:
        # convenience: relaunch under torchrun
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", "29533", *sys.argv]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_mine(args)


if __name__ == "__main__":
    sys.exit(main())
