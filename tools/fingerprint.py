"""Method fingerprints from SASS instruction counts (SURVEY.md 8(d) "ncu evidence"): proves each
kernel executes the paper's operation mix and is not a disguised GEMM.

    ncu --metrics <FP_METRICS> --csv --log-file fp.csv python tools/fingerprint.py run
    python tools/fingerprint.py summarize fp.csv > profiles/.../fingerprint.md

`run` multiplies 2048^3 operands once per method; `summarize` compares each launch's counters
with the counts the method's definition implies (n = 2048):
  K1 (DMMA.8x8x4 = 256 FMA per warp instruction): DMMA ~ n^3 / 256, DADD/DMUL/DFMA ~ 0
  K2 Kahan:        DMUL = n^3, DADD = 4 n^3 (dsub counted as DADD), DFMA = 0
  K2 Kahan fused (R22):        DFMA = n^3, DADD = 3 n^3
  K3 Winograd:     DMUL = n^2 n/2, DADD = 3 n^2 n/2 (+ 2 n^2 epilogue), DFMA = 0
  K3 Winograd fused (R22):     DFMA = n^2 n/2, DADD = 2 n^2 n/2 (+ 2 n^2)
  y/z line kernel:             DMUL = DADD = 2 n n/2 (or DFMA = 2 n n/2 fused)
  Strassen-Winograd leaves:    DMMA ~ (7/8)^d n^3 / 256 (d = 2 batched K1; d = 3 the fused combination
                               kernel, whose epilogue adds 0 DMUL / DFMA and a few DADD per output)
"""
import csv
import os
import sys

N = 2048
FP_METRICS = ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,"
              "sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum")


def run():
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    # the fused S-W combination (NEXT-1) at 2048^3, d = 3 (below its default size threshold)
    os.environ["MM_STRASSEN_FUSED_COMBINE"] = "1"
    import torch

    import paper_1106_1347_b200 as mm

    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(N, N, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(N, N, dtype=torch.float64, device="cuda", generator=g)
    for name in ("naive", "kahan", "kahan_fused", "winograd", "winograd_fused"):
        getattr(mm, name)(A, B)
    mm.strassen_winograd(A, B, levels=2)
    mm.strassen_winograd(A, B, levels=3)  # leaves in the fused combination kernel: (7/8)^3 of the DMMAs
    torch.cuda.synchronize()


def _fused(kernel: str) -> bool:
    """The FUSED template argument: the one after CV in <SimtCfg<...>, CV, FUSED[, EX]>."""
    tail = kernel[kernel.index(">") + 1:].strip(" ,>")
    args = [t.strip() for t in tail.split(",") if t.strip()]
    return len(args) >= 2 and args[1] in ("1", "true")


def expected(kernel: str):
    n3, n2 = N ** 3, N ** 2
    half = n3 // 2
    if kernel.startswith("dgemm"):
        return None  # batched Strassen leaves share the kernel; see the DMMA ratio column
    if kernel.startswith(("kahan_gemm_kernel", "kahan_tma_kernel")) and _fused(kernel):
        return {"dadd": 3 * n3, "dmul": 0, "dfma": n3, "dmma": 0}
    if kernel.startswith(("kahan_gemm_kernel", "kahan_tma_kernel")):
        return {"dadd": 4 * n3, "dmul": n3, "dfma": 0, "dmma": 0}
    if kernel.startswith("winograd_tma_kernel") and _fused(kernel):
        return {"dadd": 2 * half + 2 * n2, "dmul": 0, "dfma": half, "dmma": 0}
    if kernel.startswith("winograd_tma_kernel"):
        return {"dadd": 3 * half + 2 * n2, "dmul": half, "dfma": 0, "dmma": 0}
    if kernel.startswith("line_kernel<2, 0>"):
        return {"dadd": 0, "dmul": 0, "dfma": n2, "dmma": 0}
    if kernel.startswith("line_kernel<1, 0>"):
        return {"dadd": n2, "dmul": n2, "dfma": 0, "dmma": 0}
    return None


def summarize(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    per = {}
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mmk::", "")
        if name.startswith("at::"):
            continue  # torch's input generator
        key = (int(d["ID"]), name, d["Grid Size"])
        m = d["Metric Name"]
        short = "dmma" if "dmma" in m else m.split("_op_")[1].split("_")[0]
        per.setdefault(key, {})[short] = float(d["Metric Value"].replace(",", ""))
    print(f"# SASS fingerprints at n = {N} (ncu instruction counters; expected from the method's definition)\n")
    print("| id | kernel | grid | DADD | DMUL | DFMA | DMMA (warp inst) | expected DADD / DMUL / DFMA | DMMA x 256 / n^3 |")
    print("|---|---|---|---|---|---|---|---|---|")
    for (i, k, g), v in sorted(per.items()):
        e = expected(k)
        es = "" if e is None else f"{e['dadd']:.4g} / {e['dmul']:.4g} / {e['dfma']:.4g}"
        ratio = f"{v.get('dmma', 0) * 256 / N ** 3:.4f}" if v.get("dmma", 0) else ""
        print(f"| {i} | {k} | {g} | {v.get('dadd', 0):.4g} | {v.get('dmul', 0):.4g} | {v.get('dfma', 0):.4g} | "
              f"{v.get('dmma', 0):.4g} | {es} | {ratio} |")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    elif sys.argv[1] == "metrics":
        print(FP_METRICS)
    else:
        summarize(sys.argv[2])
