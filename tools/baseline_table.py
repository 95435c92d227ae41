"""Render BASELINE.md section 4's per-configuration table from a `tools/table_bench.py` JSONL
(device timings on one B200), an optional `tools/kernel_times.py` JSONL (kernel-only ncu times)
and `profiles/r01/oracle_timing.jsonl` (the CPU oracle on the GPU box's host), and splice it into
BASELINE.md in place of the current table.

    python tools/baseline_table.py profiles/r02/table_r02.jsonl [--kernels profiles/r02/kernel_times.jsonl] [--write]
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = ("| cfg | method | levels | GPUs | t median (ms) | kernel-only t (ms, ncu) | GFLOP/s (2NPM/t) | fraction of P64 "
          "| executed GFLOP/s (Strassen) | ‖C−N‖∞ / (‖A‖∞‖B‖∞), N = NaivKahan | ‖C−AB‖∞ / (‖A‖∞‖B‖∞), 2 rows | "
          "parity vs oracle | oracle t (1 core) | oracle t (16 cores) |")
NCOLS = 14
ORACLE_NAME = {"naive": "naive_standard", "kahan": "naive_kahan", "winograd": "winograd_original",
               "winograd_scaled": "winograd_scaled", "strassen": "strassen_paper_plan",
               "strassen_winograd": "strassen_winograd_paper_plan"}


def oracle_times(path):
    one, many = {}, {}
    for line in open(path):
        r = json.loads(line)
        if "config" not in r:
            continue
        key = (r["config"], r["method"])
        if "16 processes" in r["mode"]:
            many[key] = f"{r['seconds'] * 1e3:.0f} ms"
        elif "extrapolated_full_product_s" in r:
            one[key] = f"{r['extrapolated_full_product_s']:.0f} s (extrapolated from 512 entries)"
        else:
            one[key] = f"{r['seconds'] * 1e3:.1f} ms"
    return one, many


def kernel_times(path):
    out = {}
    if path:
        for line in open(path):
            r = json.loads(line)
            out[(r["config"], r["method"], r["levels"])] = r["kernel_ms"]
    return out


def rows(table_path, oracle_path, kernels_path=None):
    one, many = oracle_times(oracle_path)
    kt = kernel_times(kernels_path)
    out = []
    for line in open(table_path):
        r = json.loads(line)
        m, lv = r["method"], r["levels"]
        strassen = m.startswith("strassen")
        levels = "" if lv is None else ("paper plan" if lv == -1 else str(lv))
        executed = f"{r['gflops'] * (7 / 8) ** lv:.0f}" if strassen and lv is not None and lv >= 0 else ""
        parity = "bitwise vs or_*_fused (NEXT-3)" if m.endswith("_fused") else "bitwise"
        # oracle timings: the literal methods, and the paper plan for the Strassen rows
        okey = (r["config"], ORACLE_NAME.get(m, ""))
        show_oracle = (not strassen) or lv == -1
        t1 = one.get(okey, "") if show_oracle else ""
        t16 = many.get(okey, "") if show_oracle else ""
        k = kt.get((r["config"], m, lv))
        ks = f"{k:.4g}" if k is not None else ""
        ex = f"{r['rel_err_vs_exact']:.2e}" if "rel_err_vs_exact" in r else ""
        out.append(f"| {r['config']} | {m} | {levels} | 1 | {r['ms']:.4g} | {ks} | {r['gflops']:.0f} | "
                   f"{r['frac_fp64_peak']:.3f} | {executed} | {r['rel_err_vs_kahan']:.2e} | {ex} | {parity} | {t1} | "
                   f"{t16} |")
    return out


def main(argv):
    table = argv[0]
    kernels = argv[argv.index("--kernels") + 1] if "--kernels" in argv else None
    body = rows(table, os.path.join(ROOT, "profiles", "r01", "oracle_timing.jsonl"), kernels)
    text = "\n".join([HEADER, "|" + "---|" * NCOLS] + body)
    if "--write" not in argv:
        print(text)
        return
    path = os.path.join(ROOT, "BASELINE.md")
    s = open(path).read()
    start = s.index("| cfg | method | levels | GPUs |")
    end = s.find("\n\n", start)
    end = len(s) if end < 0 else end
    s = s[:start] + text + s[end:]
    s = re.sub(r"profiles/r0\d/table_\w+\.jsonl", os.path.relpath(table, ROOT), s)
    open(path, "w").write(s)
    print(f"BASELINE.md table regenerated from {table} ({len(body)} rows)")


if __name__ == "__main__":
    main(sys.argv[1:])
