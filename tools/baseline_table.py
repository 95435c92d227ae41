"""Render BASELINE.md section 4's per-configuration table from a `tools/table_bench.py` JSONL
(device timings on one B200) and `profiles/r01/oracle_timing.jsonl` (the CPU oracle on the GPU
box's host), and splice it into BASELINE.md in place of the current table.

    python tools/baseline_table.py profiles/r01/table_v9.jsonl [--write]
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = ("| cfg | method | levels | GPUs | t median (ms) | GFLOP/s (2NPM/t) | fraction of P64 | executed GFLOP/s "
          "(Strassen) | ‖C−N‖∞ / (‖A‖∞‖B‖∞), N = NaivKahan | parity vs oracle | oracle t (1 core) | "
          "oracle t (16 cores) |")
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


def rows(table_path, oracle_path):
    one, many = oracle_times(oracle_path)
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
        out.append(f"| {r['config']} | {m} | {levels} | 1 | {r['ms']:.4g} | {r['gflops']:.0f} | "
                   f"{r['frac_fp64_peak']:.3f} | {executed} | {r['rel_err_vs_kahan']:.2e} | {parity} | {t1} | {t16} |")
    return out


def main(argv):
    table = argv[0]
    body = rows(table, os.path.join(ROOT, "profiles", "r01", "oracle_timing.jsonl"))
    text = "\n".join([HEADER, "|" + "---|" * 12] + body)
    if "--write" not in argv:
        print(text)
        return
    path = os.path.join(ROOT, "BASELINE.md")
    s = open(path).read()
    start = s.index("| cfg | method | levels | GPUs |")
    end = s.find("\n\n", start)
    end = len(s) if end < 0 else end
    s = s[:start] + text + s[end:]
    s = re.sub(r"profiles/r01/table_v\d+\.jsonl", "profiles/r01/" + os.path.basename(table), s)
    open(path, "w").write(s)
    print(f"BASELINE.md table regenerated from {table} ({len(body)} rows)")


if __name__ == "__main__":
    main(sys.argv[1:])
