"""Summarise an ncu round (tools/ncu_round.sh output) into profiles/: a per-kernel share table from
the launch list and key metrics from the --set full capture, plus profiles/kernel_traffic.json
(per-launch DRAM bytes by kernel, read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").replace("mmk::", "")
    return base.strip()


def family(name: str) -> str:
    if "line_kernel<0" in name:
        return "line_kernel<0> (norm_inf)"
    if "line_kernel<1" in name or "line_kernel<2" in name:
        return "line_kernel<1> (winograd y/z)"
    for k in ("dgemm_tma_comb_kernel", "dgemm_tma_kernel", "dgemm_dmma_kernel", "kahan_tma_kernel", "kahan_gemm_kernel", "winograd_yz_kernel", "winograd_tma_kernel",
              "winograd_kernel",
              "strassen_form3_kernel", "strassen_form2_kernel", "strassen_combine2_kernel",
              "strassen_form_kernel", "strassen_combine_kernel", "norm_inf_kernel", "scale_copy_kernel",
              "lambda_kernel"):
        if k in name:
            return k
    return short(name)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def full_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared_pipe_%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_conflicts"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "dmma_inst"),
]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
              "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1}


def main(src=os.path.join(ROOT, "gpurun_out", "ncu"), dst=os.path.join(ROOT, "profiles", "r01")):
    os.makedirs(dst, exist_ok=True)
    md = [f"# ncu summary ({os.path.basename(os.path.normpath(dst))})", ""]
    L = launches(os.path.join(src, "launches.csv"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in L:
        v = float(d["Metric Value"]) * UNIT_SCALE.get(d["Metric Unit"], 1e-9)
        agg[family(d["Kernel Name"])][0] += 1
        agg[family(d["Kernel Name"])][1] += v
    tot = sum(v[1] for v in agg.values())
    md += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, bench.py --steps 2 --warmup 3)",
           "", "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
           "| kernel | launches | total ms | mean ms/launch | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        md.append(f"| {k} | {n} | {t * 1e3:.3f} | {t * 1e3 / n:.3f} | {100 * t / tot:.1f}% |")
    reps = [os.path.join(src, f) for f in sorted(os.listdir(src)) if f.endswith(".ncu-rep")]
    md += ["", "## `ncu --set full` captures (tools/quick_bench.py, c4 8192^3, one launch per kernel)", "",
           "| kernel | " + " | ".join(m[1] for m in METRICS) + " |", "|---" * (len(METRICS) + 1) + "|"]
    traffic = {}
    rows_all = []
    for rep in reps:
        hdr, units, data = full_raw(rep)
        rows_all += [(hdr, units, d) for d in data]
    for hdr, units, d in rows_all:
        kn = hdr.index("Kernel Name")
        vals = []
        rec = {}
        for m, short_name in METRICS:
            if m in hdr:
                i = hdr.index(m)
                raw = d[i]
                try:
                    v = float(raw.replace(",", ""))
                except ValueError:
                    v = None
                if v is not None and v != v:  # nan: a partially replayed launch
                    v = None
                if v is not None and units[i] in UNIT_SCALE:
                    v = v * UNIT_SCALE[units[i]]
                rec[short_name] = v
                vals.append("" if v is None else (f"{v:.4g}"))
            else:
                vals.append("n/a")
        if rec.get("dram_read") is None:
            continue  # partial replay
        md.append(f"| {short(d[kn])} | " + " | ".join(vals) + " |")
        fam = family(d[kn])
        if fam not in traffic and rec.get("dram_read") is not None:
            traffic[fam] = int(rec["dram_read"] + (rec.get("dram_write") or 0))
    hbm = os.path.join(src, "hbm_kernels.csv")
    if os.path.exists(hbm):
        rows = launches(hbm)
        per = collections.defaultdict(dict)
        for d in rows:
            key = (d["ID"], short(d["Kernel Name"]), d["Grid Size"])
            v = float(d["Metric Value"].replace(",", "")) * UNIT_SCALE.get(d["Metric Unit"], 1)
            per[key][d["Metric Name"]] = v
        md += ["", "## HBM-bound kernels (winograd_scaled + strassen_winograd at c4)", "",
               "| id | kernel | grid | time ms | DRAM read GB | DRAM write GB | achieved GB/s | dram % |", "|---|---|---|---|---|---|---|---|"]
        for (i, k, grid), m in sorted(per.items(), key=lambda x: int(x[0][0])):
            t = m.get("gpu__time_duration.sum", 0)
            rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
            md.append(f"| {i} | {k} | {grid} | {t * 1e3:.3f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                      f"{(rd + wr) / t / 1e9 if t else 0:.0f} | {m.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} |")
            fam = family(k)
            traffic.setdefault(fam, int(rd + wr))
    md += ["", "Time in seconds, bytes in bytes. `traffic` per launch (DRAM read + write) by kernel:", "",
           "```", json.dumps(traffic, indent=1), "```"]
    with open(os.path.join(dst, "ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    for d in {os.path.join(ROOT, "profiles"), dst}:
        with open(os.path.join(d, "kernel_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    # the raw ncu launch list and HBM-kernel metrics (small CSVs) travel with the summary
    for name in ("launches.csv", "hbm_kernels.csv"):
        if os.path.exists(os.path.join(src, name)):
            shutil.copyfile(os.path.join(src, name), os.path.join(dst, "ncu_" + name))
    print("\n".join(md))


if __name__ == "__main__":
    main(*sys.argv[1:])
