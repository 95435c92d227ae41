"""Print DRAM bytes, time and achieved GB/s per launch from an ncu --csv metrics log
(tools/gpu/check_hbm.sh output).  Usage: python tools/hbm_table.py gpurun_out/ncu/hbm_kernels.csv"""
import collections
import csv
import sys

TS = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "second": 1.0}
BS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    per = collections.OrderedDict()
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", ""), d["Grid Size"])
        per.setdefault(key, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    print("| id | kernel | grid | time ms | DRAM read GB | DRAM write GB | GB/s | dram % of ncu peak |")
    print("|---|---|---|---|---|---|---|---|")
    for (i, k, g), m in per.items():
        t = m["gpu__time_duration.sum"]
        tt = t[0] * TS.get(t[1], 1)
        rd = m["dram__bytes_read.sum"][0] * BS[m["dram__bytes_read.sum"][1]]
        wr = m["dram__bytes_write.sum"][0] * BS[m["dram__bytes_write.sum"][1]]
        pct = m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", (0, ""))[0]
        print(f"| {i} | {k} | {g} | {tt * 1e3:.3f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | {(rd + wr) / tt / 1e9:.0f} | {pct:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
