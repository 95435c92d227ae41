"""Kernel-only device time per method call (no host / launch overhead), for the small configs
where a call is partly host bound.

Run under ncu, it calls every method once per config and writes a manifest of how many kernels
each call launched (the library's own counter); the parser then splits ncu's launch list in that
order and sums gpu__time_duration per call:

    python tools/kernel_times.py run --configs c2,c3 --manifest m.json        # plain run first
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file k.csv \\
        python tools/kernel_times.py run --configs c2,c3 --manifest m.json
    python tools/kernel_times.py parse k.csv m.json > kernel_times.jsonl
"""
from __future__ import annotations

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METHODS = [("naive", None), ("kahan", None), ("winograd", None), ("winograd_scaled", None), ("strassen", 2),
           ("strassen", 3), ("strassen_winograd", 2), ("strassen_winograd", 3), ("kahan_fused", None),
           ("winograd_fused", None), ("winograd_scaled_fused", None)]


def run(configs, manifest):
    import torch

    import paper_1106_1347_b200 as mm
    import workload

    calls = []
    for key in configs:
        A_h, B_h = workload.operands(key)
        A, B = torch.from_numpy(A_h).cuda(), torch.from_numpy(B_h).cuda()
        C = torch.empty((A.shape[0], B.shape[1]), dtype=torch.float64, device="cuda")
        for name, lv in METHODS:
            kw = {"levels": lv} if lv is not None else {}
            for rep in range(2):  # the first call warms caches / tensor maps; the second is reported
                n0 = mm.launch_count()
                getattr(mm, name)(A, B, out=C, **kw)
                torch.cuda.synchronize()
                calls.append({"config": key, "method": name, "levels": lv, "rep": rep,
                              "launches": mm.launch_count() - n0})
        del A, B, C
        torch.cuda.empty_cache()
    with open(manifest, "w") as f:
        json.dump(calls, f)


def parse(csv_path, manifest):
    import workload

    rows = list(csv.reader(open(csv_path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    launches = []  # ms per launch, in order (one metric row per launch)
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            launches.append(float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0))
    calls = json.load(open(manifest))
    assert sum(c["launches"] for c in calls) == len(launches), (sum(c["launches"] for c in calls), len(launches))
    pos = 0
    for c in calls:
        ks = launches[pos:pos + c["launches"]]
        pos += c["launches"]
        if c["rep"] == 0:
            continue
        cfg = workload.CONFIGS[c["config"]]
        ms = sum(ks)
        print(json.dumps({"config": c["config"], "method": c["method"], "levels": c["levels"], "launches": len(ks),
                          "kernel_ms": round(ms, 5), "kernel_gflops": round(2.0 * cfg.N * cfg.P * cfg.M / ms / 1e6, 1),
                          "per_kernel_ms": [round(x, 5) for x in ks]}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        import argparse

        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("--configs", default="c2,c3")
        ap.add_argument("--manifest", required=True)
        a = ap.parse_args()
        run(a.configs.split(","), a.manifest)
    else:
        parse(sys.argv[2], sys.argv[3])
