"""Cost of the NEXT-4 panelised product on one GPU: NaivStandard, NaivKahan and WinogradOriginal at
8192^3 one-shot vs the same product as k consecutive state-carrying panels (bitwise equal; the
extra work is re-reading and re-writing the carried state once per panel, plus the partial last
k tile of each panel).  Development aid; bench.py is the contract."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1106_1347_b200 as mm  # noqa: E402
from paper_1106_1347_b200.dist import panel_bounds  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(n=8192):
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(n, n, dtype=torch.float64, device="cuda")
    E = torch.empty(n, n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    methods = sys.argv[1].split(",") if len(sys.argv) > 1 else ["naive", "kahan", "winograd"]
    for m in methods:
        ref = getattr(mm, m)(A, B)
        t1 = timed(lambda: getattr(mm, m)(A, B, out=C))
        for panels in (2, 4, 8, 16):
            b = panel_bounds(n, panels)

            def run():
                if m == "winograd":
                    mm.winograd_yz(A, B, y, z)
                for i, (k0, k1) in enumerate(b):
                    first, last = i == 0, i == len(b) - 1
                    if m == "naive":
                        mm.naive_panel(A[:, k0:k1], B[k0:k1], C, accumulate=not first)
                    elif m == "kahan":
                        mm.kahan_panel(A[:, k0:k1], B[k0:k1], C, E, accumulate=not first, keep_state=not last)
                    else:
                        mm.winograd_panel(A[:, k0:k1], B[k0:k1], C, y, z, accumulate=not first, keep_state=not last)

            t = timed(run)
            torch.cuda.synchronize()
            bad = int((C != ref).sum())
            print(json.dumps({"method": m, "n": n, "panels": panels, "ms_one_shot": round(t1, 3),
                              "ms_panels": round(t, 3), "overhead": round(t / t1 - 1, 4), "mismatches": bad}),
                  flush=True)


if __name__ == "__main__":
    main()
