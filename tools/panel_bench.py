"""Cost of the NEXT-4 panelised product on one GPU: NaivStandard at 8192^3 one-shot vs the same
product as k consecutive accumulate-mode panels (bitwise equal; the extra work is re-reading and
re-writing C once per panel).  Development aid; bench.py is the contract."""
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
    ref = mm.naive(A, B)
    t1 = timed(lambda: mm.naive(A, B, out=C))
    for panels in (2, 4, 8, 16):
        b = panel_bounds(n, panels)

        def run():
            for i, (k0, k1) in enumerate(b):
                mm.naive_panel(A[:, k0:k1], B[k0:k1], C, accumulate=i > 0)

        t = timed(run)
        torch.cuda.synchronize()
        bad = int((C != ref).sum())
        print(json.dumps({"n": n, "panels": panels, "ms_one_shot": round(t1, 3), "ms_panels": round(t, 3),
                          "mismatches": bad, "nan": int(torch.isnan(C).sum()), "ref_nan": int(torch.isnan(ref).sum())}),
              flush=True)


if __name__ == "__main__":
    main()
