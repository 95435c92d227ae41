"""Development aid: the end-to-end step of bench.py (matmul_methods on pinned host operands, c4)
timed under different copy schedules -- the growth ratio of the first method's k-panels and the
minimum height of the last method's shrinking row blocks.  bench.py is the contract."""
import functools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1106_1347_b200 as mm  # noqa: E402


def main():
    n = 8192
    g = torch.Generator().manual_seed(1)
    hA = torch.randn(n, n, dtype=torch.float64, generator=g).pin_memory()
    hB = torch.randn(n, n, dtype=torch.float64, generator=g).pin_memory()
    order = ["naive", "winograd", "winograd_scaled", "strassen", "strassen_winograd", "kahan"]
    outs = {m: torch.empty((n, n), dtype=torch.float64).pin_memory() for m in order}
    orig_rows, orig_panels = mm._shrinking_rows, mm._growing_panels
    for ratio, min_rows, blocks in ((1.4, 256, 8), (1.4, 512, 8), (1.4, 1024, 8), (1.0, 256, 8), (1.4, 256, 12),
                                    (1.25, 256, 10)):
        mm._shrinking_rows = functools.partial(orig_rows, min_rows=min_rows)
        mm._growing_panels = functools.partial(orig_panels, ratio=ratio)
        for _ in range(2):
            mm.matmul_methods(hA, hB, order, levels=3, outs=outs, row_blocks=blocks)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            mm.matmul_methods(hA, hB, order, levels=3, outs=outs, row_blocks=blocks)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"ratio": ratio, "min_rows": min_rows, "blocks": blocks,
                          "ms_per_step": round(e0.elapsed_time(e1) / 3, 3)}), flush=True)


if __name__ == "__main__":
    main()
