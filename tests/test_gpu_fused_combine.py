"""NEXT-1: the deepest Strassen-Winograd combination fused into the leaf GEMM's
epilogue (gemm_comb.cuh, running tiles in tensor memory) must give exactly the separate
combination pass's result: both settings of MM_STRASSEN_FUSED_COMBINE (read once per process, so
each runs in its own interpreter) are compared bitwise with the oracle on ragged shapes and depths
1-3, and with each other at a size where the default rule selects the fused kernel."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(r"""
    import os, sys
    sys.path.insert(0, os.environ["REPO"])
    import numpy as np, torch
    import paper_1106_1347_b200 as mm, oracle, workload
    dev = torch.device("cuda", 0)
    for (N, P, M, lv) in [(256, 256, 256, 1), (300, 200, 260, 2), (520, 384, 130, 3), (1024, 1024, 1024, 3),
                          (67, 45, 53, 2), (1030, 1026, 998, 3)]:
        A, B = workload.custom(N, P, M, seed=N + lv)
        C = mm.strassen_winograd(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), levels=lv).cpu().numpy()
        d, pad = oracle.plan(N, P, M, lv)
        assert np.array_equal(C, oracle.strassen(1, A, B, levels=d, pad=pad, base=oracle.BASE_FMA)), (N, P, M, lv)
    A, B = workload.custom(4096, 4096, 4096, seed=1)
    C = mm.strassen_winograd(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), levels=3)
    np.save(os.environ["OUT"], C.cpu().numpy())
    print("ok")
""")


def test_fused_combine_bitwise(tmp_path):
    outs = []
    for flag in ("0", "1"):
        out = str(tmp_path / f"c{flag}.npy")
        env = dict(os.environ, REPO=ROOT, OUT=out, MM_STRASSEN_FUSED_COMBINE=flag)
        r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0 and "ok" in r.stdout, (flag, r.stdout[-2000:] + r.stderr[-3000:])
        outs.append(out)
    import numpy as np

    assert np.array_equal(np.load(outs[0]), np.load(outs[1]))
