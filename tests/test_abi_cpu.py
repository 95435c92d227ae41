"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mm.h declares,
and its host-side logic (plans, workspace sizes, the lambda rule, argument errors) agrees with
the oracle.  No kernel is launched here."""
import os
import re

import numpy as np
import pytest

import oracle

mm = pytest.importorskip("paper_1106_1347_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1106_1347_b200 import build

    build.build()
    return mm.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "mm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b([A-Za-z_][A-Za-z0-9_]*)\s*\(", src)) -
                  {"if", "extern", "sizeof", "defined"})


def test_exports_every_header_symbol(L):
    names = header_functions()
    assert "mm_naive" in names and "norm_inf" in names
    for n in names:
        assert hasattr(L, n), n
    assert set(mm.EXPORTS) == set(names)


def test_version_and_status(L):
    assert b"sm_100a" in L.mm_version()
    for rc in (0, -1, -2, -3, -4, -6):
        assert L.mm_status_string(rc)


def test_strassen_plan_matches_oracle(L):
    for (N, P, M) in ((128, 128, 128), (200, 200, 200), (800, 800, 800), (1024, 1024, 1024), (10, 3, 7),
                      (4096, 1001, 3000)):
        k, m, Y = oracle.strassen_plan_paper(N, P, M)
        assert mm.strassen_plan(N, P, M, -1) == (k, Y, Y, Y)
    for lv in range(0, 5):
        for (N, P, M) in ((4096, 1001, 3000), (67, 45, 53), (8192, 8192, 8192), (1, 1, 1)):
            pad = oracle.strassen_plan_levels(N, P, M, lv, 2)
            assert mm.strassen_plan(N, P, M, lv) == (lv,) + pad


def test_workspace_sizes(L):
    assert mm.workspace_size("naive", 64, 64, 64) == 0
    assert mm.workspace_size("kahan", 64, 64, 64) == 0
    assert mm.workspace_size("winograd", 100, 7, 50) >= 8 * 150
    assert mm.workspace_size("winograd_scaled", 100, 7, 50) > mm.workspace_size("winograd", 100, 7, 50)
    assert mm.workspace_size("strassen", 64, 64, 64, 0) == 0
    s1 = mm.workspace_size("strassen_winograd", 1024, 1024, 1024, 1)
    s2 = mm.workspace_size("strassen_winograd", 1024, 1024, 1024, 2)
    # level-1 arena: S1 + T1 + H1 = 3 * 7 * 512^2 doubles
    assert s1 >= 3 * 7 * 512 * 512 * 8
    assert s2 > s1
    assert L.mm_workspace_size(0, 0, 4, 4, 0) == 0


def test_lambda_rule_matches_oracle(L):
    rng = np.random.default_rng(8)
    cases = [(1, 64), (1, 8), (8, 1), (1, 2), (1, 1), (0.0, 3.0), (5.33e8, 1.55e-3)]
    cases += [(float(rng.uniform(0.5, 1)) * 2.0 ** int(rng.integers(-60, 60)),
               float(rng.uniform(0.5, 1)) * 2.0 ** int(rng.integers(-60, 60))) for _ in range(2000)]
    for a, b in cases:
        assert mm.lambda_rule(a, b) == oracle.lam(a, b), (a, b)


def test_argument_errors_before_any_launch(L):
    # NULL pointers and bad sizes are rejected on the host (MM_ERR_ARG) -- no GPU touched
    assert L.mm_naive(None, None, None, 4, 4, 4, None) == -1
    assert L.mm_kahan(8, 16, 1 << 40, 0, 4, 4, None) == -1
    assert L.mm_strassen(8, 16, 1 << 40, 4, 4, 4, 12, None, 0, None) == -1
    assert L.norm_inf(None, 3, 3, None, None) == -1
    # aliasing C with A is rejected before the device check
    assert L.mm_naive(4096, 1 << 20, 4096, 16, 16, 16, None) == -2


def test_no_fallback_without_gpu(L):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    # well-formed arguments on a machine without a B200: unsupported, nothing computed
    assert L.mm_naive(1 << 20, 1 << 24, 1 << 28, 16, 16, 16, None) == -6


def test_dist_layer_host_errors():
    """mm_dist_* before mm_dist_init: argument errors, no crash, no GPU needed."""
    import paper_1106_1347_b200 as mm

    L = mm.lib()
    assert L.mm_dist_gemm(0, None, None, None, 1, 1, 1, 0, 0, 1, None, 0, None) == -1  # MM_ERR_ARG
    assert L.mm_dist_finalize() == -1
    assert L.mm_dist_init(0, 1, None, 0) == -1
    assert L.mm_dist_workspace_size(3, 4, 5, 6, 0) >= L.mm_workspace_size(3, 4, 5, 6, 0) + 256
    assert b"NCCL" in L.mm_status_string(-5)


def test_schedule_and_host_entry_errors():
    """mm_dist_schedule / mm_dist_step / mm_methods_host reject bad arguments on the host."""
    import ctypes

    import paper_1106_1347_b200 as mm
    from paper_1106_1347_b200 import dist as d

    L = mm.lib()
    ops = (d.DistOp * 4)()
    assert L.mm_dist_schedule(99, 64, 64, 2, 2, ops, 4) == -1  # unknown method
    assert L.mm_dist_schedule(0, 0, 64, 2, 2, ops, 4) == -1  # P < 1
    assert L.mm_dist_schedule(4, 64, 64, 9, 2, ops, 4) == -1  # levels out of range
    assert L.mm_dist_schedule(0, 8192, 8192, 2, 8, ops, 4) == -1  # the list does not fit
    assert L.mm_dist_schedule(0, 8192, 8192, 2, 1, ops, 4) == 4  # one broadcast, record, wait, full
    assert [o.op for o in ops] == [d.OP_BCAST, d.OP_RECORD, d.OP_WAIT, d.OP_FULL]
    assert L.mm_dist_step(0, None, None, None, None, 1, 1, 1, 0, 0, None, 0, None) == -1
    ids = (ctypes.c_int * 2)(0, 1)
    assert L.mm_methods_host_workspace_size(None, 2, 4, 4, 4, 0) == 0
    assert L.mm_methods_host_workspace_size(ids, 2, 4, 5, 6, 0) >= 8 * (4 * 5 + 5 * 6 + 2 * 4 * 6)
    bad = (ctypes.c_int * 1)(42)
    outs = (ctypes.c_void_p * 1)(1 << 20)
    assert L.mm_methods_host(bad, 1, 1 << 20, 1 << 21, outs, 4, 4, 4, 0, 1, 1 << 22, 1 << 20, None) == -1
    assert L.mm_methods_host(ids, 2, None, 1 << 21, outs, 4, 4, 4, 0, 1, 1 << 22, 1 << 20, None) == -1
