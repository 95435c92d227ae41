"""Pins for the oracle's Strassen and the paper's printed table."""
import os

import numpy as np
import pytest

import oracle
import workload

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_paper_padding_plans():
    # PAPER.md:286, worked by hand: X=800 -> floor(log2 800)=9, k=5, m=floor(800/32)+1=26, Y=832
    assert oracle.strassen_plan_paper(800, 800, 800) == (5, 26, 832)
    assert oracle.strassen_plan_paper(400, 400, 400) == (4, 26, 416)
    assert oracle.strassen_plan_paper(200, 200, 200) == (3, 26, 208)
    assert oracle.strassen_plan_paper(128, 128, 128) == (3, 17, 136)
    assert oracle.strassen_plan_paper(1024, 1024, 1024) == (6, 17, 1088)
    assert oracle.strassen_plan_paper(10, 3, 7) == (0, 11, 11)  # k < 0 clamped (reading R8)
    assert oracle.strassen_plan_paper(4096, 1001, 3000) == (8, 17, 4352)
    for X in range(1, 4097, 7):
        k, m, Y = oracle.strassen_plan_paper(X, 1, 1)
        assert Y >= X and Y == m * 2 ** k and (k == 0 or 16 <= m <= 32)


def test_levels_plan():
    assert oracle.strassen_plan_levels(4096, 1001, 3000, 2, 2) == (4096, 1008, 3000)
    assert oracle.strassen_plan_levels(8192, 8192, 8192, 3, 2) == (8192, 8192, 8192)
    assert oracle.strassen_plan_levels(5, 6, 7, 1, 1) == (6, 6, 8)


@pytest.mark.parametrize("variant,ops_per_node", [(0, 18), (1, 15)])
def test_structure_counts(variant, ops_per_node):
    # 7^d base products; 18 or 15 block additions per node
    A, B = workload.custom(16, 16, 16, 5)
    for d in range(4):
        oracle.strassen(variant, A, B, levels=d, pad=(16, 16, 16))
        prods, ops = oracle.strassen_counters()
        assert prods == 7 ** d
        assert ops == ops_per_node * sum(7 ** l for l in range(d))


@pytest.mark.parametrize("base", [oracle.BASE_LITERAL, oracle.BASE_FMA])
def test_depth0_is_base(base):
    A, B = workload.custom(13, 9, 6, 8)
    ref = oracle.naive_standard(A, B) if base == 0 else oracle.naive_fma(A, B)
    for v in (0, 1):
        assert np.array_equal(oracle.strassen(v, A, B, levels=0, pad=(13, 9, 6), base=base), ref)


def test_real_accuracy_vs_kahan():
    A, B = workload.operands("c1")
    K = oracle.naive_kahan(A, B)
    tol = 1e-10 * oracle.norm_inf(A) * oracle.norm_inf(B)
    for v in (0, 1):
        for lv in (1, 2, 3):
            C = oracle.strassen(v, A, B, levels=lv)
            assert oracle.norm_inf(oracle.minus(C, K)) <= tol


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("base", [0, 1])
def test_lazy_entry_bitwise(variant, base):
    cases = [((16, 16, 16), 2, None), ((21, 13, 9), 2, None), ((12, 7, 10), 3, None),
             ((11, 11, 11), -1, None), ((9, 5, 3), 1, None), ((4, 8, 6), 0, None)]
    for (N, P, M), lv, pad in cases:
        A, B = workload.custom(N, P, M, N * 100 + P)
        C = oracle.strassen(variant, A, B, levels=lv, pad=pad, base=base)
        idx = [(i, j) for i in range(N) for j in range(M)]
        got = oracle.entries_strassen(variant, A, B, idx, levels=lv, pad=pad, base=base).reshape(N, M)
        assert np.array_equal(got, C), ((N, P, M), lv)


# ---------------------------------------------------------------- the paper's printed table
def _table():
    rows = []
    with open(os.path.join(GOLDEN, "paper_table.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            n, name, val, ln = line.split()
            rows.append((int(n), name, float(val), int(ln)))
    return rows


def _deviations(n, seed=42):
    A, B = workload.paper_protocol(n, seed)
    N = oracle.naive_kahan(A, B)  # "N := NaivKahan"
    return {name: oracle.norm_inf(oracle.minus(N, oracle.paper_method(name, A, B))) for name in oracle.PAPER_METHODS}


def test_paper_table_n200_bands():
    dev = _deviations(200)
    for n, name, printed, ln in _table():
        if n != 200:
            continue
        # printed with 10 decimals: 0 => < 5e-11, 1e-10 => [5e-11, 1.5e-10); band widened by 25%
        if printed == 0.0:
            assert dev[name] < 6.25e-11, (name, ln, dev[name])
        else:
            assert 3.75e-11 <= dev[name] <= 1.875e-10, (name, ln, dev[name])


@pytest.mark.slow
def test_paper_table_n800():
    dev = _deviations(800)
    for n, name, printed, ln in _table():
        if n != 800:
            continue
        assert printed / 1.35 <= dev[name] <= printed * 1.35, (name, ln, dev[name], printed)
    # orderings the table shows
    assert dev["NaivLoopUnrollingFour"] < dev["NaivLoopUnrollingThree"] < dev["NaivLoopUnrollingTwo"] \
        < dev["NaivStandard"]
    assert dev["NaivStandard"] == dev["NaivOnArray"]
    assert dev["StrassenWinograd"] < dev["StrassenNaiv"]
    assert dev["WinogradScaled"] < dev["WinogradOriginal"]


def test_paper_protocol_lambda_tie():
    # B = 8A: ||B|| = 8 ||A|| exactly, lambda in {1, 2}; the table's WinogradScaled value supports 2
    A, B = workload.paper_protocol(64)
    assert oracle.norm_inf(B) == 8 * oracle.norm_inf(A)
    assert oracle.winograd_scaled(A, B)[1] == 2
