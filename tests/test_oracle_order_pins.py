"""Pins for the evaluation ORDER the paper writes (tests/golden/order_cases.txt).

Each golden case is a tiny input, worked by hand from the cited formula, where the order the paper
states (the Kahan loop k = 1..n; (Sum - y_i) - z_k; the row sum of the
infinity norm left to right; the Strassen / Strassen-Winograd block sums left to right,
P:279-282) yields one value and any reversal or re-association another.  Every copy of
each formula in the oracle is checked: the full product, the per-entry replicas used for sampled
checks, the resumable panel steps of NEXT-4 and the lazy per-entry Strassen.
"""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_cases():
    out = {}
    with open(os.path.join(GOLDEN, "order_cases.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            cid, method, a, b, e = line.split()
            A = np.array(eval(a, {}), dtype=np.float64)  # exact integer / power-of-two expressions
            B = None if b == "-" else np.array(eval(b, {}), dtype=np.float64)
            out[cid] = (method, A, B, np.array(eval(e, {}), dtype=np.float64))
    return out


CASES = load_cases()


def test_cases_present():
    assert set(CASES) == {"O1", "O2", "O2s", "O3", "O4", "O5"}


def test_kahan_k_order():
    _, A, B, want = CASES["O1"]
    assert oracle.naive_kahan(A, B)[0, 0] == want
    assert oracle.entry(oracle.M_KAHAN, A, B, 0, 0) == want
    assert oracle.entries(oracle.M_KAHAN, A, B, [[0, 0]])[0] == want
    # the resumable panel step (NEXT-4): one panel, and the k-panels {0}, {1, 2} and {0, 1}, {2}
    S, E = np.zeros((1, 1)), np.zeros((1, 1))
    assert oracle.naive_kahan_acc(A, B, S, E)[0][0, 0] == want
    for cut in (1, 2):
        S, E = np.zeros((1, 1)), np.zeros((1, 1))
        oracle.naive_kahan_acc(A[:, :cut], B[:cut], S, E)
        oracle.naive_kahan_acc(A[:, cut:], B[cut:], S, E)
        assert S[0, 0] == want
    # every product here is exact, so the NEXT-3 fused variant (reading R22) must agree
    assert oracle.naive_kahan_fused(A, B)[0, 0] == want
    assert oracle.entry(oracle.M_KAHAN_FUSED, A, B, 0, 0) == want
    S, E = np.zeros((1, 1)), np.zeros((1, 1))
    assert oracle.naive_kahan_acc(A, B, S, E, fused=True)[0][0, 0] == want
    # the reversed loop and plain summation both give 2^53 (order_cases.txt O1)
    assert oracle.naive_kahan(A[:, ::-1].copy(), B[::-1].copy())[0, 0] == 2.0 ** 53
    assert oracle.naive_standard(A, B)[0, 0] == 2.0 ** 53


def test_winograd_sum_minus_y_minus_z():
    _, A, B, want = CASES["O2"]
    assert oracle.winograd_original(A, B)[0, 0] == want
    assert oracle.entry(oracle.M_WINOGRAD, A, B, 0, 0) == want
    y, z = oracle.winograd_yz(A, B)
    assert (y[0], z[0]) == (1.0, 2.0 ** 53 + 2.0 ** 27)
    acc = oracle.winograd_pairs_acc(A, B, np.zeros((1, 1)))
    assert acc[0, 0] == 2.0 ** 53 + 2.0 ** 28 + 2.0 ** 26 + 2
    assert oracle.winograd_finish(acc, y, z)[0, 0] == want
    # every product here is exact, so the NEXT-3 fused variant (reading R22) must agree
    assert oracle.winograd_fused(A, B)[0, 0] == want
    assert oracle.entry(oracle.M_WINOGRAD_FUSED, A, B, 0, 0) == want
    acc = oracle.winograd_pairs_acc(A, B, np.zeros((1, 1)), fused=True)
    assert oracle.winograd_finish(acc, *oracle.winograd_yz_fused(A, B))[0, 0] == want
    # the alternatives of order_cases.txt O2 are different numbers
    assert want not in (2.0 ** 27 + 2.0 ** 26 + 2, 2.0 ** 27 + 2.0 ** 26 + 1)


def test_winograd_scaled_sum_minus_y_minus_z():
    _, A, B, want = CASES["O2s"]
    assert oracle.lam(oracle.norm_inf(A), oracle.norm_inf(B)) == 0
    C, lam = oracle.winograd_scaled(A, B)
    assert lam == 0 and np.array_equal(C, want)
    got = oracle.entries(oracle.M_WINOGRAD_SCALED, A, B, [[0, 0], [1, 0]], lam_=0)
    assert np.array_equal(got, want[:, 0])
    C, lam = oracle.winograd_scaled_fused(A, B)  # exact products: the fused variant agrees
    assert lam == 0 and np.array_equal(C, want)
    got = oracle.entries(oracle.M_WINOGRAD_SCALED_FUSED, A, B, [[0, 0], [1, 0]], lam_=0)
    assert np.array_equal(got, want[:, 0])


def test_norm_inf_row_left_to_right():
    _, X, _, want = CASES["O3"]
    assert oracle.norm_inf(X) == want
    assert oracle.norm_inf(X[:, ::-1].copy()) == 2.0 ** 53  # right to left


@pytest.mark.parametrize("cid,variant", [("O4", oracle.STRASSEN_NAIV), ("O5", oracle.STRASSEN_WINOGRAD)])
@pytest.mark.parametrize("base", [oracle.BASE_LITERAL, oracle.BASE_FMA])
def test_strassen_combination_left_to_right(cid, variant, base):
    _, A, B, want = CASES[cid]
    assert np.array_equal(oracle.strassen(variant, A, B, levels=1, pad=(2, 2, 2), base=base), want)
    ij = [[i, j] for i in range(2) for j in range(2)]
    lazy = oracle.entries_strassen(variant, A, B, ij, levels=1, pad=(2, 2, 2), base=base)
    assert np.array_equal(lazy.reshape(2, 2), want)


def test_strassen_cases_round():
    # the cases are informative: the exact products differ from the pinned floating-point values
    for cid in ("O4", "O5"):
        _, A, B, want = CASES[cid]
        exact = oracle.int64_gemm(A.astype(np.int64), B.astype(np.int64)).astype(np.float64)
        assert not np.array_equal(exact, want)
