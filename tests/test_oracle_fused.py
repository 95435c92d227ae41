"""Pins for the oracle's NEXT-3 fused variants (reading R22 in DESIGN.md):
NaivKahan with err = fma(a, b, err) and WinogradOriginal / WinogradScaled with every
multiply-add (y, z, acc, odd-P term) as one fma.  Pinned by
  * hand-derived tie cases where fused and literal differ (tests/golden/fused_cases.txt),
  * exact integer arithmetic (int64 product) over a brute-force shape sweep,
  * bitwise equality with the (pinned) literal methods whenever every product is exact,
  * the exact rational product within Brent's bounds,
  * per-entry replicas = full functions (bitwise), the same lambda as WinogradScaled.
"""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workload

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
c, d = 1 - 2.0 ** -27, 1 + 2.0 ** -27


def _cases():
    out = {}
    with open(os.path.join(GOLDEN, "fused_cases.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            cid, method, fv, lv = line.split()
            out[cid] = (method, eval(fv, {}), eval(lv, {}))  # exact powers-of-two expressions
    return out


def test_hand_derived_fused_cases():
    cs = _cases()
    A = np.array([[1.0, 1.0, c]])
    B = np.array([[1.0], [2.0 ** -53], [c]])
    assert oracle.naive_kahan_fused(A, B)[0, 0] == cs["K1"][1]
    assert oracle.naive_kahan(A, B)[0, 0] == cs["K1"][2]
    A = np.array([[0.0, 0.0, 0.0, c]])
    B = np.array([[1.0], [2.0 ** -53], [0.0], [c]])
    assert oracle.winograd_fused(A, B)[0, 0] == cs["W1"][1]
    assert oracle.winograd_original(A, B)[0, 0] == cs["W1"][2]
    A = np.array([[0.0, 1.0, c]])
    B = np.array([[0.0], [-1.0], [d]])
    assert oracle.winograd_fused(A, B)[0, 0] == cs["W2"][1]
    assert oracle.winograd_original(A, B)[0, 0] == cs["W2"][2]


@pytest.mark.parametrize("P", list(range(1, 18)))
def test_integer_exact(P):
    for N, M in ((1, 1), (3, 5), (7, 2)):
        A, B = workload.custom(N, P, M, seed=100 * P + N, variant=1)
        exact = oracle.int64_gemm(A.astype(np.int64), B.astype(np.int64)).astype(np.float64)
        assert np.array_equal(oracle.naive_kahan_fused(A, B), exact)
        assert np.array_equal(oracle.winograd_fused(A, B), exact)
        assert np.array_equal(oracle.winograd_scaled_fused(A, B)[0], exact)


def test_equal_to_literal_when_products_exact():
    # entries k / 2^10 with |k| < 2^12: every a+b has <= 14 significant bits, so every product
    # (a*b, and (a+b)(a'+b')) is exact and fma(x, y, s) = rnd(s + rnd(x y)): fused == literal
    rng = np.random.default_rng(5)
    for N, P, M in ((4, 9, 5), (6, 16, 3), (3, 33, 7), (1, 1, 1), (5, 2, 4)):
        A = rng.integers(-4095, 4096, (N, P)) / 1024.0 * 2.0 ** rng.integers(-3, 4)
        B = rng.integers(-4095, 4096, (P, M)) / 1024.0
        assert np.array_equal(oracle.naive_kahan_fused(A, B), oracle.naive_kahan(A, B))
        assert np.array_equal(oracle.winograd_fused(A, B), oracle.winograd_original(A, B))


def _exact(A, B):
    N, P, M = A.shape[0], A.shape[1], B.shape[1]
    return [[sum(Fraction(A[i, k]) * Fraction(B[k, j]) for k in range(P)) for j in range(M)] for i in range(N)]


def test_within_brent_bounds_exact_rational():
    rng = np.random.default_rng(12)
    for case in range(20):
        N, M, P = int(rng.integers(1, 6)), int(rng.integers(1, 6)), int(rng.integers(1, 40))
        sa, sb = 10.0 ** rng.uniform(-6, 6), 10.0 ** rng.uniform(-6, 6)
        A = (2 * rng.random((N, P)) - 1) * sa
        B = (2 * rng.random((P, M)) - 1) * sb
        E = _exact(A, B)
        nA, nB = oracle.norm_inf(A), oracle.norm_inf(B)

        def err(C):
            return max(sum(abs(Fraction(C[i, j]) - E[i][j]) for j in range(M)) for i in range(N))

        assert err(oracle.winograd_fused(A, B)) <= Fraction(oracle.brent_bound_unscaled(P, nA, nB)), case
        assert err(oracle.winograd_scaled_fused(A, B)[0]) <= Fraction(oracle.brent_bound_scaled(P, nA, nB)), case
        # Kahan: |C - AB| <= (2u + O(P u^2)) sum |a||b|  -> generous 4u * sum|a||b| + tiny
        K = oracle.naive_kahan_fused(A, B)
        absAB = np.abs(A) @ np.abs(B)
        for i in range(N):
            for j in range(M):
                assert abs(Fraction(K[i, j]) - E[i][j]) <= Fraction(4 * 2.0 ** -53 * absAB[i, j]) + Fraction(
                    1, 2 ** 1074), case


def test_entries_bitwise_and_lambda():
    A, B = workload.custom(9, 17, 11, seed=3)
    A = A * 1e4
    Cs, lam = oracle.winograd_scaled_fused(A, B)
    assert lam == oracle.winograd_scaled(A, B)[1] == oracle.lam(oracle.norm_inf(A), oracle.norm_inf(B))
    idx = [(i, j) for i in range(9) for j in range(11)]
    for m, C in ((oracle.M_KAHAN_FUSED, oracle.naive_kahan_fused(A, B)),
                 (oracle.M_WINOGRAD_FUSED, oracle.winograd_fused(A, B)),
                 (oracle.M_WINOGRAD_SCALED_FUSED, Cs)):
        assert np.array_equal(oracle.entries(m, A, B, idx, lam).reshape(C.shape), C), m


def test_identity_and_zero():
    A, _ = workload.custom(7, 12, 1, seed=9)
    assert np.array_equal(oracle.naive_kahan_fused(A, np.eye(12)), A)
    Z = np.zeros((12, 4))
    assert np.all(oracle.naive_kahan_fused(A, Z) == 0)
    assert np.all(oracle.winograd_fused(A, Z) == 0)
