"""Pins for the CPU oracle (oracle/), independent of the oracle's own code.

Each test checks the oracle against something the paper or mathematics fixes:
hand-computed worked examples (tests/golden/), exact integer arithmetic (an
independent int64 product), exact rational arithmetic (fractions.Fraction),
closed forms, IEEE tie cases worked out by hand, and the paper's printed table.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workload

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TWO53 = 2.0 ** 53


def _golden_2x2():
    vals = {}
    with open(os.path.join(GOLDEN, "worked_2x2.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, *v = line.split()
            vals[k] = [float(x) for x in v]
    return vals


A22 = np.array([[1.0, 2.0], [3.0, 4.0]])
B22 = np.array([[5.0, 6.0], [7.0, 8.0]])


def test_selfcheck():
    # contraction detector and the Kahan pin run at load (oracle.c or_selfcheck)
    assert oracle.lib().or_selfcheck() == 0


# ---------------------------------------------------------------- Section 1
def test_aux_examples():
    # PAPER.md:28-62; values worked by hand
    assert oracle.plus(A22, B22).tolist() == [[6, 8], [10, 12]]
    assert oracle.minus(B22, A22).tolist() == [[4, 4], [4, 4]]
    assert oracle.scalar_mul(8.0, A22).tolist() == [[8, 16], [24, 32]]
    assert oracle.norm_inf(np.array([[1.0, -2.0], [3.0, 4.0]])) == 7.0  # row sums 3, 7
    assert oracle.norm_inf(np.eye(5)) == 1.0
    assert oracle.norm_inf(np.zeros((3, 4))) == 0.0
    assert oracle.max2(3, 7) == 7 and oracle.max2(5, 5) == 5 and oracle.max2(-1.5, -2.5) == -1.5
    X = workload.custom(7, 9, 3, 1)[0]
    assert np.array_equal(oracle.plus(X, np.zeros_like(X)), X)
    assert np.all(oracle.minus(X, X) == 0.0)
    # power-of-two scaling is exact and commutes with the norm
    assert oracle.norm_inf(oracle.scalar_mul(2.0 ** -7, X)) == 2.0 ** -7 * oracle.norm_inf(X)


def test_norm_inf_exact_on_integers():
    A, _ = workload.custom(33, 17, 2, 3, variant=1)
    assert oracle.norm_inf(A) == float(np.abs(A.astype(np.int64)).sum(axis=1).max())


# ---------------------------------------------------------------- worked 2x2 example
def test_worked_2x2_all_methods():
    g = _golden_2x2()
    C = np.array(g["C"]).reshape(2, 2)
    for name in oracle.PAPER_METHODS + ("NaivKahan",):
        assert np.array_equal(oracle.paper_method(name, A22, B22), C), name
    for lv in (0, 1):
        for v in (0, 1):
            for base in (0, 1):
                assert np.array_equal(oracle.strassen(v, A22, B22, levels=lv, pad=(2, 2, 2), base=base), C)
    y, z = oracle.winograd_yz(A22, B22)
    assert y.tolist() == g["y"] and z.tolist() == g["z"]


def test_worked_2x2_strassen_H():
    g = _golden_2x2()
    assert oracle.strassen_trace(oracle.STRASSEN_NAIV, A22, B22, 1).tolist() == g["H"]
    assert oracle.strassen_trace(oracle.STRASSEN_WINOGRAD, A22, B22, 1).tolist() == g["HW"][:7]


# ---------------------------------------------------------------- integer exactness (brute force)
SIZES = (1, 2, 3, 4, 5, 7, 8, 9, 16, 17)


def _all_methods(A, B):
    out = {
        "standard": oracle.naive_standard(A, B),
        "on_array": oracle.naive_on_array(A, B),
        "kahan": oracle.naive_kahan(A, B),
        "u2": oracle.naive_unroll(2, A, B),
        "u3": oracle.naive_unroll(3, A, B),
        "u4": oracle.naive_unroll(4, A, B),
        "fma": oracle.naive_fma(A, B),
        "winograd": oracle.winograd_original(A, B),
        "winograd_scaled": oracle.winograd_scaled(A, B)[0],
        "strassen_paper": oracle.strassen(0, A, B),
        "sw_paper": oracle.strassen(1, A, B),
    }
    N, P, M = A.shape[0], A.shape[1], B.shape[1]
    for lv in (1, 2, 3):
        pad = oracle.strassen_plan_levels(N, P, M, lv, 1)
        out[f"strassen_l{lv}"] = oracle.strassen(0, A, B, levels=lv, pad=pad)
        out[f"sw_l{lv}"] = oracle.strassen(1, A, B, levels=lv, pad=pad, base=1)
    return out


def test_integer_exact_bruteforce():
    seed = 0
    for N in SIZES:
        for P in SIZES:
            for M in (1, 3, 8, 17):
                seed += 1
                A, B = workload.custom(N, P, M, seed, variant=1)
                ref = oracle.int64_gemm(A.astype(np.int64), B.astype(np.int64)).astype(np.float64)
                for name, C in _all_methods(A, B).items():
                    assert np.array_equal(C, ref), (name, N, P, M)


def test_integer_exact_wide_range():
    # entries in [-1024, 1024] at P <= 64: all partial sums stay far below 2^53
    rng = np.random.default_rng(5)
    for (N, P, M) in ((13, 64, 11), (8, 63, 8), (32, 33, 31)):
        A = rng.integers(-1024, 1025, (N, P)).astype(np.float64)
        B = rng.integers(-1024, 1025, (P, M)).astype(np.float64)
        ref = oracle.int64_gemm(A.astype(np.int64), B.astype(np.int64)).astype(np.float64)
        for name, C in _all_methods(A, B).items():
            assert np.array_equal(C, ref), name


def test_identity_and_zero():
    A, _ = workload.custom(9, 11, 4, 7)
    I = np.eye(11)
    for f in (oracle.naive_standard, oracle.naive_on_array, oracle.naive_kahan, oracle.naive_fma,
              lambda a, b: oracle.naive_unroll(2, a, b), lambda a, b: oracle.naive_unroll(3, a, b),
              lambda a, b: oracle.naive_unroll(4, a, b)):
        assert np.array_equal(f(A, I), A)  # x*1 and x + 0 are exact
    Z = np.zeros((11, 5))
    for name in oracle.PAPER_METHODS + ("NaivKahan",):
        assert np.all(oracle.paper_method(name, A, Z) == 0.0), name


# ---------------------------------------------------------------- Kahan
def _row_times_ones(f, xs):
    A = np.array([xs], dtype=np.float64)
    return f(A, np.ones((len(xs), 1)))[0, 0]


def test_kahan_pins():
    eps = 2.0 ** -53
    # [1, 2^-53 x 10]: each 2^-53 is a tie and plain summation stays at 1;
    # Kahan carries them in err: exact sum 1 + 10 * 2^-53 = 1 + 5 * 2^-52 is representable
    xs = [1.0] + [eps] * 10
    assert _row_times_ones(oracle.naive_kahan, xs) == 1.0 + 5 * 2.0 ** -52
    assert _row_times_ones(oracle.naive_standard, xs) == 1.0
    # [2^53, 1, 1]: exact sum 2^53 + 2 is representable
    assert _row_times_ones(oracle.naive_kahan, [TWO53, 1.0, 1.0]) == TWO53 + 2
    assert _row_times_ones(oracle.naive_standard, [TWO53, 1.0, 1.0]) == TWO53
    # [1e16, 1, -1e16]: ulp(1e16) = 2, so 1e16 + 1 ties back to 1e16 and the 1 is
    # lost before the cancellation in both algorithms (SPEC's 1.0 is wrong)
    assert _row_times_ones(oracle.naive_kahan, [1e16, 1.0, -1e16]) == 0.0
    assert _row_times_ones(oracle.naive_standard, [1e16, 1.0, -1e16]) == 0.0


def test_kahan_statistically_more_accurate():
    A, B = workload.custom(16, 4000, 16, 11)
    exact = _exact_product_rows(A[:4], B)
    e_k = np.abs(oracle.naive_kahan(A, B)[:4] - exact).max()
    e_s = np.abs(oracle.naive_standard(A, B)[:4] - exact).max()
    assert e_k <= e_s


def _exact_product_rows(A, B):
    # exact sum of the rounded products (Fraction), rounded once at the end
    out = np.empty((A.shape[0], B.shape[1]))
    for i in range(A.shape[0]):
        for j in range(B.shape[1]):
            s = Fraction(0)
            for k in range(A.shape[1]):
                s += Fraction(float(A[i, k] * B[k, j]))
            out[i, j] = float(s)
    return out


# ---------------------------------------------------------------- unrolling
def test_unroll_grouping_pins():
    # worked by hand with round-half-even at 2^53 (ulp 2):
    # [1, 2^53, 1, 1]: standard 1 -> 2^53+1 ties to 2^53 -> 2^53 -> 2^53;
    #   u=2 groups (1+2^53)=2^53, (1+1)=2 -> 2^53+2
    xs = [1.0, TWO53, 1.0, 1.0]
    assert _row_times_ones(oracle.naive_standard, xs) == TWO53
    assert _row_times_ones(lambda a, b: oracle.naive_unroll(2, a, b), xs) == TWO53 + 2
    # [2^53, 0, 0, 1, 1, 0]: u=3 groups (2^53), (1+1+0)=2 -> 2^53+2; u=2 groups (2^53,0),(0,1),(1,0) -> 2^53
    xs = [TWO53, 0.0, 0.0, 1.0, 1.0, 0.0]
    assert _row_times_ones(lambda a, b: oracle.naive_unroll(3, a, b), xs) == TWO53 + 2
    assert _row_times_ones(lambda a, b: oracle.naive_unroll(2, a, b), xs) == TWO53
    # [2^53, 0,0,0, 0,1,1,0]: u=4 second group = 2 -> 2^53+2; u=2, u=3 and standard -> 2^53
    xs = [TWO53, 0, 0, 0, 0, 1.0, 1.0, 0]
    assert _row_times_ones(lambda a, b: oracle.naive_unroll(4, a, b), xs) == TWO53 + 2
    for u in (2, 3):
        assert _row_times_ones(lambda a, b: oracle.naive_unroll(u, a, b), xs) == TWO53
    # odd tail appended last, in increasing k: [1, 1, 2^53] with u=2 -> (1+1) then + 2^53 = 2^53+2
    assert _row_times_ones(lambda a, b: oracle.naive_unroll(2, a, b), [1.0, 1.0, TWO53]) == TWO53 + 2


def test_on_array_bitwise_standard():
    A, B = workload.custom(20, 37, 19, 12)
    assert np.array_equal(oracle.naive_on_array(A, B), oracle.naive_standard(A, B))


# ---------------------------------------------------------------- fused reading R2 (probe P3)
def test_fma_matches_measured_dmma_semantics():
    # profiles/r01_probe/fp64_probe.jsonl, probe P3: DMMA on B200 returned these
    f = lambda xs: _row_times_ones(oracle.naive_fma, xs)
    assert f([TWO53, 1.0, 1.0, 0.0]) == TWO53
    assert f([1.0, 1.0, TWO53, 0.0]) == TWO53 + 2
    assert f([1e16, 1.0, -1e16, 1.0]) == 1.0
    # fused product: (1 + 2^-30)(1 - 2^-30) - 1 = -2^-60 exactly
    a = np.array([[1.0 + 2.0 ** -30, -1.0]])
    b = np.array([[1.0 - 2.0 ** -30], [1.0]])
    # k=0: fma(a0, b0, 0) rounds the product to 1; k=1: fma(-1, 1, 1) = 0 -- a chain, not one fused dot
    assert oracle.naive_fma(a, b)[0, 0] == 0.0
    a2 = np.array([[-1.0, 1.0 + 2.0 ** -30]])
    b2 = np.array([[1.0], [1.0 - 2.0 ** -30]])
    assert oracle.naive_fma(a2, b2)[0, 0] == -(2.0 ** -60)
    assert oracle.naive_standard(a2, b2)[0, 0] == 0.0


# ---------------------------------------------------------------- Winograd
def test_winograd_odd_p_single():
    # P=1 -> gamma=0, y=z=0, only the odd-P correction A_{i,P}B_{P,k}
    assert oracle.winograd_original(np.array([[3.0]]), np.array([[4.0]]))[0, 0] == 12.0


def test_winograd_yz_closed_form_integers():
    A, B = workload.custom(6, 9, 5, 21, variant=1)
    y, z = oracle.winograd_yz(A, B)
    Ai, Bi = A.astype(np.int64), B.astype(np.int64)
    assert y.tolist() == [float(sum(Ai[i, 2 * j] * Ai[i, 2 * j + 1] for j in range(4))) for i in range(6)]
    assert z.tolist() == [float(sum(Bi[2 * j, k] * Bi[2 * j + 1, k] for j in range(4))) for k in range(5)]


def test_lambda_pins():
    assert oracle.lam(1, 64) == 3       # 2^6 / 1: unique
    assert oracle.lam(1, 8) == 2        # tie {1, 2} -> larger |lambda| (paper protocol B = 8A)
    assert oracle.lam(8, 1) == -2       # tie {-2, -1}
    assert oracle.lam(1, 2) == 1        # tie {0, 1}
    assert oracle.lam(1, 32) == 3       # tie {2, 3}
    assert oracle.lam(1, 1) == 0
    assert oracle.lam(0.0, 3.0) == 0 and oracle.lam(3.0, 0.0) == 0
    assert oracle.lam(5.33e8, 1.55e-3) == -19  # config c3 scales


def test_lambda_bracket_property():
    # 1/2 <= 2^(2 lambda) nA / nB <= 2, checked exactly with Fractions
    rng = np.random.default_rng(3)
    for _ in range(3000):
        nA = float(rng.uniform(0.5, 1.0)) * 2.0 ** int(rng.integers(-100, 101))
        nB = float(rng.uniform(0.5, 1.0)) * 2.0 ** int(rng.integers(-100, 101))
        lam = oracle.lam(nA, nB)
        r = Fraction(2) ** (2 * lam) * Fraction(nA) / Fraction(nB)
        assert Fraction(1, 2) <= r <= 2, (nA, nB, lam)
        # and it is the only one unless the boundary is hit
        for other in (lam - 1, lam + 1):
            r2 = Fraction(2) ** (2 * other) * Fraction(nA) / Fraction(nB)
            if Fraction(1, 2) <= r2 <= 2:
                assert r == 2 or r == Fraction(1, 2)
                assert abs(lam) >= abs(other)


def test_winograd_scaled_lambda0_is_original():
    A, B = workload.custom(12, 15, 10, 31)
    C, lam = oracle.winograd_scaled(A, B)
    assert lam == 0
    assert np.array_equal(C, oracle.winograd_original(A, B))


def test_winograd_scaled_power_of_two_identity():
    # scaling by 2^lambda is exact, so scaled Winograd on (A, B) equals WinogradOriginal
    # on the explicitly scaled operands bitwise
    A, B = workload.custom(8, 13, 7, 41)
    B = B * 2.0 ** -20
    C, lam = oracle.winograd_scaled(A, B)
    assert lam != 0
    ref = oracle.winograd_original(A * 2.0 ** lam, B * 2.0 ** -lam)
    assert np.array_equal(C, ref)


def _exact(A, B):
    N, P = A.shape
    M = B.shape[1]
    return [[sum(Fraction(float(A[i, k])) * Fraction(float(B[k, j])) for k in range(P)) for j in range(M)]
            for i in range(N)]


def _norm_err(C, E):
    return max(sum(abs(Fraction(float(C[i, j])) - E[i][j]) for j in range(C.shape[1])) for i in range(C.shape[0]))


def test_winograd_within_brent_bounds_exact_rational():
    # PAPER.md:199 and :214, n := P (reading R12), u = 2^-53; exact product via Fractions
    rng = np.random.default_rng(11)
    for case in range(25):
        N, M = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        P = int(rng.integers(1, 42))
        sa, sb = 10.0 ** rng.uniform(-6, 6), 10.0 ** rng.uniform(-6, 6)
        A = (2 * rng.random((N, P)) - 1) * sa
        B = (2 * rng.random((P, M)) - 1) * sb
        E = _exact(A, B)
        nA, nB = oracle.norm_inf(A), oracle.norm_inf(B)
        e0 = _norm_err(oracle.winograd_original(A, B), E)
        e1 = _norm_err(oracle.winograd_scaled(A, B)[0], E)
        assert e0 <= Fraction(oracle.brent_bound_unscaled(P, nA, nB)), case
        assert e1 <= Fraction(oracle.brent_bound_scaled(P, nA, nB)), case


def test_brent_bound_plugins():
    # N=1, norms 1: unscaled (1+12-8)/4 * 4 = 5, scaled 9/8 * 5 = 5.625 (in units of u)
    assert oracle.brent_bound_unscaled(1, 1.0, 1.0, u=1.0) == 5.0
    assert oracle.brent_bound_scaled(1, 1.0, 1.0, u=1.0) == 5.625
    # max_{1/2 <= k <= 2} k + 2 + 1/k = 9/2 at both ends
    ks = np.linspace(0.5, 2.0, 10001)
    assert abs((ks + 2 + 1 / ks).max() - 4.5) < 1e-12


# ---------------------------------------------------------------- per-entry replicas
@pytest.mark.parametrize("shape", [(9, 17, 11), (16, 16, 16), (5, 1, 7), (12, 33, 4)])
def test_entry_replicas_bitwise(shape):
    A, B = workload.custom(*shape, seed=sum(shape))
    A = A * 1e3
    full = {
        oracle.M_STANDARD: oracle.naive_standard(A, B),
        oracle.M_ON_ARRAY: oracle.naive_on_array(A, B),
        oracle.M_KAHAN: oracle.naive_kahan(A, B),
        oracle.M_UNROLL2: oracle.naive_unroll(2, A, B),
        oracle.M_UNROLL3: oracle.naive_unroll(3, A, B),
        oracle.M_UNROLL4: oracle.naive_unroll(4, A, B),
        oracle.M_FMA: oracle.naive_fma(A, B),
        oracle.M_WINOGRAD: oracle.winograd_original(A, B),
    }
    Cs, lam = oracle.winograd_scaled(A, B)
    full[oracle.M_WINOGRAD_SCALED] = Cs
    idx = [(i, j) for i in range(shape[0]) for j in range(shape[2])]
    for m, C in full.items():
        got = oracle.entries(m, A, B, idx, lam).reshape(C.shape)
        assert np.array_equal(got, C), m


def test_unit_roundoff_accuracy_sanity():
    # every method is close to the exact product on a well-conditioned case
    A, B = workload.custom(6, 50, 6, 77)
    E = np.array([[float(x) for x in row] for row in _exact(A, B)])
    for name in oracle.PAPER_METHODS + ("NaivKahan",):
        C = oracle.paper_method(name, A, B)
        assert np.abs(C - E).max() < 1e-13 * 50, name
    assert math.isfinite(oracle.norm_inf(A))
