"""Pins for or_naive_fma_acc (reading R2 continued; the panel step of SURVEY.md 8(f) NEXT-4):
C = A B + C with every entry's fma chain started from C.  Pinned against the (separately pinned)
or_naive_fma: consecutive k-panels compose to the full product bit for bit, and a start value
with identical rows is the same as one more leading term (A' = [1 | A], B' = [c ; B])."""
import numpy as np
import pytest

import oracle
import workload


@pytest.mark.parametrize("shape", [(5, 1, 3), (7, 13, 9), (16, 40, 11), (3, 97, 4)])
def test_panels_compose_to_full_product(shape):
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N * 31 + P)
    A = A * 1e3
    full = oracle.naive_fma(A, B)
    rng = np.random.default_rng(P)
    for _ in range(4):
        cuts = sorted(set(rng.integers(1, P, size=min(3, P - 1)).tolist())) if P > 1 else []
        bounds = [0] + cuts + [P]
        C = np.zeros((N, M))
        for k0, k1 in zip(bounds[:-1], bounds[1:]):
            oracle.naive_fma_acc(A[:, k0:k1], B[k0:k1, :], C)
        assert np.array_equal(C, full), bounds


def test_start_value_is_a_leading_term():
    A, B = workload.custom(6, 21, 8, seed=4)
    c = workload.custom(1, 8, 1, seed=5)[0].reshape(-1) * 50.0
    C0 = np.tile(c, (6, 1))
    got = oracle.naive_fma_acc(A, B, C0.copy())
    A1 = np.hstack([np.ones((6, 1)), A])
    B1 = np.vstack([c.reshape(1, -1), B])
    assert np.array_equal(got, oracle.naive_fma(A1, B1))


def test_integer_exact():
    A, B = workload.custom(9, 14, 5, seed=2, variant=1)
    C0 = workload.custom(9, 5, 1, seed=3, variant=1)[0]
    exact = oracle.int64_gemm(A.astype(np.int64), B.astype(np.int64)) + C0.astype(np.int64)
    assert np.array_equal(oracle.naive_fma_acc(A, B, C0.copy()), exact.astype(np.float64))
