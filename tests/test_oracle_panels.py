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


# ---- NaivKahan / WinogradOriginal panel steps (or_naive_kahan_acc, or_winograd_pairs_acc) ----
@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("shape", [(5, 1, 3), (7, 13, 9), (16, 40, 11), (3, 97, 4)])
def test_kahan_panels_compose_to_full_product(shape, fused):
    """Pinned against the separately pinned or_naive_kahan[_fused]: the (sum, err) state carried
    across any split of k reproduces the one-shot compensated sum bit for bit."""
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N * 37 + P)
    A = A * 1e6  # large dynamic range: the carried err matters
    full = oracle.naive_kahan_fused(A, B) if fused else oracle.naive_kahan(A, B)
    rng = np.random.default_rng(P + 1)
    for _ in range(4):
        cuts = sorted(set(rng.integers(1, P, size=min(3, P - 1)).tolist())) if P > 1 else []
        bounds = [0] + cuts + [P]
        S, E = np.zeros((N, M)), np.zeros((N, M))
        for k0, k1 in zip(bounds[:-1], bounds[1:]):
            oracle.naive_kahan_acc(A[:, k0:k1], B[k0:k1, :], S, E, fused)
        assert np.array_equal(S, full), bounds


def test_kahan_state_matters():
    """Dropping the carried err at a panel boundary changes the result (the pin is sensitive)."""
    A, B = workload.custom(4, 64, 4, seed=12)
    A = A * np.array([1e16 if k % 2 == 0 else 1.0 for k in range(64)])
    full = oracle.naive_kahan(A, B)
    S, E = np.zeros((4, 4)), np.zeros((4, 4))
    oracle.naive_kahan_acc(A[:, :32], B[:32], S, E)
    E[:] = 0.0
    oracle.naive_kahan_acc(A[:, 32:], B[32:], S, E)
    assert not np.array_equal(S, full)


@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("shape", [(5, 2, 3), (7, 14, 9), (16, 40, 11), (3, 96, 4)])
def test_winograd_panels_compose_to_full_product(shape, fused):
    """Pinned against or_winograd_original / or_winograd_fused (even P): pair sums carried across
    any split at even k, then (acc - y) - z."""
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N * 41 + P)
    full = oracle.winograd_fused(A, B) if fused else oracle.winograd_original(A, B)
    y, z = oracle.winograd_yz_fused(A, B) if fused else oracle.winograd_yz(A, B)
    rng = np.random.default_rng(P + 2)
    for _ in range(4):
        cuts = sorted(set((2 * rng.integers(1, P // 2, size=2)).tolist())) if P > 2 else []
        bounds = [0] + cuts + [P]
        Acc = np.zeros((N, M))
        for k0, k1 in zip(bounds[:-1], bounds[1:]):
            oracle.winograd_pairs_acc(A[:, k0:k1], B[k0:k1, :], Acc, fused)
        assert np.array_equal(oracle.winograd_finish(Acc, y, z), full), bounds
