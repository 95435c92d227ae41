"""GPU parity at the size limit of 32-bit element offsets: one operand (or C) with more than
2^31 elements, so that any int32 row * pitch product in a kernel overflows.

  * S1: A is 70000 x 32770 (2.29e9 elements, 18.4 GB): rows >= 65533 start past 2^31 elements;
        K4/K5 lines of 32770 elements; even P (TMA paths) and odd P = 32771 (cp.async paths).
  * S2: C is 70000 x 32770 (N x M > 2^31): the epilogue stores past 2^31 elements.

Sampled entries (half of them in the rows past 2^31) are compared bitwise with the oracle's
per-entry replicas, as in test_gpu_parity.py; ||A||_inf of the 18 GB operand bitwise as well.
"""
import numpy as np
import pytest
import torch

import oracle
import workload

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_1106_1347_b200")

DEV = torch.device("cuda", 0)
N_BIG, P_BIG, SMALL = 70000, 32770, 34
ALL = ("naive", "kahan", "winograd", "winograd_scaled", "strassen", "strassen_winograd")
ORACLE_M = {"naive": oracle.M_FMA, "kahan": oracle.M_KAHAN, "winograd": oracle.M_WINOGRAD,
            "winograd_scaled": oracle.M_WINOGRAD_SCALED}


def _positions(N, M, first_big_row, seed):
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([workload.SEED, 77, seed])))
    lo = [(int(i), int(j)) for i, j in zip(rng.integers(0, N, 128), rng.integers(0, M, 128))]
    hi = [(int(i), int(j)) for i, j in zip(rng.integers(first_big_row, N, 128), rng.integers(0, M, 128))]
    corners = [(N - 1, M - 1), (N - 1, 0), (first_big_row, 0)]
    return lo + hi + corners


def _gather(C: torch.Tensor, idx):
    ii = torch.tensor([i for i, _ in idx], device=C.device)
    jj = torch.tensor([j for _, j in idx], device=C.device)
    return C[ii, jj].cpu().numpy()


def _reference(method, A, B, idx, levels):
    if method.startswith("strassen"):
        d, (Np, Pp, Mp) = oracle.plan(A.shape[0], A.shape[1], B.shape[1], levels)
        return oracle.entries_strassen(0 if method == "strassen" else 1, A, B, idx, levels=d, pad=(Np, Pp, Mp),
                                       base=oracle.BASE_FMA)
    lam = oracle.lam(oracle.norm_inf(A), oracle.norm_inf(B)) if method == "winograd_scaled" else 0
    return oracle.entries(ORACLE_M[method], A, B, idx, lam)


def _run(method, dA, dB, levels):
    if method.startswith("strassen"):
        return getattr(mm, method)(dA, dB, levels=levels)
    return getattr(mm, method)(dA, dB)


def _check_all(A, B, first_big_row, seed, methods=ALL):
    dA = torch.from_numpy(A).to(DEV)
    dB = torch.from_numpy(B).to(DEV)
    N, M = A.shape[0], B.shape[1]
    idx = _positions(N, M, first_big_row, seed)
    for method in methods:
        for levels in ((1,) if method.startswith("strassen") else (0,)):  # d=1 keeps the arena ~1.75 A
            C = _run(method, dA, dB, levels)
            got = _gather(C, idx)
            del C
            ref = _reference(method, A, B, idx, levels)
            assert np.array_equal(got, ref), (method, levels, np.abs(got - ref).max())
    mm.release_workspace()
    return dA, dB


@pytest.mark.parametrize("P", [P_BIG, P_BIG + 1])
def test_a_past_2_31_elements(P):
    A, B = workload.custom(N_BIG, P, SMALL, seed=41 + P % 2)
    assert A.size > 2 ** 31
    first_big_row = 2 ** 31 // P + 1
    methods = ALL if P % 2 == 0 else ("naive", "kahan", "winograd", "winograd_scaled")
    dA, dB = _check_all(A, B, first_big_row, seed=P % 2, methods=methods)
    # ||A||_inf over 2.3e9 elements (K4 lines of 32770 / 32771 terms)
    assert float(mm.norm_inf(dA)) == oracle.norm_inf(A)
    del dA, dB
    torch.cuda.empty_cache()


def test_c_past_2_31_elements():
    A, B = workload.custom(N_BIG, SMALL, P_BIG, seed=43)
    assert A.shape[0] * B.shape[1] > 2 ** 31
    first_big_row = 2 ** 31 // P_BIG + 1
    dA, dB = _check_all(A, B, first_big_row, seed=2)
    del dA, dB
    torch.cuda.empty_cache()
