"""GPU parity of mm_naive_ex (the accumulate-mode DMMA GEMM behind the NEXT-4 panelised
broadcast/compute overlap): C = A B + C with every entry's fma chain continued from C equals the
oracle's or_naive_fma_acc bit for bit, and consecutive k-panels compose to mm_naive bit for bit
(even panel edges -> TMA path, odd edges -> 8-byte cp.async path)."""
import numpy as np
import pytest
import torch

import oracle
import workload

pytestmark = pytest.mark.gpu
mm = pytest.importorskip("paper_1106_1347_b200")
DEV = torch.device("cuda", 0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


@pytest.mark.parametrize("shape,cuts", [((300, 1000, 260), [2, 500, 998]), ((129, 77, 65), [1, 40, 41]),
                                        ((1024, 2048, 1024), [512, 1024, 1536]), ((64, 9, 64), [3])])
def test_panels_compose_bitwise(shape, cuts):
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N + P + M)
    dA, dB = dev(A), dev(B)
    full = mm.naive(dA, dB).cpu().numpy()
    assert np.array_equal(full, oracle.naive_fma(A, B))
    C = torch.empty((N, M), dtype=torch.float64, device=DEV)
    b = [0] + cuts + [P]
    for i, (k0, k1) in enumerate(zip(b[:-1], b[1:])):
        mm.naive_panel(dA[:, k0:k1], dB[k0:k1], C, accumulate=i > 0)
    assert np.array_equal(C.cpu().numpy(), full)


def test_accumulate_matches_oracle_strided():
    A, B = workload.custom(70, 90, 50, seed=8)
    C0 = workload.custom(70, 50, 1, seed=9)[0] * 100.0
    dA, dB = dev(A), dev(B)
    # strided views: A[:, 10:74], B[10:74, 3:47], C[:, 3:47] inside a wider buffer
    dC = dev(np.hstack([np.zeros((70, 3)), C0[:, 3:47], np.zeros((70, 3))]))
    mm.naive_panel(dA[:, 10:74], dB[10:74, 3:47], dC[:, 3:47], accumulate=True)
    ref = oracle.naive_fma_acc(np.ascontiguousarray(A[:, 10:74]), np.ascontiguousarray(B[10:74, 3:47]),
                               np.ascontiguousarray(C0[:, 3:47]))
    got = dC.cpu().numpy()
    assert np.array_equal(got[:, 3:47], ref)
    assert np.all(got[:, :3] == 0) and np.all(got[:, 47:] == 0)  # nothing outside the view is touched
