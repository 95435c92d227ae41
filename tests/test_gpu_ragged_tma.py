"""The TMA-fed main loops (K1 dgemm_tma, K2 kahan_tma, K3 winograd_tma) on RAGGED shapes: they
only engage when there are enough tiles (two CTA slots per SM), so the small shape sweeps do not
reach them.  Here N and M are not multiples of any tile size and P is even but not a multiple of
the 32-deep k tiles (partial last k tile: zero-filled pairs for Winograd, an exact stop at P for
Kahan), checked bitwise on sampled entries and full rows against the oracle's per-entry replicas."""
import numpy as np
import pytest
import torch

import oracle
import workload

pytestmark = pytest.mark.gpu
mm = pytest.importorskip("paper_1106_1347_b200")


@pytest.fixture(scope="module")
def ragged():
    N, P, M = 2210, 1002, 1094
    A, B = workload.custom(N, P, M, seed=2210)
    A = A * 1e3
    return A, B, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()


@pytest.mark.parametrize("method,code", [("naive", oracle.M_FMA), ("kahan", oracle.M_KAHAN),
                                         ("winograd", oracle.M_WINOGRAD),
                                         ("winograd_scaled", oracle.M_WINOGRAD_SCALED),
                                         ("kahan_fused", oracle.M_KAHAN_FUSED),
                                         ("winograd_fused", oracle.M_WINOGRAD_FUSED)])
def test_ragged_tma_paths_bitwise(ragged, method, code):
    A, B, dA, dB = ragged
    N, P, M = A.shape[0], A.shape[1], B.shape[1]
    C = getattr(mm, method)(dA, dB).cpu().numpy()
    lam = oracle.lam(oracle.norm_inf(A), oracle.norm_inf(B))
    idx = [tuple(map(int, x)) for x in workload.sample_positions(6, N, M, 2048, 1)]
    idx += [(r, j) for r in (0, N - 1) for j in range(M)] + [(i, M - 1) for i in range(N)]
    ref = oracle.entries(code, A, B, idx, lam)
    got = np.array([C[i, j] for i, j in idx])
    assert np.array_equal(got, ref), (method, np.abs(got - ref).max())


def test_ragged_gemm_big_config_bitwise():
    """Enough 64 x 64 tiles for K1's production configuration (64 x 64 x 32, the small-problem
    64 x 32 configuration covers the shapes above), ragged N, M and a partial last k tile."""
    N, P, M = 4100, 1002, 2050
    A, B = workload.custom(N, P, M, seed=4100)
    C = mm.naive(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    idx = [tuple(map(int, x)) for x in workload.sample_positions(7, N, M, 2048, 1)]
    idx += [(N - 1, j) for j in range(M)] + [(i, M - 1) for i in range(0, N, 7)]
    ref = oracle.entries(oracle.M_FMA, A, B, idx)
    assert np.array_equal(np.array([C[i, j] for i, j in idx]), ref)


@pytest.mark.parametrize("shape", [(1, 2, 2), (37, 46, 98), (100, 258, 130), (513, 1000, 514), (1000, 66, 1024)])
def test_small_grid_tma_winograd_bitwise(shape):
    """Grids under two waves of 128 x 64 tiles with P, M even and aligned operands take the
    TMA-fed 64 x 64 small-grid kernel (winograd.cuh WinogradTmaSmall, r02): ragged N and M, a
    partial last 32-deep k tile, a single-row problem; full products against the oracle, plain,
    scaled (lambda != 0) and fused."""
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N + 7 * P + 13 * M)
    A = A * 1e4
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    assert np.array_equal(mm.winograd(dA, dB).cpu().numpy(), oracle.winograd_original(A, B)), shape
    C, lam = oracle.winograd_scaled(A, B)
    assert lam != 0
    assert np.array_equal(mm.winograd_scaled(dA, dB).cpu().numpy(), C), shape
    assert np.array_equal(mm.winograd_fused(dA, dB).cpu().numpy(), oracle.winograd_fused(A, B)), shape
