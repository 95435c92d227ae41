"""GPU parity of the NEXT-3 fused variants (reading R22) against the
oracle's or_*_fused functions, bit for bit, through the C ABI: the hand-derived tie cases of
tests/golden/fused_cases.txt, a ragged shape sweep (odd P, 8-byte aligned operands), integer
exactness, ill-scaled c3 and c4 (bench launch configuration) sampled entries."""
import numpy as np
import pytest
import torch

import oracle
import workload

pytestmark = pytest.mark.gpu
mm = pytest.importorskip("paper_1106_1347_b200")
DEV = torch.device("cuda", 0)
c, d = 1 - 2.0 ** -27, 1 + 2.0 ** -27


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


REF = {"kahan_fused": oracle.naive_kahan_fused, "winograd_fused": oracle.winograd_fused,
       "winograd_scaled_fused": lambda A, B: oracle.winograd_scaled_fused(A, B)[0]}


def test_hand_derived_cases_on_gpu():
    A, B = np.array([[1.0, 1.0, c]]), np.array([[1.0], [2.0 ** -53], [c]])
    assert host(mm.kahan_fused(dev(A), dev(B)))[0, 0] == 2 - 2.0 ** -26 + 2.0 ** -52
    assert host(mm.kahan(dev(A), dev(B)))[0, 0] == 2 - 2.0 ** -26
    A, B = np.array([[0.0, 0.0, 0.0, c]]), np.array([[1.0], [2.0 ** -53], [0.0], [c]])
    assert host(mm.winograd_fused(dev(A), dev(B)))[0, 0] == 1 - 2.0 ** -26 + 2.0 ** -53
    assert host(mm.winograd(dev(A), dev(B)))[0, 0] == 1 - 2.0 ** -26
    A, B = np.array([[0.0, 1.0, c]]), np.array([[0.0], [-1.0], [d]])
    assert host(mm.winograd_fused(dev(A), dev(B)))[0, 0] == -2.0 ** -54
    assert host(mm.winograd(dev(A), dev(B)))[0, 0] == 0.0


@pytest.mark.parametrize("shape", [(1, 1, 1), (5, 3, 7), (33, 65, 17), (64, 63, 64), (127, 128, 129),
                                   (130, 1001, 66), (257, 16, 300), (300, 512, 280)])
def test_fused_shape_sweep_bitwise(shape):
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=7 * N + P + 3 * M)
    A = A * 1e5
    dA, dB = dev(A), dev(B)
    for name, ref in REF.items():
        assert np.array_equal(host(getattr(mm, name)(dA, dB)), ref(A, B)), (name, shape)
    C, lam = mm.winograd_scaled_fused(dA, dB, return_lambda=True)
    assert lam == oracle.lam(oracle.norm_inf(A), oracle.norm_inf(B))


def test_fused_integer_exact():
    A, B = workload.custom(70, 33, 90, seed=5, variant=1)
    exact = oracle.int64_gemm(A.astype(np.int64), B.astype(np.int64)).astype(np.float64)
    for name in REF:
        assert np.array_equal(host(getattr(mm, name)(dev(A), dev(B))), exact), name


def test_fused_large_tiles_tma_path():
    # enough tiles for the TMA-fed Winograd main loop (P, M even, 16-byte aligned)
    A, B = workload.custom(1024, 256, 1024, seed=21)
    for name in ("kahan_fused", "winograd_fused"):
        got = host(getattr(mm, name)(dev(A), dev(B)))
        idx = [tuple(map(int, x)) for x in workload.sample_positions(2, 1024, 1024, 2000, 5)]
        m = oracle.M_KAHAN_FUSED if name == "kahan_fused" else oracle.M_WINOGRAD_FUSED
        ref = oracle.entries(m, A, B, idx)
        assert np.array_equal(np.array([got[i, j] for i, j in idx]), ref), name


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_fused_sampled_full_size(cfg):
    A, B = workload.operands(cfg)
    N, P, M = A.shape[0], A.shape[1], B.shape[1]
    dA, dB = dev(A), dev(B)
    lam = oracle.lam(oracle.norm_inf(A), oracle.norm_inf(B))
    idx = [tuple(map(int, x)) for x in workload.sample_positions(int(cfg[1]), N, M, 1024, 3)]
    for name, m in (("kahan_fused", oracle.M_KAHAN_FUSED), ("winograd_fused", oracle.M_WINOGRAD_FUSED),
                    ("winograd_scaled_fused", oracle.M_WINOGRAD_SCALED_FUSED)):
        C = host(getattr(mm, name)(dA, dB))
        ref = oracle.entries(m, A, B, idx, lam)
        assert np.array_equal(np.array([C[i, j] for i, j in idx]), ref), (cfg, name)
        del C
    mm.release_workspace()
