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


# ---- NaivKahan / WinogradOriginal k-panels (mm_kahan_ex / mm_winograd_ex, NEXT-4) ----------
PANEL_CASES = [((300, 1000, 260), [2, 500, 998]), ((333, 130, 66), [64, 66]), ((2210, 1002, 1094), [96, 502]),
               ((40, 8, 2), [2, 4, 6])]


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("shape,cuts", PANEL_CASES)
def test_kahan_panels_compose_bitwise(shape, cuts, fused):
    """(sum, err) carried from panel to panel in C and E: bitwise the one-shot NaivKahan."""
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N + 3 * P + M)
    A = A * 1e4
    dA, dB = dev(A), dev(B)
    full = (mm.kahan_fused if fused else mm.kahan)(dA, dB).cpu().numpy()
    C = torch.empty((N, M), dtype=torch.float64, device=DEV)
    E = torch.empty((N, M), dtype=torch.float64, device=DEV)
    b = [0] + cuts + [P]
    for i, (k0, k1) in enumerate(zip(b[:-1], b[1:])):
        mm.kahan_panel(dA[:, k0:k1], dB[k0:k1], C, E, accumulate=i > 0, keep_state=k1 < P, fused=fused)
    assert np.array_equal(C.cpu().numpy(), full)
    if N * P * M <= 300 * 1000 * 260:
        ref = oracle.naive_kahan_fused(A, B) if fused else oracle.naive_kahan(A, B)
        assert np.array_equal(full, ref)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("shape,cuts", PANEL_CASES)
def test_winograd_panels_compose_bitwise(shape, cuts, fused):
    """Raw pair sums carried in C from panel to panel, y / z of the full operands applied by the
    last panel: bitwise the one-shot WinogradOriginal."""
    N, P, M = shape
    A, B = workload.custom(N, P, M, seed=N + 5 * P + M)
    dA, dB = dev(A), dev(B)
    full = (mm.winograd_fused if fused else mm.winograd)(dA, dB).cpu().numpy()
    y = torch.empty(N, dtype=torch.float64, device=DEV)
    z = torch.empty(M, dtype=torch.float64, device=DEV)
    mm.winograd_yz(dA, dB, y, z, fused=fused)
    C = torch.empty((N, M), dtype=torch.float64, device=DEV)
    b = [0] + cuts + [P]
    for i, (k0, k1) in enumerate(zip(b[:-1], b[1:])):
        mm.winograd_panel(dA[:, k0:k1], dB[k0:k1], C, y, z, accumulate=i > 0, keep_state=k1 < P, fused=fused)
    assert np.array_equal(C.cpu().numpy(), full)
    if N * P * M <= 300 * 1000 * 260:
        ref = oracle.winograd_fused(A, B) if fused else oracle.winograd_original(A, B)
        assert np.array_equal(full, ref)


def test_panel_ex_argument_errors():
    L = mm.lib()
    A = torch.zeros((8, 10), dtype=torch.float64, device=DEV)
    B = torch.zeros((10, 6), dtype=torch.float64, device=DEV)
    C = torch.zeros((8, 6), dtype=torch.float64, device=DEV)
    E = torch.zeros((8, 6), dtype=torch.float64, device=DEV)
    p = lambda t: t.data_ptr()  # noqa: E731
    assert L.mm_kahan_ex(p(A), 10, p(B), 6, p(C), None, 8, 10, 6, 1, None) == -1      # ACCUMULATE needs E
    assert L.mm_kahan_ex(p(A) + 8, 10, p(B), 6, p(C), p(E), 8, 9, 6, 0, None) == -1  # A not 16-byte aligned
    assert L.mm_kahan_ex(p(A), 10, p(B), 6, p(C), p(E), 8, 10, 6, 8, None) == -1     # unknown flag
    assert L.mm_kahan_ex(p(A), 10, p(B), 6, p(A), p(E), 8, 10, 6, 0, None) == -2     # C aliases A
    assert L.mm_kahan_ex(p(A), 10, p(B), 6, p(C), p(C), 8, 10, 6, 2, None) == -2     # E aliases C
    assert L.mm_winograd_ex(p(A), 10, p(B), 6, p(C), None, None, 8, 9, 6, 2, None) == -1  # odd panel width
    assert L.mm_winograd_ex(p(A), 10, p(B), 6, p(C), None, None, 8, 10, 6, 0, None) == -1  # epilogue needs y, z
    assert L.mm_kahan_ex(p(A), 10, p(B), 6, p(C), p(E), 8, 10, 6, 2, None) == 0
    y = torch.zeros(8, dtype=torch.float64, device=DEV)
    z = torch.zeros(6, dtype=torch.float64, device=DEV)
    assert L.mm_winograd_yz(p(A), p(B), 8, 10, 6, p(A), p(z), 0, None) == -2   # y aliases A
    assert L.mm_winograd_yz(p(A), p(B), 8, 10, 6, p(y), p(y), 0, None) == -2   # z aliases y
    assert L.mm_winograd_ex(p(A), 10, p(B), 6, p(C), p(C), p(z), 8, 10, 6, 0, None) == -2  # y inside C
    assert L.mm_winograd_yz(p(A), p(B), 8, 10, 6, p(y), p(z), 0, None) == 0


def test_random_panel_splits_all_row_local_methods():
    """Seeded random k-splits (even cut points, 1-6 panels) of ragged TMA-path problems: every
    row-local method's panel composition is bitwise its one-shot product."""
    rng = np.random.default_rng(2024)
    for trial in range(12):
        N = int(rng.integers(1, 700))
        P = 2 * int(rng.integers(1, 400))
        M = 2 * int(rng.integers(1, 300))
        A, B = workload.custom(N, P, M, seed=7000 + trial)
        A = A * 10.0 ** rng.integers(-3, 4)
        dA, dB = dev(A), dev(B)
        ncut = int(rng.integers(0, min(5, P // 2 - 1) + 1)) if P > 2 else 0
        cuts = sorted(set((2 * rng.integers(1, P // 2, size=ncut)).tolist())) if ncut else []
        b = [0] + cuts + [P]
        C = torch.empty((N, M), dtype=torch.float64, device=DEV)
        E = torch.empty((N, M), dtype=torch.float64, device=DEV)
        y = torch.empty(N, dtype=torch.float64, device=DEV)
        z = torch.empty(M, dtype=torch.float64, device=DEV)
        for name in ("naive", "kahan", "kahan_fused", "winograd", "winograd_fused"):
            fused = name.endswith("_fused")
            if name.startswith("winograd"):
                mm.winograd_yz(dA, dB, y, z, fused=fused)
            for i, (k0, k1) in enumerate(zip(b[:-1], b[1:])):
                first, last = i == 0, k1 == P
                if name == "naive":
                    mm.naive_panel(dA[:, k0:k1], dB[k0:k1], C, accumulate=not first)
                elif name.startswith("kahan"):
                    mm.kahan_panel(dA[:, k0:k1], dB[k0:k1], C, E, accumulate=not first, keep_state=not last,
                                   fused=fused)
                else:
                    mm.winograd_panel(dA[:, k0:k1], dB[k0:k1], C, y, z, accumulate=not first, keep_state=not last,
                                      fused=fused)
            full = getattr(mm, name)(dA, dB)
            assert torch.equal(C, full), (trial, (N, P, M), b, name)
