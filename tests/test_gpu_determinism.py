"""Run-to-run determinism at full size (c4, 8192^3) as a race detector for the asynchronous
pipelines: TMA-fed kernels release a shared-memory stage to the producer through an mbarrier, and
a release issued before every read of the stage has completed lets the next TMA copy overwrite
data still being read (a write-after-read race that showed up as sporadic wrong 32x32 blocks in
accumulate mode before the release was moved after the loop back edge).  Every method must give
the same bits on every repetition, and k-panel accumulation must equal the one-shot product."""
import pytest
import torch

pytestmark = pytest.mark.gpu
mm = pytest.importorskip("paper_1106_1347_b200")


@pytest.fixture(scope="module")
def ops():
    g = torch.Generator(device="cuda").manual_seed(11061347)
    A = torch.randn(8192, 8192, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(8192, 8192, dtype=torch.float64, device="cuda", generator=g)
    yield A, B
    mm.release_workspace()


@pytest.mark.parametrize("method", ["naive", "winograd", "winograd_scaled", "strassen_winograd", "kahan_fused"])
def test_repeatable_bits(ops, method):
    A, B = ops
    f = getattr(mm, method)
    ref = f(A, B)
    out = torch.empty_like(ref)
    for _ in range(4):
        f(A, B, out=out)
        assert torch.equal(out, ref), method


def test_panel_accumulation_stress(ops):
    from paper_1106_1347_b200.dist import panel_bounds

    A, B = ops
    ref = mm.naive(A, B)
    C = torch.empty_like(ref)
    for panels in (2, 3, 8, 2, 2):
        for i, (k0, k1) in enumerate(panel_bounds(8192, panels)):
            mm.naive_panel(A[:, k0:k1], B[k0:k1], C, accumulate=i > 0)
        assert torch.equal(C, ref), panels


@pytest.mark.parametrize("method", ["strassen", "strassen_winograd"])
def test_repeatable_bits_strassen_depth3(ops, method):
    """bench.py's Strassen depth: the three-level formation pass and the two-level combination."""
    A, B = ops
    f = getattr(mm, method)
    ref = f(A, B, levels=3)
    out = torch.empty_like(ref)
    for _ in range(3):
        f(A, B, out=out, levels=3)
        assert torch.equal(out, ref), method


def test_kahan_winograd_panel_stress(ops):
    """The state-carrying K2 / K3 panel steps (NEXT-4) at full size, repeated."""
    from paper_1106_1347_b200.dist import panel_bounds

    A, B = ops
    C = torch.empty(8192, 8192, dtype=torch.float64, device="cuda")
    E = torch.empty_like(C)
    y = torch.empty(8192, dtype=torch.float64, device="cuda")
    z = torch.empty(8192, dtype=torch.float64, device="cuda")
    ref_k, ref_w = mm.kahan(A, B), mm.winograd(A, B)
    mm.winograd_yz(A, B, y, z)
    for panels in (3, 4):
        b = panel_bounds(8192, panels)
        for i, (k0, k1) in enumerate(b):
            mm.kahan_panel(A[:, k0:k1], B[k0:k1], C, E, accumulate=i > 0, keep_state=k1 < 8192)
        assert torch.equal(C, ref_k), ("kahan", panels)
        for i, (k0, k1) in enumerate(b):
            mm.winograd_panel(A[:, k0:k1], B[k0:k1], C, y, z, accumulate=i > 0, keep_state=k1 < 8192)
        assert torch.equal(C, ref_w), ("winograd", panels)
