"""The evaluation-order golden cases (tests/golden/order_cases.txt) through the C ABI.

The kernels are checked bitwise against the oracle elsewhere; these cases check them directly
against the hand-derived values the paper's order gives (Kahan's k loop; (Sum - y) - z,
P:189; the infinity-norm row sum; the Strassen / Strassen-Winograd block sums, P:279-282,
P:308-311), so an order mistake shared by kernel and oracle cannot pass.
"""
import numpy as np
import pytest
import torch

from tests.test_oracle_order_pins import CASES

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_1106_1347_b200")
DEV = torch.device("cuda", 0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("fn", ["kahan", "kahan_fused"])
def test_kahan_k_order(fn):
    _, A, B, want = CASES["O1"]
    assert host(getattr(mm, fn)(dev(A), dev(B)))[0, 0] == want


def test_kahan_panels_k_order():
    # the panel kernels need 16-byte aligned operands with even pitches: O1's row with a trailing
    # zero term (err -1/2 + 0; t = (2^53 + 2) - 1/2 rounds back to 2^53 + 2) times a 4 x 2 ones matrix
    _, A, B, want = CASES["O1"]
    A4 = np.concatenate([A, np.zeros((1, 1))], axis=1)
    dA, dB = dev(A4), dev(np.ones((4, 2)))
    C = torch.zeros((1, 2), dtype=torch.float64, device=DEV)
    E = torch.zeros((1, 2), dtype=torch.float64, device=DEV)
    mm.kahan_panel(dA[:, :2], dB[:2], C, E, accumulate=False, keep_state=True)
    mm.kahan_panel(dA[:, 2:], dB[2:], C, E, accumulate=True, keep_state=False)
    assert host(C).tolist() == [[want, want]]


@pytest.mark.parametrize("fn", ["winograd", "winograd_fused"])
def test_winograd_sum_minus_y_minus_z(fn):
    _, A, B, want = CASES["O2"]
    assert host(getattr(mm, fn)(dev(A), dev(B)))[0, 0] == want


@pytest.mark.parametrize("fn", ["winograd_scaled", "winograd_scaled_fused"])
def test_winograd_scaled_sum_minus_y_minus_z(fn):
    _, A, B, want = CASES["O2s"]
    C, lam = getattr(mm, fn)(dev(A), dev(B), return_lambda=True)
    assert lam == 0
    assert np.array_equal(host(C), want)


def test_norm_inf_row_left_to_right():
    _, X, _, want = CASES["O3"]
    assert mm.norm_inf(dev(X)).item() == want


@pytest.mark.parametrize("cid,fn", [("O4", "strassen"), ("O5", "strassen_winograd")])
def test_strassen_combination_left_to_right(cid, fn):
    # the library pads every dimension to a multiple of 2^(levels+1) (reading R10), so a 2 x 2 input
    # would sit in one quadrant; the 4 x 4 Kronecker copy with 2 x 2 constant blocks keeps the case:
    # each quadrant is one scalar of the case, each leaf product a 2-term chain = 2 x (the scalar
    # product), exact, and the doubled combination rounds exactly as the undoubled one.
    _, A, B, want = CASES[cid]
    one = np.ones((2, 2))
    C = host(getattr(mm, fn)(dev(np.kron(A, one)), dev(np.kron(B, one)), levels=1))
    assert np.array_equal(C, 2.0 * np.kron(want, one))
