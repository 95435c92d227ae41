"""GraphedProduct: a product captured once into a CUDA graph and replayed (launch-bound small
sizes).  Replays are bitwise the direct call, follow in-place updates of the inputs, and keep
working after other calls resized the shared workspace."""
import numpy as np
import pytest
import torch

import oracle
import workload

pytestmark = pytest.mark.gpu
mm = pytest.importorskip("paper_1106_1347_b200")


@pytest.mark.parametrize("method,levels", [("naive", 0), ("kahan", 0), ("winograd", 0), ("winograd_scaled", 0),
                                           ("strassen", 2), ("strassen_winograd", 2), ("strassen", 3),
                                           ("strassen_winograd", 3), ("kahan_fused", 0), ("winograd_fused", 0)])
def test_graph_replay_bitwise(method, levels):
    A, B = workload.custom(130, 98, 120, seed=4)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    kw = {"levels": levels} if method.startswith("strassen") else {}
    direct = getattr(mm, method)(dA, dB, **kw).clone()
    g = mm.GraphedProduct(method, dA, dB, **kw)
    assert torch.equal(g.replay(), direct)
    # new inputs in place -> the replay computes the new product
    A2, B2 = workload.custom(130, 98, 120, seed=5)
    dA.copy_(torch.from_numpy(A2))
    dB.copy_(torch.from_numpy(B2))
    big = mm.naive(torch.ones(2048, 2048, dtype=torch.float64, device="cuda"),
                   torch.ones(2048, 2048, dtype=torch.float64, device="cuda"))  # churn the allocator
    mm.release_workspace()
    del big
    got = g.replay().cpu().numpy()
    ref = getattr(mm, method)(dA, dB, **kw).cpu().numpy()
    assert np.array_equal(got, ref)
    if method == "naive":
        assert np.array_equal(got, oracle.naive_fma(A2, B2))
