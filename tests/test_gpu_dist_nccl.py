"""The multi-GPU driver (paper_1106_1347_b200.dist) on the real GPU stack: a one-rank NCCL process
group on cuda:0, so the broadcast (plain and the NEXT-4 panelised async one, whose work.wait()
makes the compute stream wait on NCCL's stream) and the max-all-reduce of ||A|| run through NCCL
and the local products through the C ABI.  Every method's result must equal the single-GPU call
bit for bit, both through the torch.distributed driver and through the C ABI's own NCCL layer
(mm_dist_*).  (Only one GPU is available to this test suite; world_size 2 is covered on gloo.)"""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(r"""
    import os, sys
    sys.path.insert(0, os.environ["REPO"])
    import torch, torch.distributed as dist
    import paper_1106_1347_b200 as mm
    from paper_1106_1347_b200.dist import dist_gemm
    import workload
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    A, B = workload.custom(700, 1024, 520, seed=3)
    dA = torch.from_numpy(A * 1e3).to(dev)
    hB = torch.from_numpy(B).to(dev)
    for m in ("naive", "kahan", "winograd", "winograd_scaled", "strassen", "strassen_winograd", "kahan_fused",
              "winograd_fused", "winograd_scaled_fused"):
        kw = {"levels": 2} if m.startswith("strassen") else {}
        ref = getattr(mm, m)(dA, hB, **kw)
        for panels in (1, 4, 7):
            Bw = hB.clone()
            C = dist_gemm(m, dA, Bw, levels=2, panels=panels)
            torch.cuda.synchronize()
            assert torch.equal(C, ref), (m, panels)
    # odd P: Kahan / Winograd fall back to one broadcast + the one-shot kernel (cp.async paths)
    A3, B3 = workload.custom(300, 1001, 260, seed=4)
    dA3, hB3 = torch.from_numpy(A3).to(dev), torch.from_numpy(B3).to(dev)
    for m in ("naive", "kahan", "winograd", "winograd_scaled"):
        ref = getattr(mm, m)(dA3, hB3)
        C = dist_gemm(m, dA3, hB3.clone(), panels=4)
        torch.cuda.synchronize()
        assert torch.equal(C, ref), ("odd P", m)
    # the C ABI's own layer (mm_dist_*): NCCL driven from libmm_b200.so
    from paper_1106_1347_b200.dist import NativeComm
    comm = NativeComm()
    for m in ("naive", "kahan", "winograd", "winograd_scaled", "strassen", "strassen_winograd",
              "kahan_fused", "winograd_fused", "winograd_scaled_fused"):
        kw = {"levels": 2} if m.startswith("strassen") else {}
        ref = getattr(mm, m)(dA, hB, **kw)
        for panels in (1, 3, 8):
            Bw = hB.clone()
            C = comm.gemm(m, dA, Bw, levels=2, panels=panels)
            torch.cuda.synchronize()
            assert torch.equal(C, ref), ("native", m, panels)
            assert torch.equal(Bw, hB)
    for m in ("naive", "kahan", "winograd", "kahan_fused", "winograd_fused"):
        ref = getattr(mm, m)(dA3, hB3)
        C = comm.gemm(m, dA3, hB3.clone(), panels=5)
        torch.cuda.synchronize()
        assert torch.equal(C, ref), ("native odd P", m)
    # a rank without rows still takes part (the product is empty)
    C0 = comm.gemm("winograd_scaled", dA[:0], hB.clone())
    torch.cuda.synchronize()
    assert C0.shape == (0, hB.shape[1])
    # the alternative partition (Strassen's seven products on the ranks): all seven on this rank,
    # through the torch.distributed driver and through mm_dist_strassen7; padded shapes included
    from paper_1106_1347_b200.dist import strassen7
    for (n, p_, m_) in ((700, 1024, 520), (300, 1001, 260)):
        X, Y = workload.custom(n, p_, m_, seed=n + p_)
        dX, dY = torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev)
        for m in ("strassen", "strassen_winograd"):
            for lv in (1, 2, 3):
                ref = getattr(mm, m)(dX, dY, levels=lv)
                C = strassen7(m, dX.clone(), dY.clone(), levels=lv)
                C2 = comm.strassen7(m, dX.clone(), dY.clone(), levels=lv)
                torch.cuda.synchronize()
                assert torch.equal(C, ref), ("s7 torch", m, lv, n)
                assert torch.equal(C2, ref), ("s7 native", m, lv, n)
    comm.close()
    dist.destroy_process_group()
    print("nccl world-1 ok")
""")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dist_gemm_over_nccl_one_rank():
    env = dict(os.environ, REPO=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "nccl world-1 ok" in r.stdout
