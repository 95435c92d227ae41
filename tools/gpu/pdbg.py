import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1106_1347_b200 as mm
from paper_1106_1347_b200.dist import panel_bounds
n = 8192
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
B = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
ref = mm.naive(A, B)
P1 = torch.empty_like(ref); P2 = torch.empty_like(ref)
mm.naive_panel(A[:, :4096], B[:4096], P1, accumulate=False)
mm.naive_panel(A[:, 4096:], B[4096:], P2, accumulate=False)
C = torch.empty(n, n, dtype=torch.float64, device="cuda")
for it in range(12):
    C.fill_(float(it + 1) * 1000.0)
    mm.naive_panel(A[:, :4096], B[:4096], C, accumulate=False)
    torch.cuda.synchronize()
    n1 = int((C != P1).sum())
    mm.naive_panel(A[:, 4096:], B[4096:], C, accumulate=True)
    torch.cuda.synchronize()
    bad = (C != ref); nb = int(bad.sum())
    print("it", it, "after panel1 mismatches vs P1:", n1, "final mismatches:", nb, flush=True)
    if nb:
        idx = bad.nonzero()[:3].tolist()
        for i, j in idx:
            print("   ", i, j, "C", float(C[i, j]), "ref", float(ref[i, j]), "P1", float(P1[i, j]), "P2", float(P2[i, j]),
                  "C-ref", float(C[i, j] - ref[i, j]), "C-P2", float(C[i, j] - P2[i, j]), flush=True)
