import os, sys, json, torch, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1106_1347_b200 as mm, oracle, workload
dev = torch.device("cuda", 0)
# correctness vs the oracle (bitwise), several shapes / depths incl. ragged and padding
for (N, P, M, lv) in [(256, 256, 256, 1), (256, 256, 256, 2), (300, 200, 260, 2), (520, 384, 130, 3), (1024, 1024, 1024, 3), (67, 45, 53, 2)]:
    A, B = workload.custom(N, P, M, seed=N + lv)
    C = mm.strassen_winograd(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), levels=lv).cpu().numpy()
    d, pad = oracle.plan(N, P, M, lv)
    R = oracle.strassen(1, A, B, levels=d, pad=pad, base=oracle.BASE_FMA)
    print(json.dumps({"shape": [N, P, M], "levels": lv, "bitwise": bool(np.array_equal(C, R)), "maxdiff": float(np.abs(C - R).max())}), flush=True)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(8192, 8192, dtype=torch.float64, device=dev, generator=g)
B = torch.randn(8192, 8192, dtype=torch.float64, device=dev, generator=g)
Cref = None
for lv in (2, 3):
    C = torch.empty(8192, 8192, dtype=torch.float64, device=dev)
    mm.strassen_winograd(A, B, out=C, levels=lv)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); mm.strassen_winograd(A, B, out=C, levels=lv); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"fused": os.environ.get("MM_STRASSEN_FUSED_COMBINE", "0"), "levels": lv, "ms": sorted(ts)[2], "checksum": float(C.double().sum().item())}), flush=True)
