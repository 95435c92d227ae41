import torch, json
x = torch.empty(2816*1024*1024//8, dtype=torch.float64, device="cuda")
y = torch.empty(537*1024*1024//8, dtype=torch.float64, device="cuda")
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: x.fill_(1.0)); print(json.dumps({"op": "fill 2.95 GB (write only)", "ms": round(ms, 4), "GBps": round(x.numel()*8/ms/1e6)}))
ms = t(lambda: x.zero_()); print(json.dumps({"op": "zero_ 2.95 GB", "ms": round(ms, 4), "GBps": round(x.numel()*8/ms/1e6)}))
xs = x[:y.numel()*5]
ms = t(lambda: xs.view(5, -1).copy_(y.expand(5, -1))); print(json.dumps({"op": "read 0.56 GB x5 broadcast -> write 2.8 GB", "ms": round(ms, 4), "GBps_total": round((y.numel()*8 + xs.numel()*8)/ms/1e6)}))
