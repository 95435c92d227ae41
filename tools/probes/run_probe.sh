#!/bin/bash
# Runs the FP64 probes on a B200 box; outputs under gpurun_out/probe/
set -x
mkdir -p gpurun_out/probe
nvidia-smi > gpurun_out/probe/nvidia-smi.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/probe/clocks.csv &
SMI=$!
./tools/probes/fp64_probe > gpurun_out/probe/fp64_probe.jsonl 2>&1
python - <<'PY' > gpurun_out/probe/torch_dgemm.txt 2>&1
import torch, time
for n in (1024, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device='cuda'); b = torch.randn(n, n, dtype=torch.float64, device='cuda')
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"torch.matmul f64 n={n}: {ms:.3f} ms, {2*n**3/ms/1e9:.2f} TFLOP/s")
PY
kill $SMI
lscpu > gpurun_out/probe/lscpu.txt 2>&1
python -c "import os; print(os.cpu_count(), len(os.sched_getaffinity(0)))" >> gpurun_out/probe/lscpu.txt
free -g >> gpurun_out/probe/lscpu.txt
