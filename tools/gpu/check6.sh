set -x
mkdir -p gpurun_out/ncu
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "matmul" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['ms_per_step'], d['e2e'])"
QB="python tools/quick_bench.py --methods winograd --reps 1"
$QB > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:winograd_tma_kernel -c 1 -o gpurun_out/ncu/full_winograd $QB > gpurun_out/ncu/ncu_full_winograd.log 2>&1; echo ncu rc=$?
