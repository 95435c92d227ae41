# GPU tests + quick c4 timing of every method (+ optional per-config table)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.txt | grep -v "^  "
timeout 600 python tools/quick_bench.py --reps 3 > gpurun_out/qb.jsonl 2>&1; echo qb rc=$?; cat gpurun_out/qb.jsonl
[ "${TABLE:-0}" = 1 ] && timeout 900 python tools/table_bench.py --reps 5 > gpurun_out/table.jsonl 2>&1; echo table rc=$?
