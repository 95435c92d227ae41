set -x
mkdir -p gpurun_out
timeout 300 python tools/gpu/pdbg.py 2>&1 | grep -c mismatch
timeout 300 python tools/panel_bench.py
timeout 600 python tools/quick_bench.py --reps 3 > gpurun_out/qb.jsonl 2>&1; echo qb rc=$?; cat gpurun_out/qb.jsonl
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.txt
