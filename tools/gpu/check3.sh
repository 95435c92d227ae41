set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_panels.py tests/test_gpu_fused.py -x -q > gpurun_out/pytest_new.txt 2>&1; echo new rc=$?
tail -3 gpurun_out/pytest_new.txt
timeout 600 python tools/panel_bench.py > gpurun_out/panel_bench.jsonl 2>&1; echo pb rc=$?; cat gpurun_out/panel_bench.jsonl
timeout 600 python tools/quick_bench.py --methods naive,strassen_winograd --reps 3; echo qb rc=$?
