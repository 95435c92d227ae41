set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_paper.py -x -q > gpurun_out/pytest_new.txt 2>&1; echo new rc=$?
tail -5 gpurun_out/pytest_new.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python tools/quick_bench.py --reps 3 > gpurun_out/qb.jsonl 2>&1; echo qb rc=$?; cat gpurun_out/qb.jsonl
timeout 900 python tools/paper_experiment.py --sizes 200,400,800,1600,3200,4096,8192 --json gpurun_out/paper_experiment.jsonl > gpurun_out/paper_experiment.txt 2>&1; echo exp rc=$?
tail -30 gpurun_out/paper_experiment.txt
