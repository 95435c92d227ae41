set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paper.py -x -q > gpurun_out/pytest_paper.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_paper.txt
timeout 900 python tools/paper_experiment.py --sizes 200,400,800,1600,3200,8192 --json gpurun_out/paper_experiment.jsonl > gpurun_out/paper_experiment.txt 2>&1; echo exp rc=$?
cat gpurun_out/paper_experiment.txt
