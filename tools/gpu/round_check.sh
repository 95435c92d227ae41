# full round check: smoke, GPU tests, bench (plain), then the ncu round (each ncu pass after its plain run)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
[ "${NO_NCU:-0}" = 1 ] || timeout 1200 bash tools/ncu_round.sh
# summarise the ncu round here and drop two of the three --set full reports (gpurun copies back
# at most 64 MiB of gpurun_out/; the Kahan report is kept for source-level reading)
mkdir -p gpurun_out/ncu_sum
python tools/ncu_summary.py gpurun_out/ncu gpurun_out/ncu_sum > /dev/null 2>&1
python tools/hbm_table.py gpurun_out/ncu/hbm_kernels.csv > gpurun_out/ncu_sum/hbm_kernels.md 2>/dev/null
python tools/fingerprint.py summarize gpurun_out/ncu/fingerprint.csv > gpurun_out/ncu_sum/fingerprint.md 2>/dev/null
rm -f gpurun_out/ncu/full_naive.ncu-rep gpurun_out/ncu/full_winograd.ncu-rep
# the paper's section-3 experiment on the GPU (Python and plain-C clients) and the per-config table
timeout 900 python tools/paper_experiment.py --sizes 200,400,800,1600,3200,4096,8192 --json gpurun_out/paper_experiment.jsonl > gpurun_out/paper_experiment.txt 2>&1; echo paper rc=$?
./tools/mmtest -O 800 -R 10 > gpurun_out/mmtest.txt 2>&1; echo mmtest rc=$?
timeout 900 python tools/table_bench.py --reps 5 > gpurun_out/table.jsonl 2> gpurun_out/table.err; echo table rc=$?
# kernel-only (ncu) times per method call at c2 / c3
python tools/kernel_times.py run --configs c2,c3 --manifest gpurun_out/kt_manifest.json > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kt.csv \
    python tools/kernel_times.py run --configs c2,c3 --manifest gpurun_out/kt_manifest.json > /dev/null 2>&1 && \
python tools/kernel_times.py parse gpurun_out/kt.csv gpurun_out/kt_manifest.json > gpurun_out/kernel_times.jsonl; echo kt rc=$?
# per-rank schedule timing at the c4 shard shapes (modelled E_g) and BASELINE.json's c5 config on one GPU
timeout 900 python tools/shard_model.py --out gpurun_out/shard_model_c4.jsonl > gpurun_out/shard_model.log 2>&1; echo shard rc=$?
timeout 1200 python bench.py --config c5 --methods naive,strassen_winograd --levels 2 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 rc=$?
