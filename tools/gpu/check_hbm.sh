# GPU tests + quick timing + HBM-kernel ncu metrics (each ncu pass only after its plain run exits 0)
set -x
mkdir -p gpurun_out/ncu
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.txt
QB="python tools/quick_bench.py --reps 3"
timeout 600 $QB > gpurun_out/qb.jsonl 2>&1; echo qb rc=$?; cat gpurun_out/qb.jsonl
QB1="python tools/quick_bench.py --methods winograd,winograd_scaled,strassen,strassen_winograd --reps 1"
$QB1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"strassen_form|strassen_combine|line_kernel|norm_inf|scale_copy|winograd_yz" --csv \
    --log-file gpurun_out/ncu/hbm_kernels.csv $QB1 > gpurun_out/ncu/ncu_hbm.log 2>&1
echo hbm rc=$?
