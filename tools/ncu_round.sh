#!/bin/bash
# ncu evidence for a round: (1) the launch list of a short bench run, (2) one --set full capture
# of each dominant kernel, (3) DRAM bytes + duration of every HBM-bound kernel.  Each ncu command
# runs only after the identical plain command exited 0 in this same call.
set -u
OUT=gpurun_out/ncu
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$BENCH > $OUT/plain_bench.json 2> $OUT/plain_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_bench.log 2>&1
echo "launch list rc=$?"
for M in naive kahan winograd strassen_winograd; do
  QB="python tools/quick_bench.py --methods $M --reps 1 --levels 3"
  case $M in naive) K=dgemm_tma_kernel;; kahan) K=kahan_tma_kernel;; winograd) K=winograd_tma_kernel;;
             strassen_winograd) K=dgemm_tma_comb_kernel;; esac
  $QB > $OUT/plain_qb_$M.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o $OUT/full_$M $QB > $OUT/ncu_full_$M.log 2>&1
  echo "full $M rc=$?"
done
QB="python tools/quick_bench.py --methods winograd_scaled,strassen_winograd --reps 1 --levels 3"
$QB > $OUT/plain_qb_hbm.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"strassen_form|strassen_combine|line_kernel" --csv \
    --log-file $OUT/hbm_kernels.csv $QB > $OUT/ncu_hbm.log 2>&1
echo "hbm rc=$?"
# SASS instruction fingerprints of every method (DADD / DMUL / DFMA / DMMA counts)
python tools/fingerprint.py run > $OUT/plain_fp.log 2>&1 && \
ncu --metrics $(python tools/fingerprint.py metrics) --csv --log-file $OUT/fingerprint.csv \
    python tools/fingerprint.py run > $OUT/ncu_fp.log 2>&1
echo "fingerprint rc=$?"
