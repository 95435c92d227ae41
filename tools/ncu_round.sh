#!/bin/bash
# ncu evidence for a round: (1) the launch list of a short bench run, (2) one --set full capture
# of the dominant kernels on a short dedicated command.  Each ncu command runs only after the
# identical plain command exited 0 in this same call.
set -u
OUT=gpurun_out/ncu
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$BENCH > $OUT/plain_bench.json 2> $OUT/plain_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_bench.log 2>&1
echo "launch list rc=$?"
QB="python tools/quick_bench.py --methods naive,kahan,winograd,strassen_winograd --reps 1"
$QB > $OUT/plain_qb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dgemm_dmma|kahan_gemm|winograd_kernel|strassen_form|strassen_combine|winograd_yz" -c 8 -o $OUT/full $QB > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
