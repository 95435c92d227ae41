# Weak r01 #7: DRAM bytes per launch of K1 / K2 / K3 against the rasterisation group height
# (tile rows per group).  Plain timing runs first, then one ncu pass per binary (dram bytes only).
set -x
mkdir -p gpurun_out/raster
mkdir -p gpurun_out/raster
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo"
$NV -o /tmp/gemm_tune tools/tune/gemm_tune.cu || exit 1
for G in 4 8 16 32; do $NV -DSIMT_GROUP_M=$G -o /tmp/simt_tune_g$G tools/tune/simt_tune.cu || exit 1; done
timeout 300 /tmp/gemm_tune g 5 > gpurun_out/raster/k1_times.jsonl 2>&1; echo k1 rc=$?
for G in 4 8 16 32; do
  timeout 300 /tmp/simt_tune_g$G x 2 > gpurun_out/raster/k3_g$G.jsonl 2>&1; echo k3 g$G rc=$?
  timeout 300 /tmp/simt_tune_g$G y 2 > gpurun_out/raster/k2_g$G.jsonl 2>&1; echo k2 g$G rc=$?
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/raster/k1_ncu.csv /tmp/gemm_tune g 1 > /dev/null 2>&1; echo ncu k1 rc=$?
for G in 4 8 16 32; do
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"tma" --log-file gpurun_out/raster/k3_g$G.csv /tmp/simt_tune_g$G x 1 > /dev/null 2>&1; echo ncu k3 g$G rc=$?
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"tma" --log-file gpurun_out/raster/k2_g$G.csv /tmp/simt_tune_g$G y 1 > /dev/null 2>&1; echo ncu k2 g$G rc=$?
done
