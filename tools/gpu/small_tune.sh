# c2 (1024^3) small-grid configurations of K1 / K2 / K3, TMA-fed (r02)
mkdir -p gpurun_out/small
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo"
$NV -o /tmp/gemm_tune tools/tune/gemm_tune.cu || exit 1
$NV -o /tmp/simt_tune tools/tune/simt_tune.cu || exit 1
timeout 300 /tmp/gemm_tune 1024 50 s > gpurun_out/small/k1_c2.jsonl 2>&1; echo k1 rc=$?
timeout 300 /tmp/simt_tune st > gpurun_out/small/simt_c2.jsonl 2>&1; echo simt rc=$?
cat gpurun_out/small/*.jsonl
