# r02: c3 odd-P TMA tile variants of K2 / K3 (simt_tune o) and K1 k-panel launches at the c4 shard
# heights (gemm_tune panel)
mkdir -p gpurun_out/shape
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo"
$NV -o /tmp/gemm_tune tools/tune/gemm_tune.cu || exit 1
$NV -o /tmp/simt_tune tools/tune/simt_tune.cu || exit 1
timeout 300 /tmp/simt_tune o > gpurun_out/shape/c3_odd.jsonl 2>&1; echo odd rc=$?
timeout 300 /tmp/gemm_tune panel > gpurun_out/shape/k1_panel.jsonl 2>&1; echo panel rc=$?
timeout 300 /tmp/simt_tune h > gpurun_out/shape/k3_shard.jsonl 2>&1; echo shard rc=$?
cat gpurun_out/shape/*.jsonl
