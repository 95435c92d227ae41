# NVLS multicast probe (tools/probes/mc_probe.cu) on one GPU
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mc_probe tools/probes/mc_probe.cu -lcuda || exit 1
timeout 120 /tmp/mc_probe > gpurun_out/mc_probe.jsonl 2>&1; echo mc rc=$?; cat gpurun_out/mc_probe.jsonl
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; nvidia-smi -q | grep -i -A3 "fabric\|nvlink" | head -40 >> gpurun_out/topo.txt
