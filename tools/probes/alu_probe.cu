// FP64 SIMT throughput probe (sm_100a): separately rounded DADD and DMUL, and DFMA, with enough
// independent chains per thread that latency cannot limit issue -- the measured ceiling of the
// "alu" roofline the Kahan and Winograd kernels are reported against (the
// derived figure is 148 SMs x 64 lanes x 1.965 GHz = 18.61 T op/s).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_probe alu_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int OP, int NACC>
__global__ void __launch_bounds__(256) k_alu(double* out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      if (OP == 0) acc[i] = __dadd_rn(acc[i], a);
      else if (OP == 1) acc[i] = __dmul_rn(acc[i], a);
      else acc[i] = __fma_rn(acc[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int OP, int NACC>
void run(const char* name, double* out, int sms, int blocks_per_sm, int threads) {
  const int iters = 4096;
  dim3 grid(sms * blocks_per_sm);
  k_alu<OP, NACC><<<grid, threads>>>(out, 16, 1.0000001, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_alu<OP, NACC><<<grid, threads>>>(out, iters, 1.0000001, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 5.0 * double(grid.x) * threads * iters * NACC;
  printf("{\"probe\":\"alu\",\"op\":\"%s\",\"nacc\":%d,\"threads\":%d,\"blocks_per_sm\":%d,\"T_inst_per_s\":%.3f,\"err\":\"%s\"}\n",
         name, NACC, threads, blocks_per_sm, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int bps : {2, 4, 8}) {
    run<0, 16>("dadd", out, sms, bps, 256);
    run<1, 16>("dmul", out, sms, bps, 256);
    run<2, 16>("dfma", out, sms, bps, 256);
  }
  run<0, 32>("dadd", out, sms, 4, 256);
  run<2, 32>("dfma", out, sms, 4, 256);
  return 0;
}
