// FP64 latency probe (sm_100a): one warp, NACC independent dependent chains of DADD / DMUL / DFMA,
// cycles per chain step from clock64 -- NACC = 1 is the dependent latency the order-faithful line
// sums (one chain of P DADDs per line, lines.cuh) and the Winograd / Kahan term chains pay; larger
// NACC shows how many independent chains one warp needs to reach the issue limit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int OP, int NACC>
__global__ void k_lat(double* out, long long* cyc, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      if (OP == 0) acc[i] = __dadd_rn(acc[i], a);
      else if (OP == 1) acc[i] = __dmul_rn(acc[i], a);
      else acc[i] = __fma_rn(acc[i], a, b);
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP, int NACC>
void run(const char* name, double* out, long long* cyc) {
  const int iters = 1 << 14;
  k_lat<OP, NACC><<<1, 32>>>(out, cyc, 64, 1.0000001, 1e-7);
  k_lat<OP, NACC><<<1, 32>>>(out, cyc, iters, 1.0000001, 1e-7);
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("{\"op\": \"%s\", \"chains_per_thread\": %d, \"warps\": 1, \"cycles_per_step\": %.2f, "
         "\"cycles_per_op\": %.2f}\n",
         name, NACC, double(c) / iters, double(c) / iters / NACC);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  run<0, 1>("dadd", out, cyc);
  run<1, 1>("dmul", out, cyc);
  run<2, 1>("dfma", out, cyc);
  run<0, 2>("dadd", out, cyc);
  run<0, 4>("dadd", out, cyc);
  run<0, 8>("dadd", out, cyc);
  run<0, 16>("dadd", out, cyc);
  run<0, 32>("dadd", out, cyc);
  return 0;
}
