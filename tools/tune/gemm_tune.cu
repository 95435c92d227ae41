// gemm_tune.cu -- development harness: times alternative K1 tile configurations on B200 and
// checks they are bitwise identical (they all walk k in the same order).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gemm_tune gemm_tune.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_1106_1347_b200/csrc/gemm_tma.cuh"

using namespace mmk;

__global__ void fill(double* x, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[i] = double(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
  }
}

__global__ void cmp(const double* a, const double* b, int64_t n, unsigned long long* bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    if (a[i] != b[i]) atomicAdd(bad, 1ull);
}

template <class CF, bool TMA = false>
void run(const char* name, const double* A, const double* B, double* C, const double* Cref, int64_t n, int reps,
         unsigned long long* bad) {
  GemmProblem pr{A, B, C, n, n, n, n, n, n, 0, 0, 0, 1};
  cudaMemset(C, 0, n * n * 8);
  auto go = [&]() { return TMA ? launch_dgemm_tma<CF>(pr, 0) : launch_dgemm_cfg<CF>(pr, 0); };
  if (go() != cudaSuccess) {
    printf("{\"cfg\":\"%s\",\"error\":\"%s\"}\n", name, cudaGetErrorString(cudaGetLastError()));
    return;
  }
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  unsigned long long nb = 0;
  if (Cref) {
    cudaMemset(bad, 0, 8);
    cmp<<<1024, 256>>>(C, Cref, n * n, bad);
    cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"cfg\":\"%s\",\"n\":%lld,\"threads\":%d,\"smem\":%zu,\"ms\":%.3f,\"tflops\":%.2f,\"mismatch\":%llu,\"err\":\"%s\"}\n",
         name, (long long)n, CF::THREADS, CF::SMEM, ms, 2.0 * n * n * n / ms / 1e9, nb, cudaGetErrorString(err));
  fflush(stdout);
}

// rectangular problem N x P x M through a given path (config c3 is 4096 x 1001 x 3000)
template <class CF, bool TMA>
void run_rect(const char* name, const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
              int reps) {
  GemmProblem pr{A, B, C, N, P, M, P, M, M, 0, 0, 0, 1};
  auto go = [&]() { return TMA ? launch_dgemm_tma<CF>(pr, 0) : launch_dgemm_cfg<CF>(pr, 0); };
  go();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("{\"cfg\":\"%s\",\"N\":%lld,\"P\":%lld,\"M\":%lld,\"ms\":%.4f,\"tflops\":%.2f,\"err\":\"%s\"}\n", name,
         (long long)N, (long long)P, (long long)M, ms, 2.0 * N * P * M / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "panel") {  // k-panel launches of the g = 2 / 4 / 8 c4 shards (r02)
    double *A, *B, *C;
    cudaMalloc(&A, 4096ll * 1024 * 8);
    cudaMalloc(&B, 1024ll * 8192 * 8);
    cudaMalloc(&C, 4096ll * 8192 * 8);
    fill<<<1024, 256>>>(A, 4096ll * 1024, 1);
    fill<<<1024, 256>>>(B, 1024ll * 8192, 2);
    for (int64_t rows : {1024, 2048, 4096}) {
      run_rect<GemmCfg<64, 64, 2, 2, 2, 3, 32>, true>("tma_64x64_s2_3cta_bk32", A, B, C, rows, 1024, 8192, 20);
      run_rect<GemmCfg<64, 64, 2, 2, 2, 2, 32>, true>("tma_64x64_s2_2cta_bk32", A, B, C, rows, 1024, 8192, 20);
      run_rect<GemmCfg<64, 64, 2, 2, 3, 2, 32>, true>("tma_64x64_s3_2cta_bk32", A, B, C, rows, 1024, 8192, 20);
      run_rect<GemmCfg<64, 32, 2, 1, 4, 6, 16>, true>("tma_64x32_s4_6cta_bk16", A, B, C, rows, 1024, 8192, 20);
      run_rect<GemmCfg<128, 64, 2, 2, 3, 2, 32>, true>("tma_128x64_s3_2cta_bk32", A, B, C, rows, 1024, 8192, 20);
    }
    return 0;
  }
  if (argc > 1 && std::string(argv[1]) == "c3") {
    double *A, *B, *C;
    cudaMalloc(&A, 4096 * 1002 * 8);
    cudaMalloc(&B, 1002 * 3000 * 8);
    cudaMalloc(&C, 4096 * 3000 * 8);
    fill<<<1024, 256>>>(A, 4096 * 1002, 1);
    fill<<<1024, 256>>>(B, 1002 * 3000, 2);
    run_rect<GemmCfg<128, 64, 2, 2, 4, 2>, false>("cpasync_128x64_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 4>, false>("cpasync_64x64_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 2, 3, 32>, false>("cpasync_64x64_s2_3cta_bk32_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 3, 2, 32>, false>("cpasync_64x64_s3_2cta_bk32_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 3, 3, 16>, false>("cpasync_64x64_s3_3cta_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 5, 3, 16>, false>("cpasync_64x64_s5_3cta_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 3, 16>, false>("cpasync_64x64_s4_3cta_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 2, 3, 16>, false>("cpasync_64x64_s2_3cta_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 32, 2, 1, 4, 6>, false>("cpasync_64x32_w2x1_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<32, 64, 1, 2, 4, 6>, false>("cpasync_32x64_w1x2_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 3, 4>, false>("cpasync_64x64_s3_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 4, 32>, false>("cpasync_64x64_bk32_P1001", A, B, C, 4096, 1001, 3000, 20);
    run_rect<GemmCfg<128, 64, 2, 2, 4, 2>, false>("cpasync_128x64_P1000", A, B, C, 4096, 1000, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 3>, true>("tma_64x64_P1000", A, B, C, 4096, 1000, 3000, 20);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 3>, true>("tma_64x64_P1002", A, B, C, 4096, 1002, 3000, 20);
    double *A2, *B2, *C2;
    cudaMalloc(&A2, 8192ll * 8192 * 8);
    cudaMalloc(&B2, 8192ll * 8192 * 8);
    cudaMalloc(&C2, 8192ll * 8192 * 8);
    fill<<<1024, 256>>>(A2, 8192ll * 8192, 1);
    fill<<<1024, 256>>>(B2, 8192ll * 8192, 2);
    run_rect<GemmCfg<128, 64, 2, 2, 4, 2>, false>("cpasync_128x64_P8191", A2, B2, C2, 8192, 8191, 8192, 3);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 4>, false>("cpasync_64x64_P8191", A2, B2, C2, 8192, 8191, 8192, 3);
    run_rect<GemmCfg<64, 64, 2, 2, 2, 3, 32>, false>("cpasync_64x64_s2_3cta_bk32_P8191", A2, B2, C2, 8192, 8191, 8192, 3);
    run_rect<GemmCfg<64, 64, 2, 2, 3, 2, 32>, false>("cpasync_64x64_s3_2cta_bk32_P8191", A2, B2, C2, 8192, 8191, 8192, 3);
    run_rect<GemmCfg<64, 64, 2, 2, 3, 3, 16>, false>("cpasync_64x64_s3_3cta_P8191", A2, B2, C2, 8192, 8191, 8192, 3);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 3, 16>, false>("cpasync_64x64_s4_3cta_P8191", A2, B2, C2, 8192, 8191, 8192, 3);
    run_rect<GemmCfg<64, 64, 2, 2, 3, 3, 16>, false>("cpasync_64x64_s3_3cta_2048_P2047", A2, B2, C2, 2048, 2047, 2048, 10);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 3, 16>, false>("cpasync_64x64_s4_3cta_2048_P2047", A2, B2, C2, 2048, 2047, 2048, 10);
    run_rect<GemmCfg<64, 64, 2, 2, 3, 4>, false>("cpasync_64x64_s3_P8191", A2, B2, C2, 8192, 8191, 8192, 3);
    run_rect<GemmCfg<128, 64, 2, 2, 4, 2>, false>("cpasync_128x64_2048_P2047", A2, B2, C2, 2048, 2047, 2048, 10);
    run_rect<GemmCfg<64, 64, 2, 2, 4, 4>, false>("cpasync_64x64_2048_P2047", A2, B2, C2, 2048, 2047, 2048, 10);
    return 0;
  }
  const bool raster = argc > 1 && argv[1][0] == 'g';  // production K1 with GROUP_M varied (L2 reuse / DRAM bytes)
  int64_t n = argc > 1 && !raster ? atoll(argv[1]) : 8192;
  int reps = argc > 2 ? atoi(argv[2]) : 3;
  double *A, *B, *C, *R;
  unsigned long long* bad;
  cudaMalloc(&A, n * n * 8);
  cudaMalloc(&B, n * n * 8);
  cudaMalloc(&C, n * n * 8);
  cudaMalloc(&R, n * n * 8);
  cudaMalloc(&bad, 8);
  fill<<<1024, 256>>>(A, n * n, 1);
  fill<<<1024, 256>>>(B, n * n, 2);
  run<GemmCfg<64, 64, 2, 2, 2, 3, 32>, true>("tma_64x64_s2_3cta_bk32", A, B, R, nullptr, n, reps, bad);
  if (n == 1024 && argc > 3) {  // "1024 <reps> s": small-grid TMA configurations at 1024^3 (r02)
    run<GemmCfg<64, 32, 2, 1, 4, 6, 16>, true>("tma_64x32_w2x1_s4_6cta_bk16", A, B, C, R, n, reps, bad);
    run<GemmCfg<32, 32, 1, 1, 2, 8, 32>, true>("tma_32x32_w1_s2_8cta_bk32", A, B, C, R, n, reps, bad);
    run<GemmCfg<32, 32, 1, 1, 3, 8, 32>, true>("tma_32x32_w1_s3_8cta_bk32", A, B, C, R, n, reps, bad);
    run<GemmCfg<32, 32, 1, 1, 4, 8, 16>, true>("tma_32x32_w1_s4_8cta_bk16", A, B, C, R, n, reps, bad);
    run<GemmCfg<32, 64, 1, 2, 3, 6, 32>, true>("tma_32x64_w1x2_s3_6cta_bk32", A, B, C, R, n, reps, bad);
    run<GemmCfg<64, 32, 2, 1, 3, 6, 32>, true>("tma_64x32_w2x1_s3_6cta_bk32", A, B, C, R, n, reps, bad);
    run<GemmCfg<32, 32, 1, 1, 2, 12, 32>, true>("tma_32x32_w1_s2_12cta_bk32", A, B, C, R, n, reps, bad);
    return 0;
  }
  if (raster) {
    run<GemmCfg<64, 64, 2, 2, 2, 3, 32, 4>, true>("tma_64x64_group4", A, B, C, R, n, reps, bad);
    run<GemmCfg<64, 64, 2, 2, 2, 3, 32, 8>, true>("tma_64x64_group8", A, B, C, R, n, reps, bad);
    run<GemmCfg<64, 64, 2, 2, 2, 3, 32, 16>, true>("tma_64x64_group16", A, B, C, R, n, reps, bad);
    run<GemmCfg<64, 64, 2, 2, 2, 3, 32, 24>, true>("tma_64x64_group24", A, B, C, R, n, reps, bad);
    run<GemmCfg<64, 64, 2, 2, 2, 3, 32, 32>, true>("tma_64x64_group32", A, B, C, R, n, reps, bad);
    return 0;
  }
  run<GemmCfg<64, 64, 2, 2, 2, 2, 32>, true>("tma_64x64_s2_2cta_bk32", A, B, C, R, n, reps, bad);
  run<GemmCfg<64, 64, 2, 2, 3, 2, 32>, true>("tma_64x64_s3_2cta_bk32", A, B, C, R, n, reps, bad);
  run<GemmCfg<128, 64, 4, 2, 2, 2, 32>, true>("tma_128x64_w4x2_s2_2cta_bk32", A, B, C, R, n, reps, bad);
  return 0;
}
