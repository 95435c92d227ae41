// simt_tune.cu -- development harness: times alternative tile configurations of the FP64
// SIMT kernels (K2 Kahan, K3 Winograd) on B200 and checks that each is bitwise identical to
// the first (every configuration walks k / j in the same order per entry).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o simt_tune simt_tune.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_1106_1347_b200/csrc/kahan.cuh"
#include "../../paper_1106_1347_b200/csrc/winograd.cuh"

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

struct Ctx {
  double *A, *B, *C, *R, *y, *z;
  unsigned long long* bad;
  int64_t n;
  int reps;
};

template <class F>
void timeit(const char* kind, const char* name, int threads, size_t smem, Ctx& c, const double* ref, F f,
            double ops_per_entry_k) {
  cudaMemset(c.C, 0, c.n * c.n * 8);
  f();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < c.reps; ++r) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= c.reps;
  unsigned long long nb = 0;
  if (ref) {
    cudaMemset(c.bad, 0, 8);
    cmp<<<1024, 256>>>(c.C, ref, c.n * c.n, c.bad);
    cudaMemcpy(&nb, c.bad, 8, cudaMemcpyDeviceToHost);
  }
  const double n = double(c.n);
  printf("{\"kernel\":\"%s\",\"cfg\":\"%s\",\"n\":%lld,\"threads\":%d,\"smem\":%zu,\"ms\":%.3f,\"gflops_2npm\":%.1f,"
         "\"fp64_op_rate_T\":%.3f,\"mismatch\":%llu,\"err\":\"%s\"}\n",
         kind, name, (long long)c.n, threads, smem, ms, 2 * n * n * n / ms / 1e6, ops_per_entry_k * n * n * n / ms / 1e9,
         nb, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

template <class CF>
void kahan(const char* name, Ctx& c, bool first) {
  if (first) cudaMemset(c.R, 0, c.n * c.n * 8);
  timeit("kahan", name, CF::THREADS, CF::SMEM, c, first ? nullptr : c.R,
         [&] { launch_kahan<CF>(c.A, c.B, c.C, c.n, c.n, c.n, 0); }, 5.0);
  if (first) cudaMemcpy(c.R, c.C, c.n * c.n * 8, cudaMemcpyDeviceToDevice);
}

template <class CF>
void wino(const char* name, Ctx& c, bool first) {
  timeit("winograd", name, CF::THREADS, CF::SMEM, c, first ? nullptr : c.R,
         [&] { launch_winograd<CF>(c.A, c.B, c.C, c.y, c.z, c.n, c.n, c.n, 0); }, 2.0);
  if (first) cudaMemcpy(c.R, c.C, c.n * c.n * 8, cudaMemcpyDeviceToDevice);
}

template <class CF>
void kahan_tma(const char* name, Ctx& c) {
  timeit("kahan", name, CF::THREADS, SimtTmaLayout<CF>::SMEM, c, c.R,
         [&] { launch_kahan_tma<CF>(c.A, c.B, c.C, c.n, c.n, c.n, 0); }, 5.0);
}
template <class CF>
void wino_tma(const char* name, Ctx& c) {
  timeit("winograd", name, CF::THREADS, SimtTmaLayout<CF>::SMEM, c, c.R, [&] {
    launch_yz(c.A, c.B, c.y, c.z, c.n, c.n, c.n, nullptr, nullptr, nullptr, nullptr, nullptr, 0);
    launch_winograd_pairs_tma<CF, false>(c.A, c.B, c.C, c.y, c.z, c.n, c.n, c.n, 0);
  }, 2.0);
}
// c3-shaped rectangular runs (odd P = 1001: cp.async paths)
template <class CF>
void rect(const char* kind, const char* name, const double* A, const double* B, double* C, double* y, double* z,
          int64_t N, int64_t P, int64_t M) {
  auto go = [&]() {
    if (kind[0] == 'k') launch_kahan<CF>(A, B, C, N, P, M, 0);
    else launch_winograd<CF>(A, B, C, y, z, N, P, M, 0);
  };
  go();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"kernel\":\"%s\",\"cfg\":\"%s\",\"N\":%lld,\"P\":%lld,\"M\":%lld,\"ms\":%.4f,\"err\":\"%s\"}\n", kind,
         name, (long long)N, (long long)P, (long long)M, ms / 10, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

// c3 after the odd-P repack (A at the even pitch P + 1 = 1002): TMA-fed K2 / K3 tile variants, each
// compared bitwise with the first of its kind (r02)
struct OddCtx {
  double *A, *B, *C, *R, *y, *z;
  unsigned long long* bad;
  bool have_ref = false;
};
template <class F>
void odd_time(const char* kind, const char* name, OddCtx& c, F f) {
  const int64_t N = 4096, M = 3000;
  cudaMemset(c.C, 0, N * M * 8);
  f();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long nb = 0;
  if (c.have_ref) {
    cudaMemset(c.bad, 0, 8);
    cmp<<<1024, 256>>>(c.C, c.R, N * M, c.bad);
    cudaMemcpy(&nb, c.bad, 8, cudaMemcpyDeviceToHost);
  } else {
    cudaMemcpy(c.R, c.C, N * M * 8, cudaMemcpyDeviceToDevice);
    c.have_ref = true;
  }
  printf("{\"kernel\":\"%s\",\"cfg\":\"%s\",\"N\":4096,\"P\":1001,\"M\":3000,\"ms\":%.4f,\"mismatch\":%llu,"
         "\"err\":\"%s\"}\n",
         kind, name, ms / 20, nb, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}
template <class CF>
void odd_wino(const char* name, OddCtx& c) {
  odd_time("winograd", name, c, [&] {
    launch_winograd_pairs_tma_odd<CF, false>(c.A, 1002, c.B, 3000, c.C, c.y, c.z, 4096, 1001, 3000, 0);
  });
}
template <class CF>
void odd_kahan(const char* name, OddCtx& c) {
  odd_time("kahan", name, c, [&] {
    launch_kahan_tma_ex<CF, false>(c.A, 1002, c.B, 3000, c.C, nullptr, 4096, 1001, 3000, 0, 0);
  });
}

// K3 at the c4 shard heights of the g-GPU row partition (rows x 8192 x 8192), r02
template <class CF>
void shard_wino(const char* name, Ctx& c, int64_t rows, bool first) {
  const int64_t n = c.n;
  cudaMemset(c.C, 0, rows * n * 8);
  auto go = [&] { launch_winograd_pairs_tma<CF, false>(c.A, c.B, c.C, c.y, c.z, rows, n, n, 0); };
  go();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < c.reps; ++r) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long nb = 0;
  if (first) {
    cudaMemcpy(c.R, c.C, rows * n * 8, cudaMemcpyDeviceToDevice);
  } else {
    cudaMemset(c.bad, 0, 8);
    cmp<<<1024, 256>>>(c.C, c.R, rows * n, c.bad);
    cudaMemcpy(&nb, c.bad, 8, cudaMemcpyDeviceToHost);
  }
  printf("{\"kernel\":\"winograd\",\"cfg\":\"%s\",\"N\":%lld,\"P\":%lld,\"M\":%lld,\"ms\":%.4f,"
         "\"fp64_op_rate_T\":%.3f,\"mismatch\":%llu,\"err\":\"%s\"}\n",
         name, (long long)rows, (long long)n, (long long)n, ms / c.reps, 2.0 * rows * n * n / (ms / c.reps) / 1e9, nb,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

// the g = 8 c4 Winograd panel schedule on one GPU: 1024 rows, four 2048-deep k-panels accumulated
// with mm_winograd_ex's flags (compile with -DMMK_WINO_UNROLL=2 / 8 to compare unrolls), r02
void panel_wino(Ctx& c, int64_t rows, int np) {
  const int64_t n = c.n, kp = n / np;
  auto go = [&] {
    for (int i = 0; i < np; ++i) {
      const int f = (i > 0 ? SIMT_EX_ACC : 0) | (i < np - 1 ? SIMT_EX_KEEP : 0);
      launch_winograd_tma_ex<WinogradTma, false>(c.A + i * kp, n, c.B + i * kp * n, n, c.C, c.y, c.z, rows, kp, n, f,
                                                 0);
    }
  };
  go();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < c.reps; ++r) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"kernel\":\"winograd_panels\",\"unroll\":%d,\"rows\":%lld,\"panels\":%d,\"ms\":%.4f,\"err\":\"%s\"}\n",
         kWinoUnroll, (long long)rows, np, ms / c.reps, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

void panel_kahan(Ctx& c, double* E, int64_t rows, int np) {
  const int64_t n = c.n, kp = n / np;
  auto go = [&] {
    for (int i = 0; i < np; ++i) {
      const int f = (i > 0 ? SIMT_EX_ACC : 0) | (i < np - 1 ? SIMT_EX_KEEP : 0);
      launch_kahan_tma_ex<KahanTma, false>(c.A + i * kp, n, c.B + i * kp * n, n, c.C, E, rows, kp, n, f, 0);
    }
  };
  go();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"kernel\":\"kahan_panels\",\"unroll\":%d,\"rows\":%lld,\"panels\":%d,\"ms\":%.4f,\"err\":\"%s\"}\n",
         kKahanUnroll, (long long)rows, np, ms / 3, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'K') {  // the Kahan panel schedule (compile with -DMMK_KAHAN_UNROLL=k)
    Ctx c;
    c.n = 8192;
    double* E;
    cudaMalloc(&c.A, c.n * c.n * 8);
    cudaMalloc(&c.B, c.n * c.n * 8);
    cudaMalloc(&c.C, c.n * c.n * 8);
    cudaMalloc(&E, c.n * c.n * 8);
    fill<<<1024, 256>>>(c.A, c.n * c.n, 1);
    fill<<<1024, 256>>>(c.B, c.n * c.n, 2);
    for (int64_t rows : {1024, 4096}) panel_kahan(c, E, rows, 4);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'e') {
    Ctx c;
    c.n = 8192;
    c.reps = 10;
    cudaMalloc(&c.A, c.n * c.n * 8);
    cudaMalloc(&c.B, c.n * c.n * 8);
    cudaMalloc(&c.C, c.n * c.n * 8);
    cudaMalloc(&c.y, c.n * 8);
    cudaMalloc(&c.z, c.n * 8);
    fill<<<1024, 256>>>(c.A, c.n * c.n, 1);
    fill<<<1024, 256>>>(c.B, c.n * c.n, 2);
    cudaMemset(c.y, 0, c.n * 8);
    cudaMemset(c.z, 0, c.n * 8);
    for (int64_t rows : {1024, 2048, 4096, 8192}) panel_wino(c, rows, 4);
    panel_wino(c, 8192, 1);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'h') {
    Ctx c;
    c.n = 8192;
    c.reps = 10;
    cudaMalloc(&c.A, c.n * c.n * 8);
    cudaMalloc(&c.B, c.n * c.n * 8);
    cudaMalloc(&c.C, c.n * c.n * 8);
    cudaMalloc(&c.R, c.n * c.n * 8);
    cudaMalloc(&c.y, c.n * 8);
    cudaMalloc(&c.z, c.n * 8);
    cudaMalloc(&c.bad, 8);
    fill<<<1024, 256>>>(c.A, c.n * c.n, 1);
    fill<<<1024, 256>>>(c.B, c.n * c.n, 2);
    cudaMemset(c.y, 0, c.n * 8);
    cudaMemset(c.z, 0, c.n * 8);
    std::vector<int64_t> heights = {1024, 2048, 4096};
    if (argc > 2) heights = {atoll(argv[2])};  // "h 8192": one height
    for (int64_t rows : heights) {
      shard_wino<WinogradTma>("tma_128x64_t8x8_s2_2cta_bk32", c, rows, true);
      shard_wino<SimtCfg<112, 64, 7, 8, 3, 2, 16>>("tma_112x64_t7x8_s3_2cta_bk16", c, rows, false);
      shard_wino<WinogradTma96>("tma_96x64_t6x8_s3_3cta_bk16", c, rows, false);
      shard_wino<SimtCfg<112, 64, 7, 8, 2, 2, 32>>("tma_112x64_t7x8_s2_2cta_bk32", c, rows, false);
      shard_wino<SimtCfg<64, 64, 4, 8, 3, 2, 32>>("tma_64x64_t4x8_s3_2cta_bk32", c, rows, false);
      shard_wino<SimtCfg<64, 64, 4, 8, 2, 3, 32>>("tma_64x64_t4x8_s2_3cta_bk32", c, rows, false);
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'o') {
    OddCtx c;
    cudaMalloc(&c.A, 4096 * 1002 * 8);
    cudaMalloc(&c.B, 1001 * 3000 * 8);
    cudaMalloc(&c.C, 4096 * 3000 * 8);
    cudaMalloc(&c.R, 4096 * 3000 * 8);
    cudaMalloc(&c.y, 4096 * 8);
    cudaMalloc(&c.z, 3000 * 8);
    cudaMalloc(&c.bad, 8);
    fill<<<1024, 256>>>(c.A, 4096 * 1002, 1);
    fill<<<1024, 256>>>(c.B, 1001 * 3000, 2);
    cudaMemset(c.y, 0, 4096 * 8);
    cudaMemset(c.z, 0, 3000 * 8);
    odd_wino<WinogradTma>("wino_tma_128x64_t8x8_s2_2cta_bk32", c);
    odd_wino<WinogradTma96>("wino_tma_96x64_t6x8_s3_3cta_bk16", c);
    odd_wino<SimtCfg<112, 64, 7, 8, 2, 2, 32>>("wino_tma_112x64_t7x8_s2_2cta_bk32", c);
    odd_wino<SimtCfg<112, 64, 7, 8, 3, 2, 16>>("wino_tma_112x64_t7x8_s3_2cta_bk16", c);
    odd_wino<SimtCfg<64, 64, 4, 8, 3, 3, 32>>("wino_tma_64x64_t4x8_s3_3cta_bk32", c);
    odd_wino<SimtCfg<80, 64, 5, 8, 2, 3, 32>>("wino_tma_80x64_t5x8_s2_3cta_bk32", c);
    c.have_ref = false;
    odd_kahan<KahanTma>("kahan_tma_64x64_t4x8_s3_2cta_bk32", c);
    odd_kahan<SimtCfg<48, 64, 3, 8, 3, 3, 32>>("kahan_tma_48x64_t3x8_s3_3cta_bk32", c);
    odd_kahan<SimtCfg<48, 64, 3, 8, 2, 3, 32>>("kahan_tma_48x64_t3x8_s2_3cta_bk32", c);
    odd_kahan<SimtCfg<32, 64, 2, 8, 3, 4, 32>>("kahan_tma_32x64_t2x8_s3_4cta_bk32", c);
    odd_kahan<SimtCfg<80, 64, 5, 8, 2, 2, 32>>("kahan_tma_80x64_t5x8_s2_2cta_bk32", c);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'c') {
    double *A, *B, *C, *y, *z;
    cudaMalloc(&A, 4096 * 1002 * 8);
    cudaMalloc(&B, 1002 * 3000 * 8);
    cudaMalloc(&C, 4096 * 3000 * 8);
    cudaMalloc(&y, 4096 * 8);
    cudaMalloc(&z, 3000 * 8);
    fill<<<1024, 256>>>(A, 4096 * 1002, 1);
    fill<<<1024, 256>>>(B, 1002 * 3000, 2);
    rect<SimtCfg<128, 64, 8, 8, 3, 2>>("winograd", "128x64_t8x8_s3_2cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<64, 64, 4, 8, 3, 2>>("winograd", "64x64_t4x8_s3_2cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<64, 64, 8, 8, 3, 4>>("winograd", "64x64_t8x8_s3_4cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<96, 64, 6, 8, 3, 3>>("winograd", "96x64_t6x8_s3_3cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<96, 64, 6, 8, 2, 3>>("winograd", "96x64_t6x8_s2_3cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<128, 64, 8, 8, 2, 2>>("winograd", "128x64_t8x8_s2_2cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<128, 64, 8, 8, 3, 2, 32>>("winograd", "128x64_t8x8_s3_2cta_bk32", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<64, 64, 4, 8, 3, 2>>("kahan", "64x64_t4x8_s3_2cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<64, 64, 8, 4, 3, 2>>("kahan", "64x64_t8x4_s3_2cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<32, 64, 4, 8, 3, 3>>("kahan", "32x64_t4x8_s3_3cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<48, 64, 3, 8, 3, 3>>("kahan", "48x64_t3x8_s3_3cta", A, B, C, y, z, 4096, 1001, 3000);
    rect<SimtCfg<64, 64, 4, 8, 2, 2, 32>>("kahan", "64x64_t4x8_s2_2cta_bk32", A, B, C, y, z, 4096, 1001, 3000);
    return 0;
  }
  const bool wino_only = argc > 1 && argv[1][0] == 'w';
  const bool kahan_only = argc > 1 && argv[1][0] == 'k';
  Ctx c;
  c.n = argc > 1 && !wino_only && !kahan_only && argv[1][0] != 'x' && argv[1][0] != 'y' ? atoll(argv[1]) : 8192;
  c.reps = argc > 2 ? atoi(argv[2]) : 2;
  cudaMalloc(&c.A, c.n * c.n * 8);
  cudaMalloc(&c.B, c.n * c.n * 8);
  cudaMalloc(&c.C, c.n * c.n * 8);
  cudaMalloc(&c.R, c.n * c.n * 8);
  cudaMalloc(&c.y, c.n * 8);
  cudaMalloc(&c.z, c.n * 8);
  cudaMalloc(&c.bad, 8);
  fill<<<1024, 256>>>(c.A, c.n * c.n, 1);
  fill<<<1024, 256>>>(c.B, c.n * c.n, 2);
  // SimtCfg<BM, BN, TM, TN, STAGES, MINB, BK>
  if (argc > 1 && argv[1][0] == 's') {  // 1024^3 (config c2): small-grid configurations, cp.async kernels
    c.n = 1024;
    c.reps = 20;
    cudaMalloc(&c.A, c.n * c.n * 8);
    cudaMalloc(&c.B, c.n * c.n * 8);
    cudaMalloc(&c.C, c.n * c.n * 8);
    cudaMalloc(&c.R, c.n * c.n * 8);
    cudaMalloc(&c.y, c.n * 8);
    cudaMalloc(&c.z, c.n * 8);
    cudaMalloc(&c.bad, 8);
    fill<<<1024, 256>>>(c.A, c.n * c.n, 1);
    fill<<<1024, 256>>>(c.B, c.n * c.n, 2);
    wino<SimtCfg<64, 64, 4, 8, 3, 2>>("wino_64x64_t4x8_s3_2cta", c, true);
    wino<SimtCfg<32, 32, 2, 4, 3, 4>>("wino_32x32_t2x4_s3_4cta", c, false);
    wino<SimtCfg<64, 32, 4, 4, 3, 4>>("wino_64x32_t4x4_s3_4cta", c, false);
    wino<SimtCfg<32, 64, 2, 8, 3, 4>>("wino_32x64_t2x8_s3_4cta", c, false);
    wino<SimtCfg<64, 64, 8, 8, 3, 4>>("wino_64x64_t8x8_s3_4cta", c, false);
    kahan<SimtCfg<32, 32, 2, 4, 3, 4>>("kahan_32x32_t2x4_s3_4cta", c, true);
    kahan<SimtCfg<32, 32, 2, 4, 4, 6>>("kahan_32x32_t2x4_s4_6cta", c, false);
    kahan<SimtCfg<32, 64, 2, 8, 3, 4>>("kahan_32x64_t2x8_s3_4cta", c, false);
    if (argv[1][1] == 't') {  // "st": TMA-fed small-grid configurations at 1024^3 (r02)
      wino<SimtCfg<64, 64, 4, 8, 3, 2>>("wino_64x64_t4x8_s3_2cta", c, true);
      wino_tma<SimtCfg<64, 64, 4, 8, 2, 2, 32>>("wino_tma_64x64_t4x8_s2_2cta_bk32", c);
      wino_tma<SimtCfg<64, 64, 4, 8, 3, 2, 32>>("wino_tma_64x64_t4x8_s3_2cta_bk32", c);
      wino_tma<SimtCfg<64, 64, 4, 8, 4, 2, 16>>("wino_tma_64x64_t4x8_s4_2cta_bk16", c);
      wino_tma<SimtCfg<64, 64, 4, 8, 2, 3, 32>>("wino_tma_64x64_t4x8_s2_3cta_bk32", c);
      wino_tma<SimtCfg<32, 64, 2, 8, 3, 4, 32>>("wino_tma_32x64_t2x8_s3_4cta_bk32", c);
      wino_tma<SimtCfg<64, 64, 8, 8, 3, 4, 32>>("wino_tma_64x64_t8x8_s3_4cta_bk32", c);
      wino_tma<SimtCfg<64, 64, 8, 8, 4, 4, 16>>("wino_tma_64x64_t8x8_s4_4cta_bk16", c);
      kahan<SimtCfg<32, 32, 2, 4, 3, 4>>("kahan_32x32_t2x4_s3_4cta", c, true);
      kahan_tma<SimtCfg<32, 32, 2, 4, 3, 4, 32>>("kahan_tma_32x32_t2x4_s3_4cta_bk32", c);
      kahan_tma<SimtCfg<32, 32, 2, 4, 4, 6, 16>>("kahan_tma_32x32_t2x4_s4_6cta_bk16", c);
      kahan_tma<SimtCfg<32, 64, 2, 8, 3, 4, 32>>("kahan_tma_32x64_t2x8_s3_4cta_bk32", c);
      kahan_tma<SimtCfg<64, 32, 4, 4, 3, 4, 32>>("kahan_tma_64x32_t4x4_s3_4cta_bk32", c);
      kahan_tma<SimtCfg<64, 64, 4, 8, 3, 2, 32>>("kahan_tma_64x64_t4x8_s3_2cta_bk32", c);
    }
    return 0;
  }
  if (kahan_only) {  // K2 configurations only
    kahan<SimtCfg<64, 64, 4, 8, 2, 2, 32>>("cpasync_64x64_s2_bk32", c, true);
    kahan_tma<SimtCfg<64, 64, 4, 8, 3, 2, 32>>("tma_64x64_s3_2cta_bk32", c);
    kahan_tma<SimtCfg<64, 64, 4, 8, 2, 3, 32>>("tma_64x64_s2_3cta_bk32", c);
    kahan_tma<SimtCfg<64, 64, 4, 8, 4, 3, 16>>("tma_64x64_s4_3cta_bk16", c);
    kahan_tma<SimtCfg<48, 64, 3, 8, 4, 3, 16>>("tma_48x64_t3x8_s4_3cta_bk16", c);
    kahan_tma<SimtCfg<48, 64, 3, 8, 2, 3, 32>>("tma_48x64_t3x8_s2_3cta_bk32", c);
    kahan_tma<SimtCfg<64, 64, 4, 8, 6, 2, 16>>("tma_64x64_s6_2cta_bk16", c);
    kahan_tma<SimtCfg<64, 64, 4, 8, 5, 2, 16>>("tma_64x64_s5_2cta_bk16", c);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'x') {  // the production K3 configuration only (schedule variants)
    wino<SimtCfg<128, 64, 8, 8, 3, 2>>("cpasync_128x64_bk16", c, true);
    wino_tma<SimtCfg<128, 64, 8, 8, 2, 2, 32>>("tma_128x64_s2_2cta_bk32", c);
    wino_tma<SimtCfg<128, 64, 8, 8, 3, 2, 32>>("tma_128x64_s3_2cta_bk32", c);
    if (argv[1][1] == 'd') {  // "xd": deeper rings of 16-deep k tiles in the same shared memory (r02)
      wino_tma<SimtCfg<128, 64, 8, 8, 4, 2, 16>>("tma_128x64_s4_2cta_bk16", c);
      wino_tma<SimtCfg<128, 64, 8, 8, 3, 2, 16>>("tma_128x64_s3_2cta_bk16", c);
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'y') {  // the production K2 configuration only (unroll variants)
    kahan<SimtCfg<64, 64, 4, 8, 2, 2, 32>>("cpasync_64x64_s2_bk32", c, true);
    kahan_tma<SimtCfg<64, 64, 4, 8, 3, 2, 32>>("tma_64x64_s3_2cta_bk32", c);
    return 0;
  }
  if (wino_only) {  // K3 configurations only
    wino<SimtCfg<128, 64, 8, 8, 3, 2>>("cpasync_128x64_bk16", c, true);
    wino_tma<SimtCfg<128, 64, 8, 8, 2, 2, 32>>("tma_128x64_s2_2cta_bk32", c);
    wino_tma<SimtCfg<128, 64, 8, 8, 3, 1, 32>>("tma_128x64_s3_1cta_bk32", c);
    wino_tma<SimtCfg<64, 64, 8, 8, 2, 3, 32>>("tma_64x64_t8x8_s2_3cta_bk32", c);
    wino_tma<SimtCfg<64, 64, 4, 8, 3, 3, 32>>("tma_64x64_t4x8_s3_3cta_bk32", c);
    wino_tma<SimtCfg<128, 64, 8, 8, 2, 3, 16>>("tma_128x64_s2_3cta_bk16", c);
    wino_tma<SimtCfg<128, 64, 8, 8, 3, 3, 16>>("tma_128x64_s3_3cta_bk16", c);
    wino_tma<SimtCfg<96, 64, 6, 8, 3, 3, 16>>("tma_96x64_t6x8_s3_3cta_bk16", c);
    wino_tma<SimtCfg<96, 64, 6, 8, 2, 3, 16>>("tma_96x64_t6x8_s2_3cta_bk16", c);
    return 0;
  }
  kahan<SimtCfg<64, 64, 4, 8, 2, 2, 32>>("cpasync_64x64_s2_bk32", c, true);
  kahan_tma<SimtCfg<64, 64, 4, 8, 3, 2, 32>>("tma_64x64_s3_2cta_bk32", c);
  kahan_tma<SimtCfg<64, 64, 4, 8, 2, 3, 32>>("tma_64x64_s2_3cta_bk32", c);
  wino<SimtCfg<128, 64, 8, 8, 3, 2>>("cpasync_128x64_bk16", c, true);
  wino_tma<SimtCfg<128, 64, 8, 8, 2, 2, 32>>("tma_128x64_s2_2cta_bk32", c);
  wino_tma<SimtCfg<64, 64, 8, 8, 2, 3, 32>>("tma_64x64_t8x8_s2_3cta_bk32", c);
  return 0;
}
