// TMA probe: does a tiled tensor map whose inner extent is an odd number of doubles (8 mod 16
// bytes) load correctly?  (The paired-row maps of gemm_tma.cuh for odd pitches.)  Loads one
// [32 rows][16 cols] box with the 128-byte swizzle at (x, y) and reports CUDA errors and a checksum.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe tma_probe.cu
#include <cstdio>
#include <cstdlib>

#include "../../paper_1106_1347_b200/csrc/tma.cuh"

using namespace mmk;

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap map, int x, int y, double* out) {
  __shared__ __align__(1024) double t[32 * 16];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 32 * 16 * 8);
    tma3(t, &map, x, y, 0, &bar);
  }
  mbar_wait(&bar, 0);
  double s = 0;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) s += t[i];
  atomicAdd(out, s);
}

int main(int argc, char** argv) {
  const int rows = 64, lda = 1001;
  double* A;
  cudaMalloc(&A, size_t(rows) * lda * 8 + 256);
  cudaMemset(A, 0, size_t(rows) * lda * 8);
  double* out;
  cudaMalloc(&out, 8);
  const int64_t w0 = argc > 1 ? atoll(argv[1]) : 1001;
  for (int64_t w : {w0}) {
    CUtensorMap map;
    bool ok = tma_encode_3d(&map, A, rows / 2, w, 2 * lda, 1, 0, 32);
    cudaMemset(out, 0, 8);
    const int x = argc > 2 ? atoi(argv[2]) : 0;
    if (ok) k<<<1, 128>>>(map, x, 0, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"inner_extent_doubles\": %lld, \"x\": %d, \"encoded\": %d, \"err\": \"%s\"}\n", (long long)w, x,
           int(ok), cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;  // a sticky error: the context is gone
  }
  return 0;
}
