// common.cuh -- shared device helpers for the sm_100a FP64 kernels (product path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler is attached

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "this library is built for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace mmk {

// host-side count of kernel launches (mm_launch_count)
inline std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}
inline void note_launch() { launch_counter().fetch_add(1, std::memory_order_relaxed); }

// NVTX range for the life of a scope (ABI calls, Strassen levels): visible in nsys / ncu --nvtx
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Opt kernel KERN into `bytes` of dynamic shared memory on the CURRENT device, once per
// (kernel, device): the attribute is per device, so a process driving several GPUs needs it on each.
template <auto KERN>
inline cudaError_t smem_attr_once(size_t bytes) {
  constexpr int kMaxDev = 64;
  static std::atomic<bool> done[kMaxDev];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!done[dev].load(std::memory_order_acquire)) {
    e = cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e != cudaSuccess) return e;
    done[dev].store(true, std::memory_order_release);
  }
  return cudaSuccess;
}

// ---- asynchronous global -> shared copies (LDGSTS).  src_size = 0 zero-fills the
// destination without reading global memory (used for out-of-range tile elements).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- FP64 tensor core: D(8x8) = A(8x4, row) * B(4x8, col) + C.  On sm_100a this is
// SASS DMMA.8x8x4; probe P3 (profiles/r01_probe) shows each output is the chain
// fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))) -- k increasing, fused.
// Fragments (PTX ISA, mma.m8n8k4 .f64): lane = 4g + t;  a = A[g][t];  b = B[t][g];
// c/d = {C[g][2t], C[g][2t+1]}.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- order-faithful scalar FP64 ops (no contraction into DFMA)
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

__host__ __device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace mmk
