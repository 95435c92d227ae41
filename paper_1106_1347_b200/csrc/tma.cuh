// tma.cuh -- Tensor Memory Accelerator helpers for sm_100a (product path).
//
// Host: 2-D tensor maps of row-major float64 matrices, encoded with the driver's
// cuTensorMapEncodeTiled (fetched through cudaGetDriverEntryPoint, so the library does not
// link libcuda).  Device: mbarrier primitives and the 2-D tiled bulk-tensor copy
// global -> shared whose completion is counted in bytes on an mbarrier (expect_tx).
// TMA needs a 16-byte aligned base and a row pitch that is a multiple of 16 bytes (an even
// number of doubles); callers fall back to cp.async for other operands (e.g. P = 1001).
// Out-of-bounds box elements are filled with +0.0.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace mmk {

// ---- device: mbarrier + copies
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// orders this thread's prior generic-proxy shared-memory accesses before later async-proxy
// (TMA) accesses to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive once all prior cp.async of this thread have landed (counts as this thread's arrival)
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// box at (x = column, y = row) of the tensor map -> shared dst; completes tx bytes on bar
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// shared src -> box at (x = column, y = row) of the tensor map (async proxy; bulk_group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// all but the N most recent bulk groups have finished READING shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---- host: tensor map encoding
inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

// can X (rows x cols, leading dimension ld doubles) be described by a TMA tensor map?
inline bool tma_ok(const void* X, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(X) & 15) == 0 && ld % 2 == 0 && tma_encoder() != nullptr;
}

// Encoded maps are cached (the same operands recur call after call: bench loops, Strassen levels,
// the e2e path); a map is a pure function of (address, dims, strides, box, swizzle), so a hit
// is valid even if the memory was freed and reallocated at the same address.
struct TmaKey {
  const void* p;
  uint64_t dims[3], strides[2];
  uint32_t box[3];
  int rank, swizzle;
  bool operator==(const TmaKey& o) const {
    return p == o.p && rank == o.rank && swizzle == o.swizzle && dims[0] == o.dims[0] && dims[1] == o.dims[1] &&
           dims[2] == o.dims[2] && strides[0] == o.strides[0] && strides[1] == o.strides[1] && box[0] == o.box[0] &&
           box[1] == o.box[1] && box[2] == o.box[2];
  }
};

inline bool tma_encode_key(CUtensorMap* map, const TmaKey& k) {
  constexpr int CAP = 32;
  static std::mutex mu;
  static TmaKey keys[CAP];
  static CUtensorMap maps[CAP];
  static int used = 0, next = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    for (int i = 0; i < used; ++i)
      if (keys[i] == k) {
        *map = maps[i];
        return true;
      }
  }
  auto enc = tma_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {k.dims[0], k.dims[1], k.dims[2]};
  cuuint64_t strides[2] = {k.strides[0], k.strides[1]};
  cuuint32_t box[3] = {k.box[0], k.box[1], k.box[2]};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cuuint32_t(k.rank), const_cast<void*>(k.p), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   k.swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  std::lock_guard<std::mutex> g(mu);
  keys[next] = k;
  maps[next] = *map;
  next = (next + 1) % CAP;
  if (used < CAP) ++used;
  return true;
}

// 2-D map of a row-major float64 matrix: box = box_rows x box_cols doubles
// swizzle128: box_cols must be 16 (128-byte rows); 16-byte chunk c of box row r lands at chunk c ^ (r % 8)
inline bool tma_encode_2d(CUtensorMap* map, const double* X, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                          int box_cols, bool swizzle128) {
  TmaKey k{};
  k.p = X;
  k.rank = 2;
  k.swizzle = swizzle128 ? 1 : 0;
  k.dims[0] = uint64_t(cols);
  k.dims[1] = uint64_t(rows);
  k.strides[0] = uint64_t(ld) * sizeof(double);
  k.box[0] = uint32_t(box_cols);
  k.box[1] = uint32_t(box_rows);
  return tma_encode_key(map, k);
}

// 3-D map {columns, rows, batch} of `batch` row-major float64 matrices bstride doubles apart;
// box = box_rows x 16 doubles x 1, 128-byte swizzle
inline bool tma_encode_3d(CUtensorMap* map, const double* X, int64_t rows, int64_t cols, int64_t ld, int64_t batch,
                          int64_t bstride, int box_rows) {
  TmaKey k{};
  k.p = X;
  k.rank = 3;
  k.swizzle = 1;
  k.dims[0] = uint64_t(cols);
  k.dims[1] = uint64_t(rows);
  k.dims[2] = uint64_t(batch);
  k.strides[0] = uint64_t(ld) * 8;
  k.strides[1] = uint64_t(batch > 1 ? bstride : rows * ld) * 8;
  k.box[0] = 16;
  k.box[1] = uint32_t(box_rows);
  k.box[2] = 1;
  return tma_encode_key(map, k);
}

}  // namespace mmk
