// norm_lambda.cuh -- K4 norm_inf and K5 the lambda rule.
//
// K4: ||X||_inf = max_i sum_j |X_ij|.  One thread owns one row and sums it left to right
// (the oracle's order, so row sums -- and hence lambda -- are bit-identical to the CPU
// oracle); the 32 x 32 tiles are streamed through shared memory with a 4-deep cp.async
// ring so global reads stay coalesced.  The max over rows is order-free: each block
// reduces its rows and issues one atomicMax on the IEEE bit pattern (non-negative doubles
// order like their uint64 images).  HBM-bound: 8 * rows * cols bytes read once.
//
// K5: lambda with 1/2 <= 2^(2 lambda) nA / nB <= 2, computed exactly from frexp
// (reading R7, ties -> larger |lambda|, zero norm -> 0), plus the exact scale factors
// 2^lambda and 2^-lambda, on one device thread.
#pragma once
#include "common.cuh"

namespace mmk {

// ---- line streaming: one warp owns 32 "lines" (rows of X, or columns of X) and streams them
// through shared memory in 32 x LS_TK tiles with an LS_STAGES-deep cp.async ring; every global
// read is a coalesced 256-byte segment and each lane then walks its own line in index order.
constexpr int LS_LINES = 32, LS_TK = 64, LS_STAGES = 5;
constexpr int LS_ROWPITCH = LS_TK + 1;       // row-lines tile [32][TK+1]  (lane reads its row)
constexpr int LS_COLPITCH = LS_LINES + 1;    // column-lines tile [TK][33] (lane reads its column)
constexpr int LS_TILE = LS_LINES * LS_ROWPITCH > LS_TK * LS_COLPITCH ? LS_LINES * LS_ROWPITCH : LS_TK * LS_COLPITCH;
constexpr size_t LS_SMEM = size_t(LS_STAGES) * LS_TILE * sizeof(double);

// rows [r0, r0+32) x columns [c0, c0+TK) of row-major X (ld) -> t[r][c]; zero outside rv x cv
__device__ __forceinline__ void ls_load_rowlines(double* t, const double* __restrict__ X, int64_t ld, int64_t r0,
                                                 int64_t c0, int64_t rv, int64_t cv, int lane) {
#pragma unroll 8
  for (int r = 0; r < LS_LINES; ++r) {
#pragma unroll
    for (int h = 0; h < LS_TK / 32; ++h) {
      const int64_t gr = r0 + r, gc = c0 + lane + 32 * h;
      const bool v = gr < rv && gc < cv;
      cp_async8(t + r * LS_ROWPITCH + lane + 32 * h, v ? X + gr * ld + gc : X, v);
    }
  }
}

// rows [k0, k0+TK) x columns [l0, l0+32) of row-major X (ld) -> t[k][c]; zero outside kv x lv
__device__ __forceinline__ void ls_load_collines(double* t, const double* __restrict__ X, int64_t ld, int64_t k0,
                                                 int64_t l0, int64_t kv, int64_t lv, int lane) {
#pragma unroll 8
  for (int k = 0; k < LS_TK; ++k) {
    const int64_t gk = k0 + k, gc = l0 + lane;
    const bool v = gk < kv && gc < lv;
    cp_async8(t + k * LS_COLPITCH + lane, v ? X + gk * ld + gc : X, v);
  }
}

__global__ void __launch_bounds__(LS_LINES) norm_inf_kernel(const double* __restrict__ X, int64_t rows,
                                                            int64_t cols, unsigned long long* __restrict__ out) {
  extern __shared__ __align__(16) double ls_smem[];
  const int lane = threadIdx.x;
  const int64_t r0 = int64_t(blockIdx.x) * LS_LINES;
  const int64_t KT = cdiv(cols, LS_TK);
#pragma unroll
  for (int s = 0; s < LS_STAGES - 1; ++s) {
    if (s < KT) ls_load_rowlines(ls_smem + s * LS_TILE, X, cols, r0, int64_t(s) * LS_TK, rows, cols, lane);
    cp_async_commit();
  }
  double sum = 0.0;
  for (int64_t kt = 0; kt < KT; ++kt) {
    cp_async_wait<LS_STAGES - 2>();
    __syncwarp();
    {
      const int64_t nk = kt + LS_STAGES - 1;
      if (nk < KT)
        ls_load_rowlines(ls_smem + (nk % LS_STAGES) * LS_TILE, X, cols, r0, nk * LS_TK, rows, cols, lane);
      cp_async_commit();
    }
    const double* t = ls_smem + (kt % LS_STAGES) * LS_TILE + lane * LS_ROWPITCH;
    const int64_t rem_c = cols - kt * LS_TK;
    const int n = int(rem_c < LS_TK ? rem_c : LS_TK);
    for (int j = 0; j < n; ++j) sum = dadd(sum, fabs(t[j]));  // row sum, left to right
    __syncwarp();
  }
  cp_async_wait<0>();
  // order-free max over the block's rows (rows past the end contribute +0)
  double m = (r0 + lane < rows) ? sum : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// The rule of P:206-208 (shared by the device kernel and the host test entry point).
__host__ __device__ inline int lambda_rule(double nA, double nB) {
  if (nA == 0.0 || nB == 0.0) return 0;
  int eA, eB;
  const double mA = frexp(nA, &eA);
  const double mB = frexp(nB, &eB);
  const int d = eB - eA;
  if (d % 2 == 0) return d / 2;
  if (mA < mB) return (d + 1) / 2;
  if (mA > mB) return (d - 1) / 2;
  return d > 0 ? (d + 1) / 2 : (d - 1) / 2;
}

// norms[0] = ||A||, norms[1] = ||B|| (as uint64 bit patterns from norm_inf_kernel)
// -> lam[0] = lambda, scale[0] = 2^lambda, scale[1] = 2^-lambda
__global__ void lambda_kernel(const unsigned long long* __restrict__ norms, int* __restrict__ lam,
                              double* __restrict__ scale) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double nA = __longlong_as_double(static_cast<long long>(norms[0]));
    const double nB = __longlong_as_double(static_cast<long long>(norms[1]));
    const int l = lambda_rule(nA, nB);
    lam[0] = l;
    scale[0] = ldexp(1.0, l);
    scale[1] = ldexp(1.0, -l);
  }
}

// out: device uint64 slot, zeroed here then max-reduced
inline cudaError_t launch_norm_inf(const double* X, int64_t rows, int64_t cols, unsigned long long* out,
                                   cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(norm_inf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(LS_SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  norm_inf_kernel<<<unsigned(cdiv(rows, LS_LINES)), LS_LINES, LS_SMEM, st>>>(X, rows, cols, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace mmk
