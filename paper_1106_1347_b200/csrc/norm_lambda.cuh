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

namespace nrm {
constexpr int ROWS = 32;  // rows per block (one warp)
constexpr int TK = 32;    // columns per stage
constexpr int STAGES = 4;
}  // namespace nrm

__global__ void __launch_bounds__(nrm::ROWS) norm_inf_kernel(const double* __restrict__ X, int64_t rows,
                                                             int64_t cols, unsigned long long* __restrict__ out) {
  using namespace nrm;
  __shared__ __align__(16) double tile[STAGES][ROWS][TK + 1];
  const int lane = threadIdx.x;
  const int64_t r0 = int64_t(blockIdx.x) * ROWS;
  const int64_t KT = cdiv(cols, TK);
  auto load = [&](int64_t kt, int s) {
    const int64_t c0 = kt * TK;
    // each lane copies column c0+lane of all 32 rows: one 256-byte coalesced row segment per step
#pragma unroll 8
    for (int rr = 0; rr < ROWS; ++rr) {
      const int64_t gr = r0 + rr, gc = c0 + lane;
      const bool v = gr < rows && gc < cols;
      cp_async8(&tile[s][rr][lane], v ? X + gr * cols + gc : X, v);
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load(s, s);
    cp_async_commit();
  }
  double sum = 0.0;
  for (int64_t kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncwarp();
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < KT) load(nk, int(nk % STAGES));
      cp_async_commit();
    }
    const int s = int(kt % STAGES);
    const int64_t rem_c = cols - kt * TK;
    const int n = int(rem_c < TK ? rem_c : TK);
    // zero-filled columns would add +0, which is harmless, but stop at the true end anyway
    for (int j = 0; j < n; ++j) sum = dadd(sum, fabs(tile[s][lane][j]));
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
  norm_inf_kernel<<<unsigned(cdiv(rows, nrm::ROWS)), nrm::ROWS, 0, st>>>(X, rows, cols, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace mmk
