// kahan.cuh -- K2: NaivKahan.  Each C entry is the Kahan-compensated sum of the
// products x_k = A_ik B_kj, k = 0..P-1 in order, with the update of P:122-132:
//     err = err + x;  t = sum + err;  err = (sum - t) + err;  sum = t;      result = sum.
// Every operation is a separately rounded FP64 SIMT op (__dmul_rn / __dadd_rn /
// __dsub_rn, never contracted into DFMA), so the result equals the oracle's
// or_naive_kahan bit for bit.  5 FP64 ops per term -> ceiling 1/5 of the DFMA-pipe
// rate in 2NPM/t terms.
//
// CTA tile 64 x 128, 256 threads (16 x 16), thread tile 4 x 8 (rows 4*ty..4*ty+3, columns
// 2*tx + 32*c + {0,1}, c < 4, so each B read is a conflict-free 16-byte LDS.128).
// Operands staged with a 3-deep cp.async ring; the k-loop stops exactly at P (padded
// terms are NOT no-ops for the compensated update).
#pragma once
#include "common.cuh"

namespace mmk {
namespace kahan {
constexpr int BM = 64, BN = 128, BK = 16, THREADS = 256, STAGES = 3;
constexpr int A_ELEMS = BM * BK, B_ELEMS = BK * BN;
constexpr size_t SMEM = size_t(STAGES) * (A_ELEMS + B_ELEMS) * sizeof(double);
}  // namespace kahan

template <int AV, int BV>
__device__ __forceinline__ void kahan_load_tile(double* As, double* Bs, const double* __restrict__ A,
                                                const double* __restrict__ B, int64_t N, int64_t P, int64_t M,
                                                int64_t m0, int64_t n0, int64_t k0, int tid) {
  using namespace kahan;
  if (AV == 2) {
#pragma unroll
    for (int i = 0; i < (A_ELEMS / 2) / THREADS; ++i) {
      int c = tid + i * THREADS;
      int r = c >> 3, kp = (c & 7) * 2;
      int64_t gm = m0 + r, gk = k0 + kp;
      bool v = gm < N && gk < P;
      cp_async16(As + r * BK + kp, v ? A + gm * P + gk : A, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < A_ELEMS / THREADS; ++i) {
      int e = tid + i * THREADS;
      int r = e >> 4, kk = e & 15;
      int64_t gm = m0 + r, gk = k0 + kk;
      bool v = gm < N && gk < P;
      cp_async8(As + r * BK + kk, v ? A + gm * P + gk : A, v);
    }
  }
  if (BV == 2) {
#pragma unroll
    for (int i = 0; i < (B_ELEMS / 2) / THREADS; ++i) {
      int c = tid + i * THREADS;
      int kr = c >> 6, np = (c & 63) * 2;
      int64_t gk = k0 + kr, gn = n0 + np;
      bool v = gk < P && gn < M;
      cp_async16(Bs + kr * BN + np, v ? B + gk * M + gn : B, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < B_ELEMS / THREADS; ++i) {
      int e = tid + i * THREADS;
      int kr = e >> 7, nn = e & 127;
      int64_t gk = k0 + kr, gn = n0 + nn;
      bool v = gk < P && gn < M;
      cp_async8(Bs + kr * BN + nn, v ? B + gk * M + gn : B, v);
    }
  }
}

struct KahanState {
  double sum[4][8], err[4][8];
};

__device__ __forceinline__ void kahan_step(KahanState& s, const double* As, const double* Bs, int kk, int ty,
                                           int tx) {
  using namespace kahan;
  double a[4], b[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = As[(4 * ty + i) * BK + kk];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double2 v = *reinterpret_cast<const double2*>(Bs + kk * BN + 2 * tx + 32 * c);
    b[2 * c] = v.x;
    b[2 * c + 1] = v.y;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double x = dmul(a[i], b[j]);
      double e = dadd(s.err[i][j], x);
      const double t = dadd(s.sum[i][j], e);
      e = dadd(dsub(s.sum[i][j], t), e);
      s.sum[i][j] = t;
      s.err[i][j] = e;
    }
}

template <int AV, int BV, int CV>
__global__ void __launch_bounds__(kahan::THREADS, 1)
    kahan_gemm_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C, int64_t N,
                      int64_t P, int64_t M) {
  using namespace kahan;
  extern __shared__ __align__(128) double smem[];
  double* As_base = smem;
  double* Bs_base = smem + STAGES * A_ELEMS;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = int64_t(blockIdx.y) * BM, n0 = int64_t(blockIdx.x) * BN;

  KahanState s;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) s.sum[i][j] = s.err[i][j] = 0.0;

  const int KT = int(cdiv(P, BK));
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < KT)
      kahan_load_tile<AV, BV>(As_base + st * A_ELEMS, Bs_base + st * B_ELEMS, A, B, N, P, M, m0, n0,
                              int64_t(st) * BK, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT)
        kahan_load_tile<AV, BV>(As_base + (nk % STAGES) * A_ELEMS, Bs_base + (nk % STAGES) * B_ELEMS, A, B, N, P,
                                M, m0, n0, int64_t(nk) * BK, tid);
      cp_async_commit();
    }
    const double* As = As_base + (kt % STAGES) * A_ELEMS;
    const double* Bs = Bs_base + (kt % STAGES) * B_ELEMS;
    const int64_t k0 = int64_t(kt) * BK;
    if (k0 + BK <= P) {
#pragma unroll 4
      for (int kk = 0; kk < BK; ++kk) kahan_step(s, As, Bs, kk, ty, tx);
    } else {
      const int kmax = int(P - k0);
      for (int kk = 0; kk < kmax; ++kk) kahan_step(s, As, Bs, kk, ty, tx);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + 4 * ty + i;
    if (row >= N) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t col = n0 + 2 * tx + 32 * c;
      if (CV == 2 && col + 1 < M) {
        *reinterpret_cast<double2*>(C + row * M + col) = make_double2(s.sum[i][2 * c], s.sum[i][2 * c + 1]);
      } else {
        if (col < M) C[row * M + col] = s.sum[i][2 * c];
        if (col + 1 < M) C[row * M + col + 1] = s.sum[i][2 * c + 1];
      }
    }
  }
}

template <int AV, int BV, int CV>
cudaError_t launch_kahan_t(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                           cudaStream_t st) {
  using namespace kahan;
  auto kern = kahan_gemm_kernel<AV, BV, CV>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(unsigned(cdiv(M, BN)), unsigned(cdiv(N, BM)));
  kern<<<grid, THREADS, SMEM, st>>>(A, B, C, N, P, M);
  note_launch();
  return cudaGetLastError();
}

inline cudaError_t launch_kahan(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                                cudaStream_t st) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool av = al(A) && P % 2 == 0, bv = al(B) && M % 2 == 0, cv = al(C) && M % 2 == 0;
  if (av && bv && cv) return launch_kahan_t<2, 2, 2>(A, B, C, N, P, M, st);
  if (bv && cv) return launch_kahan_t<1, 2, 2>(A, B, C, N, P, M, st);
  if (av) return launch_kahan_t<2, 1, 1>(A, B, C, N, P, M, st);
  return launch_kahan_t<1, 1, 1>(A, B, C, N, P, M, st);
}

}  // namespace mmk
