// kahan.cuh -- K2: NaivKahan.  Each C entry is the Kahan-compensated sum of the
// products x_k = A_ik B_kj, k = 0..P-1 in order, with the update of P:122-132:
//     err = err + x;  t = sum + err;  err = (sum - t) + err;  sum = t;      result = sum.
// Every operation is a separately rounded FP64 SIMT op (__dmul_rn / __dadd_rn /
// __dsub_rn, never contracted into DFMA), so the result equals the oracle's
// or_naive_kahan bit for bit.  5 FP64 ops per term -> ceiling 1/5 of the DFMA rate in
// 2NPM/t terms.
//
// CTA tile BM x BN, thread tile TM x TN: thread (ty, tx) owns rows ty*TM + i and columns
// 2*tx + 2*TXN*c + {0,1} (TXN = BN/TN threads along N), so each B read is a conflict-free
// 16-byte LDS.128; A rows are padded to BK+2 doubles so the TM row reads of different ty
// fall in different banks.  Operands staged with a STAGES-deep cp.async ring; the k-loop
// stops exactly at P (padded terms are NOT no-ops for the compensated update).
#pragma once
#include "simt_tile.cuh"
#include "simt_tma.cuh"

#include <type_traits>

namespace mmk {

// 64 x 64 x 32 tiles, 128 threads of 4 x 8 outputs, double-buffered, 2 CTAs per SM
// (tools/tune/simt_tune.cu; 157.5 vs 158.0 ms for 16-deep k tiles, profiles/r01/simt_tune_bk32.jsonl)
using KahanDefault = SimtCfg<64, 64, 4, 8, 2, 2, 32>;

// FUSED (NEXT-3, reading R22): err = fma(a, b, err) replaces x = a*b; err = err + x
template <class CF, bool FUSED>
__device__ __forceinline__ void kahan_step(double (&sum)[CF::TM][CF::TN], double (&err)[CF::TM][CF::TN],
                                           const double* As, const double* Bs, int kk, int ty, int tx) {
  double b[CF::TN];
#pragma unroll
  for (int c = 0; c < CF::TN / 2; ++c) {
    double2 v = *reinterpret_cast<const double2*>(Bs + kk * CF::BN + 2 * tx + 2 * CF::TXN * c);
    b[2 * c] = v.x;
    b[2 * c + 1] = v.y;
  }
  // A's value of row i is read just before its TN updates (B's stay in registers)
#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    const double a = As[simt_row<CF>(ty, i) * CF::APITCH + kk];
#pragma unroll
    for (int j = 0; j < CF::TN; ++j) {
      double e = FUSED ? __fma_rn(a, b[j], err[i][j]) : dadd(err[i][j], dmul(a, b[j]));
      const double t = dadd(sum[i][j], e);
      e = dadd(dsub(sum[i][j], t), e);
      sum[i][j] = t;
      err[i][j] = e;
    }
  }
}

template <class CF, int AV, int BV, int CV, bool FUSED>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB)
    kahan_gemm_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C, int64_t N,
                      int64_t P, int64_t M) {
  constexpr int BK = CF::BK, STAGES = CF::STAGES;
  extern __shared__ __align__(128) double smem[];
  double* As_base = smem;
  double* Bs_base = smem + STAGES * CF::A_ELEMS;
  const int tid = threadIdx.x, tx = tid % CF::TXN, ty = tid / CF::TXN;
  int64_t m0, n0;
  simt_tile_coords(N, M, CF::BM, CF::BN, m0, n0);

  double sum[CF::TM][CF::TN], err[CF::TM][CF::TN];
#pragma unroll
  for (int i = 0; i < CF::TM; ++i)
#pragma unroll
    for (int j = 0; j < CF::TN; ++j) sum[i][j] = err[i][j] = 0.0;

  const int KT = int(cdiv(P, BK));
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < KT)
      simt_load_tile<CF, AV, BV>(As_base + st * CF::A_ELEMS, Bs_base + st * CF::B_ELEMS, A, B, N, P, M, P, m0, n0,
                                 int64_t(st) * BK, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT)
        simt_load_tile<CF, AV, BV>(As_base + (nk % STAGES) * CF::A_ELEMS, Bs_base + (nk % STAGES) * CF::B_ELEMS, A,
                                   B, N, P, M, P, m0, n0, int64_t(nk) * BK, tid);
      cp_async_commit();
    }
    const double* As = As_base + (kt % STAGES) * CF::A_ELEMS;
    const double* Bs = Bs_base + (kt % STAGES) * CF::B_ELEMS;
    const int64_t k0 = int64_t(kt) * BK;
    if (k0 + BK <= P) {
#pragma unroll 4
      for (int kk = 0; kk < BK; ++kk) kahan_step<CF, FUSED>(sum, err, As, Bs, kk, ty, tx);
    } else {
      const int kmax = int(P - k0);
      for (int kk = 0; kk < kmax; ++kk) kahan_step<CF, FUSED>(sum, err, As, Bs, kk, ty, tx);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    const int64_t row = m0 + simt_row<CF>(ty, i);
    if (row >= N) continue;
#pragma unroll
    for (int c = 0; c < CF::TN / 2; ++c) {
      const int64_t col = n0 + 2 * tx + 2 * CF::TXN * c;
      if (CV == 2 && col + 1 < M) {
        *reinterpret_cast<double2*>(C + row * M + col) = make_double2(sum[i][2 * c], sum[i][2 * c + 1]);
      } else {
        if (col < M) C[row * M + col] = sum[i][2 * c];
        if (col + 1 < M) C[row * M + col + 1] = sum[i][2 * c + 1];
      }
    }
  }
}

template <class CF, int AV, int BV, int CV, bool FUSED>
cudaError_t launch_kahan_t(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                           cudaStream_t st) {
  constexpr auto kern = kahan_gemm_kernel<CF, AV, BV, CV, FUSED>;
  cudaError_t e = smem_attr_once<kern>(CF::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(cdiv(M, CF::BN) * cdiv(N, CF::BM)));
  kern<<<grid, CF::THREADS, CF::SMEM, st>>>(A, B, C, N, P, M);
  note_launch();
  return cudaGetLastError();
}

template <class CF, bool FUSED>
inline cudaError_t launch_kahan_cfg(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                                    cudaStream_t st) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool av = al(A) && P % 2 == 0, bv = al(B) && M % 2 == 0, cv = al(C) && M % 2 == 0;
  if (av && bv && cv) return launch_kahan_t<CF, 2, 2, 2, FUSED>(A, B, C, N, P, M, st);
  if (bv && cv) return launch_kahan_t<CF, 1, 2, 2, FUSED>(A, B, C, N, P, M, st);
  if (av) return launch_kahan_t<CF, 2, 1, 1, FUSED>(A, B, C, N, P, M, st);
  return launch_kahan_t<CF, 1, 1, 1, FUSED>(A, B, C, N, P, M, st);
}

// fewer 64 x 64 tiles than the two CTA slots per SM (e.g. 1024^3): 32 x 32 tiles, 64 threads of
// 2 x 4 outputs, 4 CTAs per SM -- 0.351 vs 0.373 ms at 1024^3 (profiles/r01/simt_tune_small.jsonl)
using KahanSmall = SimtCfg<32, 32, 2, 4, 3, 4>;
// TMA-fed main loop (simt_tma.cuh) for 16-byte aligned operands with P, M even: 64 x 64 x 32
// tiles, 3 stages -- 157.0 vs 157.5 ms at 8192^3 (profiles/r01/simt_tune_tma_bk32.jsonl)
using KahanTma = SimtCfg<64, 64, 4, 8, 3, 2, 32>;

template <class CF = void, bool FUSED = false>
inline cudaError_t launch_kahan(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                                cudaStream_t st, int sms = 148) {
  if (!std::is_void<CF>::value)
    return launch_kahan_cfg<typename std::conditional<std::is_void<CF>::value, KahanDefault, CF>::type, FUSED>(
        A, B, C, N, P, M, st);
  if (cdiv(N, KahanDefault::BM) * cdiv(M, KahanDefault::BN) < 2 * int64_t(sms))
    return launch_kahan_cfg<KahanSmall, FUSED>(A, B, C, N, P, M, st);
  if (simt_tma_ok(A, B, N, P, M)) return launch_kahan_tma<KahanTma, FUSED>(A, B, C, N, P, M, st);
  return launch_kahan_cfg<KahanDefault, FUSED>(A, B, C, N, P, M, st);
}

}  // namespace mmk
