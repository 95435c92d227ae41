// winograd.cuh -- K3: WinogradOriginal / WinogradScaled.
//
// 0-based form of P:189-192 (reading R5): gamma = floor(P/2),
//   y_i = sum_{j<gamma} A[i][2j] A[i][2j+1]            z_k = sum_{j<gamma} B[2j][k] B[2j+1][k]
//   acc_ik = sum_{j<gamma} (A[i][2j] + B[2j+1][k]) (A[i][2j+1] + B[2j][k])
//   C_ik = (acc_ik - y_i) - z_k  [ + A[i][P-1] B[P-1][k] when P is odd ]
// Sums run in increasing j, every op is a separately rounded FP64 SIMT op, so the result
// equals the oracle's or_winograd_original bit for bit -- required, because on ill-scaled
// inputs (config c3) two equally valid summation orders differ by ~50 in the inf-norm.
//
// WinogradScaled runs the pair-sum kernel on the copies 2^lambda A and 2^-lambda B
// (MultiplyWithScalar; exact power-of-two scalings), which the y/z pass writes while it
// computes y and z on them; lambda is derived on the device from the two norms -- no host round
// trip.
//
// Kernels:
//  * line_kernel<LN_PAIRS> (lines.cuh): y (one lane per row of A) and z (one lane per column of
//    B), sequential sums streamed by bulk copies, HBM-bound; optionally also the scaled copies.
//  * winograd_kernel: SimtCfg tiles (below); the pair loop covers columns 0..2*gamma-1 only
//    (the odd column never enters acc).
#pragma once
#include "lines.cuh"
#include "simt_tile.cuh"
#include "simt_tma.cuh"

#include <type_traits>

namespace mmk {

// ---------------------------------------------------------------- main pair-sum kernel
// 128 x 64 tiles, 128 threads of 8 x 8 outputs, 2 CTAs per SM; 64 x 64 tiles of 4 x 8 when the
// big tiles would leave SMs idle (tools/tune/simt_tune.cu, profiles/r01/simt_tune*.jsonl)
using WinogradDefault = SimtCfg<128, 64, 8, 8, 3, 2>;
using WinogradSmall = SimtCfg<64, 64, 4, 8, 3, 2>;
// cp.async alternative with a finer tile grid (better last-wave fill on some shapes)
using Winograd96 = SimtCfg<96, 64, 6, 8, 2, 3>;
// TMA-fed main loop (simt_tma.cuh) for 16-byte aligned operands with P, M even: 32-deep k tiles,
// double-buffered -- 65.1 vs 65.6 ms (16-deep, 4 stages) at 8192^3
using WinogradTma = SimtCfg<128, 64, 8, 8, 2, 2, 32>;
// ... and a finer tile grid for shapes whose last wave of 128 x 64 tiles is mostly empty (c3: 5.08
// waves; 96 x 64 at 3 CTAs per SM: 4.55), 2.5% slower per tile at 8192^3 (66.7 vs 65.1 ms)
using WinogradTma96 = SimtCfg<96, 64, 6, 8, 3, 3, 16>;
// ... and the small-grid tiles (fewer than two waves of 128 x 64 tiles, e.g. c2 = 1024^3), TMA-fed:
// 0.177 vs 0.191 ms for the cp.async WinogradSmall at 1024^3, bitwise equal (tools/tune/simt_tune.cu
// st, profiles/r02/small_tune.md)
using WinogradTmaSmall = SimtCfg<64, 64, 4, 8, 3, 2, 32>;

// odd P on even-pitch copies (repack.cuh / WinogradScaled's 2^lambda A): the TMA pair kernel with
// the odd term in its epilogue, on the tile grid that fills its last wave better
template <bool FUSED>
inline cudaError_t launch_winograd_pairs_tma_odd_auto(const double* As, int64_t lda, const double* Bs, int64_t ldb,
                                                      double* C, const double* y, const double* z, int64_t N,
                                                      int64_t P, int64_t M, cudaStream_t st, int sms) {
  const int64_t t128 = cdiv(N, WinogradTma::BM) * cdiv(M, WinogradTma::BN);
  const int64_t t96 = cdiv(N, WinogradTma96::BM) * cdiv(M, WinogradTma96::BN);
  const double f128 = double(t128) / double(cdiv(t128, 2 * int64_t(sms)) * 2 * sms);
  const double f96 = 0.975 * double(t96) / double(cdiv(t96, 3 * int64_t(sms)) * 3 * sms);
  if (f96 > f128) return launch_winograd_pairs_tma_odd<WinogradTma96, FUSED>(As, lda, Bs, ldb, C, y, z, N, P, M, st);
  return launch_winograd_pairs_tma_odd<WinogradTma, FUSED>(As, lda, Bs, ldb, C, y, z, N, P, M, st);
}

// The tiles are loaded with kend = 2*gamma: columns/rows >= 2*gamma are zero-filled, so the
// odd column never enters acc.  A zero-filled pair adds (0+0)(0+0) = +0 to acc, which leaves
// acc unchanged (acc starts at +0 and can never become -0), so the last tile needs no guard.
template <class CF, int AV, int BV, int CV, bool FUSED>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB)
    winograd_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                    const double* __restrict__ y, const double* __restrict__ z, int64_t N, int64_t P, int64_t M) {
  constexpr int BK = CF::BK, STAGES = CF::STAGES, TM = CF::TM, TN = CF::TN;
  extern __shared__ __align__(128) double smem[];
  double* As_base = smem;
  double* Bs_base = smem + STAGES * CF::A_ELEMS;
  const int tid = threadIdx.x, tx = tid % CF::TXN, ty = tid / CF::TXN;
  int64_t m0, n0;
  simt_tile_coords(N, M, CF::BM, CF::BN, m0, n0);
  const int64_t Kend = 2 * (P / 2);

  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

  const int KT = int(cdiv(Kend, BK));
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < KT)
      simt_load_tile<CF, AV, BV>(As_base + st * CF::A_ELEMS, Bs_base + st * CF::B_ELEMS, A, B, N, P, M, Kend, m0,
                                 n0, int64_t(st) * BK, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT)
        simt_load_tile<CF, AV, BV>(As_base + (nk % STAGES) * CF::A_ELEMS, Bs_base + (nk % STAGES) * CF::B_ELEMS, A,
                                   B, N, P, M, Kend, m0, n0, int64_t(nk) * BK, tid);
      cp_async_commit();
    }
    const double* As = As_base + (kt % STAGES) * CF::A_ELEMS;
    const double* Bs = Bs_base + (kt % STAGES) * CF::B_ELEMS;
#pragma unroll 2
    for (int jp = 0; jp < BK / 2; ++jp) {
      double a0[TM], a1[TM], b0[TN], b1[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        double2 v = *reinterpret_cast<const double2*>(As + simt_row<CF>(ty, i) * CF::APITCH + 2 * jp);
        a0[i] = v.x;
        a1[i] = v.y;
      }
#pragma unroll
      for (int c = 0; c < TN / 2; ++c) {
        double2 u = *reinterpret_cast<const double2*>(Bs + (2 * jp) * CF::BN + 2 * tx + 2 * CF::TXN * c);
        double2 w = *reinterpret_cast<const double2*>(Bs + (2 * jp + 1) * CF::BN + 2 * tx + 2 * CF::TXN * c);
        b0[2 * c] = u.x;
        b0[2 * c + 1] = u.y;
        b1[2 * c] = w.x;
        b1[2 * c + 1] = w.y;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = wino_pair<FUSED>(acc[i][j], a0[i], a1[i], b0[j], b1[j]);
    }
  }
  cp_async_wait<0>();

  const bool odd = (P & 1) != 0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t row = m0 + simt_row<CF>(ty, i);
    if (row >= N) continue;
    const double yi = y[row];
    const double alast = odd ? A[row * P + (P - 1)] : 0.0;
#pragma unroll
    for (int c = 0; c < TN / 2; ++c) {
      const int64_t col = n0 + 2 * tx + 2 * CF::TXN * c;
      double out[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t cc = col + e;
        double v = 0.0;
        if (cc < M) {
          v = dsub(dsub(acc[i][2 * c + e], yi), z[cc]);             // (acc - y_i) - z_k
          if (odd) v = FUSED ? __fma_rn(alast, B[(P - 1) * M + cc], v)    // + A_{i,P} B_{P,k}
                             : dadd(v, dmul(alast, B[(P - 1) * M + cc]));
        }
        out[e] = v;
      }
      if (CV == 2 && col + 1 < M) {
        *reinterpret_cast<double2*>(C + row * M + col) = make_double2(out[0], out[1]);
      } else {
        if (col < M) C[row * M + col] = out[0];
        if (col + 1 < M) C[row * M + col + 1] = out[1];
      }
    }
  }
}

template <class CF, int AV, int BV, int CV, bool FUSED>
cudaError_t launch_winograd_t(const double* A, const double* B, double* C, const double* y, const double* z,
                              int64_t N, int64_t P, int64_t M, cudaStream_t st) {
  constexpr auto kern = winograd_kernel<CF, AV, BV, CV, FUSED>;
  cudaError_t e = smem_attr_once<kern>(CF::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(cdiv(M, CF::BN) * cdiv(N, CF::BM)));
  kern<<<grid, CF::THREADS, CF::SMEM, st>>>(A, B, C, y, z, N, P, M);
  note_launch();
  return cudaGetLastError();
}

// y, z: device buffers of N and M doubles.
template <class CF, bool FUSED>
inline cudaError_t launch_winograd_main(const double* A, const double* B, double* C, const double* y,
                                        const double* z, int64_t N, int64_t P, int64_t M, cudaStream_t st) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool av = al(A) && P % 2 == 0, bv = al(B) && M % 2 == 0, cv = al(C) && M % 2 == 0;
  if (av && bv && cv) return launch_winograd_t<CF, 2, 2, 2, FUSED>(A, B, C, y, z, N, P, M, st);
  if (bv && cv) return launch_winograd_t<CF, 1, 2, 2, FUSED>(A, B, C, y, z, N, P, M, st);
  return launch_winograd_t<CF, 1, 1, 1, FUSED>(A, B, C, y, z, N, P, M, st);
}

// the pair-sum kernel with the tile configuration chosen by problem size (y, z already computed)
template <class CF = void, bool FUSED = false>
inline cudaError_t launch_winograd_pairs(const double* A, const double* B, double* C, const double* y,
                                         const double* z, int64_t N, int64_t P, int64_t M, cudaStream_t st,
                                         int sms = 148) {
  if (!std::is_void<CF>::value)
    return launch_winograd_main<typename std::conditional<std::is_void<CF>::value, WinogradDefault, CF>::type,
                                FUSED>(A, B, C, y, z, N, P, M, st);
  const int64_t big_tiles = cdiv(N, WinogradDefault::BM) * cdiv(M, WinogradDefault::BN);
  if (big_tiles >= 2 * int64_t(sms)) {
    if (simt_tma_ok(A, B, N, P, M))
      return launch_winograd_pairs_tma<WinogradTma, FUSED>(A, B, C, y, z, N, P, M, st);
    // cp.async path: 128 x 64 tiles at 2 CTAs/SM unless 96 x 64 tiles at 3 CTAs/SM (3% slower per
    // tile) fill their last wave enough better -- e.g. c3, 5.08 vs 4.55 waves: 1.73 vs 1.78 ms
    // (profiles/r01/simt_tune_c3_v2.jsonl)
    const int64_t t96 = cdiv(N, Winograd96::BM) * cdiv(M, Winograd96::BN);
    const double f128 = double(big_tiles) / double(cdiv(big_tiles, 2 * int64_t(sms)) * 2 * sms);
    const double f96 = 0.97 * double(t96) / double(cdiv(t96, 3 * int64_t(sms)) * 3 * sms);
    if (f96 > f128) return launch_winograd_main<Winograd96, FUSED>(A, B, C, y, z, N, P, M, st);
    return launch_winograd_main<WinogradDefault, FUSED>(A, B, C, y, z, N, P, M, st);
  }
  if (simt_tma_ok(A, B, N, P, M))
    return launch_winograd_pairs_tma<WinogradTmaSmall, FUSED>(A, B, C, y, z, N, P, M, st);
  return launch_winograd_main<WinogradSmall, FUSED>(A, B, C, y, z, N, P, M, st);
}

// WinogradOriginal: y/z pass, then the pair sums.  FUSED: the NEXT-3 variant (reading R22)
template <class CF = void, bool FUSED = false>
inline cudaError_t launch_winograd(const double* A, const double* B, double* C, double* y, double* z, int64_t N,
                                   int64_t P, int64_t M, cudaStream_t st, int sms = 148) {
  cudaError_t e = launch_yz(A, B, y, z, N, P, M, nullptr, nullptr, nullptr, nullptr, nullptr, st, FUSED);
  if (e != cudaSuccess) return e;
  return launch_winograd_pairs<CF, FUSED>(A, B, C, y, z, N, P, M, st, sms);
}

// row pitch reserved for the copy 2^lambda A in the WinogradScaled workspace: P, or P + 1 when P is
// odd (a pitch a TMA tensor map can describe)
inline int64_t scaled_pitch(int64_t P) { return P + (P & 1); }

// WinogradScaled: norms (one launch, K4) -> lambda, exact copies 2^lambda A and
// 2^-lambda B, and their y / z (one fused launch) -> pair sums on the copies.  C is not rescaled
// (P:216).  Norms are device {||A||, ||B||} bit patterns: given (e.g. the distributed driver's
// all-reduced ||A||) or, when given == nullptr, computed into `norms`.
template <bool FUSED = false>
inline cudaError_t launch_winograd_scaled(const double* A, const double* B, double* C, int64_t N, int64_t P,
                                          int64_t M, unsigned long long* norms, const unsigned long long* given,
                                          int* lam, double* scale, double* y, double* z, double* As, double* Bs,
                                          cudaStream_t st, int sms = 148) {
  cudaError_t e = cudaSuccess;
  // odd P: the copy of A gets the even pitch P + 1 (scaled_pitch), which a tensor map can
  // describe, so the TMA-fed pair kernel runs with the odd term in its epilogue (c3: the cp.async
  // kernel otherwise)
  const bool odd_tma = (P & 1) && P > 1 && M % 2 == 0 && tma_ok(As, P + 1) && tma_ok(Bs, M) &&
                       cdiv(N, WinogradTma::BM) * cdiv(M, WinogradTma::BN) >= 2 * int64_t(sms) && N <= INT32_MAX &&
                       M <= INT32_MAX;
  const int64_t lda = odd_tma ? P + 1 : P;  // As occupies N x scaled_pitch(P) doubles either way
  if (!given) e = launch_norms(A, N, P, B, P, M, norms, st);
  if (e == cudaSuccess)
    e = launch_yz(A, B, y, z, N, P, M, As, Bs, given ? given : norms, lam, scale, st, FUSED, lda);
  if (e != cudaSuccess) return e;
  if (odd_tma) return launch_winograd_pairs_tma_odd_auto<FUSED>(As, lda, Bs, M, C, y, z, N, P, M, st, sms);
  return launch_winograd_pairs<void, FUSED>(As, Bs, C, y, z, N, P, M, st, sms);
}

}  // namespace mmk
