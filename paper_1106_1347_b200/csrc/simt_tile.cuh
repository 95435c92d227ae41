// simt_tile.cuh -- tile configuration and cp.async tile loader shared by the FP64 SIMT
// kernels (K2 Kahan, K3 Winograd).  Product path only.
#pragma once
#include "common.cuh"

namespace mmk {

// CTA tile BM x BN x BK, thread tile TM x TN, STAGES-deep cp.async ring, MINB CTAs per SM.
// A rows are padded to BK + 2 doubles: (BK + 2) / 2 16-byte units is odd for BK = 16, 32, so the
// row reads of the 4 thread rows of a warp fall in distinct banks.
template <int BM_, int BN_, int TM_, int TN_, int STAGES_, int MINB_, int BK_ = 16>
struct SimtCfg {
  static constexpr int BM = BM_, BN = BN_, TM = TM_, TN = TN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int BK = BK_, APITCH = BK + 2;
  static constexpr int TXN = BN / TN, TYM = BM / TM, THREADS = TXN * TYM;
  static constexpr int A_ELEMS = BM * APITCH, B_ELEMS = BK * BN;
  static constexpr size_t SMEM = size_t(STAGES) * (A_ELEMS + B_ELEMS) * sizeof(double);
  static_assert(TN % 2 == 0, "columns are handled in pairs");
  static_assert((BM * BK / 2) % THREADS == 0 && (BK * BN / 2) % THREADS == 0, "loader split");
};

// A tile (BM x BK, rows padded to APITCH) and B tile (BK x BN); `kend` bounds k (zero fill past it)
template <class CF, int AV, int BV>
__device__ __forceinline__ void simt_load_tile(double* As, double* Bs, const double* __restrict__ A,
                                               const double* __restrict__ B, int64_t N, int64_t P, int64_t M,
                                               int64_t kend, int64_t m0, int64_t n0, int64_t k0, int tid) {
  constexpr int BK = CF::BK, BN = CF::BN, T = CF::THREADS, AP = CF::APITCH;
  if (AV == 2) {
#pragma unroll
    for (int i = 0; i < (CF::BM * BK / 2) / T; ++i) {
      int c = tid + i * T;
      int r = c / (BK / 2), kp = (c % (BK / 2)) * 2;
      int64_t gm = m0 + r, gk = k0 + kp;
      bool v = gm < N && gk < kend;
      cp_async16(As + r * AP + kp, v ? A + gm * P + gk : A, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < (CF::BM * BK) / T; ++i) {
      int e = tid + i * T;
      int r = e / BK, kk = e % BK;
      int64_t gm = m0 + r, gk = k0 + kk;
      bool v = gm < N && gk < kend;
      cp_async8(As + r * AP + kk, v ? A + gm * P + gk : A, v);
    }
  }
  if (BV == 2) {
#pragma unroll
    for (int i = 0; i < (BK * BN / 2) / T; ++i) {
      int c = tid + i * T;
      int kr = c / (BN / 2), np = (c % (BN / 2)) * 2;
      int64_t gk = k0 + kr, gn = n0 + np;
      bool v = gk < kend && gn < M;
      cp_async16(Bs + kr * BN + np, v ? B + gk * M + gn : B, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < (BK * BN) / T; ++i) {
      int e = tid + i * T;
      int kr = e / BN, nn = e % BN;
      int64_t gk = k0 + kr, gn = n0 + nn;
      bool v = gk < kend && gn < M;
      cp_async8(Bs + kr * BN + nn, v ? B + gk * M + gn : B, v);
    }
  }
}

// Output row of thread row-index ty, i-th of its TM rows: rows are interleaved across threads
// (ty + TYM*i) so that the A-row reads of the different ty in one warp fall in different
// bank groups (APITCH = 18 doubles, TYM*... consecutive rows are 144 B apart).
template <class CF>
__device__ __forceinline__ int simt_row(int ty, int i) {
  return ty + CF::TYM * i;
}

// Grouped rasterisation of a 1-D grid of BM x BN tiles (8 tile rows per group) for L2 reuse.
__device__ __forceinline__ void simt_tile_coords(int64_t N, int64_t M, int BM, int BN, int64_t& m0, int64_t& n0) {
#ifndef SIMT_GROUP_M
#define SIMT_GROUP_M 8
#endif
  constexpr int GROUP = SIMT_GROUP_M;
  const int64_t tiles_m = cdiv(N, BM), tiles_n = cdiv(M, BN);
  const int64_t tile = blockIdx.x;
  const int64_t group = tile / (GROUP * tiles_n);
  const int64_t first = group * GROUP;
  const int64_t gsize = (tiles_m - first) < GROUP ? (tiles_m - first) : GROUP;
  const int64_t in_group = tile - group * GROUP * tiles_n;
  m0 = (first + in_group % gsize) * BM;
  n0 = (in_group / gsize) * BN;
}

// One Winograd pair: acc + (a0 + b1)(a1 + b0), the product separately rounded (the
// paper's method) or, FUSED (NEXT-3, reading R22), fma(a0 + b1, a1 + b0, acc).
template <bool FUSED>
__device__ __forceinline__ double wino_pair(double acc, double a0, double a1, double b0, double b1) {
  return FUSED ? __fma_rn(dadd(a0, b1), dadd(a1, b0), acc) : dadd(acc, dmul(dadd(a0, b1), dadd(a1, b0)));
}

}  // namespace mmk
