// gemm_dmma.cuh -- K1: FP64 tensor-core GEMM C = A B for sm_100a (NaivStandard;
// also the Strassen base case alpha_{m,0}, batched over 7^d products).
//
// Design:
//  * CTA tile BM x BN x 16 doubles, WARPS_M x WARPS_N warps, warp tile (BM/WARPS_M) x
//    (BN/WARPS_N) made of 8 x 8 DMMA.8x8x4 fragments accumulating in registers.
//  * Operands staged global -> shared with cp.async (LDGSTS) in a STAGES-deep ring; 16-byte
//    copies when the operand's rows are 16-byte aligned, else 8-byte copies (e.g. P = 1001).
//    Out-of-range elements are zero-filled by the copy engine.
//  * Shared layouts are XOR-swizzled so every fragment load is bank-conflict free:
//      As[m][k]  at m*16 + (k ^ 4*(m & 3))        (thread (g,t) reads row g, column t)
//      Bs[k][n]  at k*BN + (n ^ 4*(k & 3))        (thread (g,t) reads row t, column g)
//  * k is walked in increasing order, 4 per DMMA: each C entry is exactly
//    fma(A[i][P-1], B[P-1][j], ... fma(A[i][0], B[0][j], 0)) -- the oracle's or_naive_fma
//    (probe P3 established DMMA's chain semantics).  No tile shape, grid or batch changes
//    that order (no split-K), so sharded and unsharded runs agree bitwise.
//  * Grid: blockIdx.x = tile id with GROUP_M-row rasterisation for L2 reuse,
//    blockIdx.y/z = batch index (Strassen's 7^d products).
#pragma once
#include "common.cuh"

namespace mmk {

struct GemmProblem {
  const double* A;
  const double* B;
  double* C;
  int64_t N, P, M;        // per-problem sizes
  int64_t lda, ldb, ldc;  // leading dimensions (elements)
  int64_t sA, sB, sC;     // batch strides (elements)
  int64_t batch;
  int accumulate = 0;     // 1: every entry's fma chain starts from C's current value (C = A B + C)
};

template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_, int MIN_BLOCKS_ = 1, int BK_ = 16,
          int GROUP_M_ = 8>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_;
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, STAGES = STAGES_, MIN_BLOCKS = MIN_BLOCKS_;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MI = WTM / 8, NJ = WTN / 8;
  static constexpr int A_ELEMS = BM * BK, B_ELEMS = BK * BN;
  static constexpr int GROUP_M = GROUP_M_;  // tile rows per rasterisation group (L2 reuse)
  static constexpr size_t SMEM = size_t(STAGES) * (A_ELEMS + B_ELEMS) * sizeof(double);
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile must be a multiple of the 8x8 fragment");
  static_assert((A_ELEMS / 2) % THREADS == 0 && (B_ELEMS / 2) % THREADS == 0, "loader split");
  static_assert(BN % 16 == 0, "B swizzle needs BN % 16 == 0");
  static_assert(BK == 16 || BK == 32, "A swizzle assumes 16- or 32-double rows");
};

// the production configuration: 128 x 64 tiles, 4 warps of 64 x 32, 4 stages, 2 CTAs per SM
// (tools/tune/gemm_tune.cu compares the alternatives; profiles/r01/gemm_tune*.jsonl).
// Two independent CTAs per SM let one CTA's barrier/refill overlap the other's DMMAs.
using GemmDefault = GemmCfg<128, 64, 2, 2, 4, 2>;
// small problems (fewer than two full waves of default tiles) and every odd-pitch A: 64 x 64
// tiles, 4 warps of 32 x 32, 3 stages, 3 CTAs per SM (4 CTAs per SM cap the registers at 128:
// c3 4096 x 1001 x 3000 0.795 vs 0.848 ms, 8192 x 8191 x 8192 33.4 vs 35.5 ms, 2048 x 2047 x 2048
// 0.550 vs 0.587 ms; tools/tune/gemm_tune.cu c3, profiles/r01/gemm_tune_oddP.jsonl)
using GemmSmall = GemmCfg<64, 64, 2, 2, 3, 3>;

template <class CF, int AV, int BV>
__device__ __forceinline__ void gemm_load_tile(double* As, double* Bs, const double* __restrict__ A,
                                               const double* __restrict__ B, int64_t lda, int64_t ldb, int64_t N,
                                               int64_t P, int64_t M, int64_t m0, int64_t n0, int64_t k0, int tid) {
  constexpr int BK = CF::BK, BN = CF::BN, T = CF::THREADS;
  if (AV == 2) {
#pragma unroll
    for (int i = 0; i < (CF::A_ELEMS / 2) / T; ++i) {
      int c = tid + i * T;
      int r = c / (BK / 2), kp = (c % (BK / 2)) * 2;
      int64_t gm = m0 + r, gk = k0 + kp;
      bool v = (gm < N) && (gk < P);
      cp_async16(As + r * BK + (kp ^ ((r & 3) << 2)), v ? (A + gm * lda + gk) : A, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < CF::A_ELEMS / T; ++i) {
      int e = tid + i * T;
      int r = e / BK, kk = e % BK;
      int64_t gm = m0 + r, gk = k0 + kk;
      bool v = (gm < N) && (gk < P);
      cp_async8(As + r * BK + (kk ^ ((r & 3) << 2)), v ? (A + gm * lda + gk) : A, v);
    }
  }
  if (BV == 2) {
#pragma unroll
    for (int i = 0; i < (CF::B_ELEMS / 2) / T; ++i) {
      int c = tid + i * T;
      int kr = c / (BN / 2), np = (c % (BN / 2)) * 2;
      int64_t gk = k0 + kr, gn = n0 + np;
      bool v = (gk < P) && (gn < M);
      cp_async16(Bs + kr * BN + (np ^ ((kr & 3) << 2)), v ? (B + gk * ldb + gn) : B, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < CF::B_ELEMS / T; ++i) {
      int e = tid + i * T;
      int kr = e / BN, nn = e % BN;
      int64_t gk = k0 + kr, gn = n0 + nn;
      bool v = (gk < P) && (gn < M);
      cp_async8(Bs + kr * BN + (nn ^ ((kr & 3) << 2)), v ? (B + gk * ldb + gn) : B, v);
    }
  }
}

template <class CF, int AV, int BV, int CV>
__global__ void __launch_bounds__(CF::THREADS, CF::MIN_BLOCKS) dgemm_dmma_kernel(GemmProblem pr) {
  constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, STAGES = CF::STAGES, MI = CF::MI, NJ = CF::NJ;
  extern __shared__ __align__(128) double smem[];
  double* As_base = smem;
  double* Bs_base = smem + STAGES * CF::A_ELEMS;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / CF::WARPS_N, wn = warp % CF::WARPS_N;

  const int64_t bidx = int64_t(blockIdx.y) + int64_t(gridDim.y) * blockIdx.z;
  if (bidx >= pr.batch) return;
  const double* __restrict__ A = pr.A + bidx * pr.sA;
  const double* __restrict__ B = pr.B + bidx * pr.sB;
  double* __restrict__ C = pr.C + bidx * pr.sC;
  const int tiles_m = int(cdiv(pr.N, BM)), tiles_n = int(cdiv(pr.M, BN));
  const int tile = blockIdx.x;
  const int group = tile / (CF::GROUP_M * tiles_n);
  const int first_m = group * CF::GROUP_M;
  const int gsize = min(tiles_m - first_m, CF::GROUP_M);
  const int in_group = tile - group * CF::GROUP_M * tiles_n;
  const int64_t m0 = int64_t(first_m + in_group % gsize) * BM, n0 = int64_t(in_group / gsize) * BN;

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (pr.accumulate) {  // continue each entry's chain from C (same mapping as the epilogue)
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int64_t row = m0 + wm * CF::WTM + g + 8 * mi;
      if (row >= pr.N) continue;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) {
        const int64_t col = n0 + wn * CF::WTN + 8 * nj + 2 * t;
        if (col < pr.M) acc[mi][nj][0] = C[row * pr.ldc + col];
        if (col + 1 < pr.M) acc[mi][nj][1] = C[row * pr.ldc + col + 1];
      }
    }
  }

  const int KT = int(cdiv(pr.P, BK));
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT)
      gemm_load_tile<CF, AV, BV>(As_base + s * CF::A_ELEMS, Bs_base + s * CF::B_ELEMS, A, B, pr.lda, pr.ldb, pr.N,
                                 pr.P, pr.M, m0, n0, int64_t(s) * BK, tid);
    cp_async_commit();
  }

  const int a_row0 = wm * CF::WTM + g;  // + 8*mi ; (a_row0 + 8 mi) & 3 == g & 3
  const int b_col0 = wn * CF::WTN + g;  // + 8*nj
  const int a_sw = (g & 3) << 2, b_sw = t << 2;

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) {
        const int s = nk % STAGES;
        gemm_load_tile<CF, AV, BV>(As_base + s * CF::A_ELEMS, Bs_base + s * CF::B_ELEMS, A, B, pr.lda, pr.ldb,
                                   pr.N, pr.P, pr.M, m0, n0, int64_t(nk) * BK, tid);
      }
      cp_async_commit();
    }
    const double* As = As_base + (kt % STAGES) * CF::A_ELEMS;
    const double* Bs = Bs_base + (kt % STAGES) * CF::B_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + t;
      double af[MI], bf[NJ];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = As[(a_row0 + 8 * mi) * BK + (k ^ a_sw)];
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) bf[nj] = Bs[k * BN + ((b_col0 + 8 * nj) ^ b_sw)];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t row = m0 + a_row0 + 8 * mi;
    if (row >= pr.N) continue;
    double* crow = C + row * pr.ldc;
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj) {
      const int64_t col = n0 + wn * CF::WTN + 8 * nj + 2 * t;
      if (CV == 2 && col + 1 < pr.M) {
        *reinterpret_cast<double2*>(crow + col) = make_double2(acc[mi][nj][0], acc[mi][nj][1]);
      } else {
        if (col < pr.M) crow[col] = acc[mi][nj][0];
        if (col + 1 < pr.M) crow[col + 1] = acc[mi][nj][1];
      }
    }
  }
}

// ---- host-side launcher ------------------------------------------------------
template <class CF, int AV, int BV, int CV>
cudaError_t launch_dgemm_t(const GemmProblem& pr, cudaStream_t st) {
  constexpr auto kern = dgemm_dmma_kernel<CF, AV, BV, CV>;
  cudaError_t e = smem_attr_once<kern>(CF::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles = cdiv(pr.N, CF::BM) * cdiv(pr.M, CF::BN);
  dim3 grid(unsigned(tiles), 1, 1);
  if (pr.batch <= 65535) {
    grid.y = unsigned(pr.batch);
  } else {
    grid.y = 65535;
    grid.z = unsigned(cdiv(pr.batch, 65535));
  }
  kern<<<grid, CF::THREADS, CF::SMEM, st>>>(pr);
  note_launch();
  return cudaGetLastError();
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// chooses the 16-byte or 8-byte loaders per operand
template <class CF>
inline cudaError_t launch_dgemm_cfg(const GemmProblem& pr, cudaStream_t st) {
  const bool av = aligned16(pr.A) && (pr.lda % 2 == 0) && (pr.batch == 1 || pr.sA % 2 == 0);
  const bool bv = aligned16(pr.B) && (pr.ldb % 2 == 0) && (pr.batch == 1 || pr.sB % 2 == 0);
  const bool cv = aligned16(pr.C) && (pr.ldc % 2 == 0) && (pr.batch == 1 || pr.sC % 2 == 0);
  if (av && bv && cv) return launch_dgemm_t<CF, 2, 2, 2>(pr, st);
  if (av && bv) return launch_dgemm_t<CF, 2, 2, 1>(pr, st);
  if (av && cv) return launch_dgemm_t<CF, 2, 1, 2>(pr, st);
  if (bv && cv) return launch_dgemm_t<CF, 1, 2, 2>(pr, st);
  if (av) return launch_dgemm_t<CF, 2, 1, 1>(pr, st);
  if (bv) return launch_dgemm_t<CF, 1, 2, 1>(pr, st);
  if (cv) return launch_dgemm_t<CF, 1, 1, 2>(pr, st);
  return launch_dgemm_t<CF, 1, 1, 1>(pr, st);
}

// tile configuration by problem size (the per-entry arithmetic is identical for both)
// Operands reaching this path are those TMA cannot describe; when A's rows are only 8-byte
// aligned (odd P) the 64 x 64 configuration is faster than 128 x 64 at every size measured (c3
// 4096 x 1001 x 3000: 0.85 vs 1.06 ms at 4 CTAs per SM, 0.795 ms at 3; 8192 x 8191 x 8192: 30.9 vs 27.9 TF;
// profiles/r01/gemm_tune_oddP.jsonl)
// tiny batched problems with an odd pitch (the paper plan's order-17 leaves): one warp per
// 32 x 32 tile
using GemmTiny = GemmCfg<32, 32, 1, 1, 4, 8>;

inline cudaError_t launch_dgemm_cpasync(const GemmProblem& pr, cudaStream_t st, int sms = 148) {
  if (pr.N <= 32 && pr.M <= 32 && pr.batch > 1) return launch_dgemm_cfg<GemmTiny>(pr, st);
  const bool a16 = (reinterpret_cast<uintptr_t>(pr.A) & 15) == 0 && pr.lda % 2 == 0 && (pr.batch == 1 || pr.sA % 2 == 0);
  const int64_t tiles = cdiv(pr.N, GemmDefault::BM) * cdiv(pr.M, GemmDefault::BN) * pr.batch;
  if (a16 && tiles >= 4 * int64_t(sms)) return launch_dgemm_cfg<GemmDefault>(pr, st);
  return launch_dgemm_cfg<GemmSmall>(pr, st);
}

}  // namespace mmk
