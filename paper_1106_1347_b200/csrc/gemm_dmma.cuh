// gemm_dmma.cuh -- K1: FP64 tensor-core GEMM C = A B for sm_100a (NaivStandard;
// also the Strassen base case alpha_{m,0}, batched over 7^d products).
//
// Design:
//  * CTA tile 128 x 128 x 16 (doubles), 256 threads = 8 warps in a 2 (M) x 4 (N) grid,
//    warp tile 64 x 32 = 8 x 4 DMMA.8x8x4 fragments, 64 FP64 accumulators per thread.
//  * Operands staged global -> shared with cp.async (LDGSTS) in a STAGES-deep ring; 16-byte
//    copies when the operand's rows are 16-byte aligned, else 8-byte copies (e.g. P = 1001).
//    Out-of-range elements are zero-filled by the copy engine.
//  * Shared layouts are XOR-swizzled so every fragment load is bank-conflict free:
//      As[m][k]  at m*16  + (k ^ 4*(m & 3))        (thread (g,t) reads row g, column t)
//      Bs[k][n]  at k*128 + (n ^ 4*(k & 3))        (thread (g,t) reads row t, column g)
//  * k is walked in increasing order, 4 per DMMA, accumulating in registers: each C entry
//    is exactly fma(A_i,P-1 B_P-1,j, ... fma(A_i0 B_0j, 0)) -- the oracle's or_naive_fma.
//    Tile shape, grid and batch never change that order (no split-K), so sharded and
//    unsharded runs agree bitwise.
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
};

namespace gemm {
constexpr int BM = 128, BN = 128, BK = 16;
constexpr int WM = 64, WN = 32;
constexpr int THREADS = 256;
constexpr int GROUP_M = 8;
constexpr int A_ELEMS = BM * BK;  // 2048 doubles
constexpr int B_ELEMS = BK * BN;  // 2048 doubles
template <int STAGES>
constexpr size_t smem_bytes() {
  return size_t(STAGES) * (A_ELEMS + B_ELEMS) * sizeof(double);
}
}  // namespace gemm

template <int AV, int BV>
__device__ __forceinline__ void gemm_load_tile(double* As, double* Bs, const double* __restrict__ A,
                                               const double* __restrict__ B, int64_t lda, int64_t ldb, int64_t N,
                                               int64_t P, int64_t M, int64_t m0, int64_t n0, int64_t k0, int tid) {
  using namespace gemm;
  // ---- A tile: BM rows x BK k
  if (AV == 2) {
#pragma unroll
    for (int i = 0; i < (A_ELEMS / 2) / THREADS; ++i) {  // 4 x 16-byte chunks per thread
      int c = tid + i * THREADS;
      int r = c >> 3, kp = (c & 7) * 2;
      int64_t gm = m0 + r, gk = k0 + kp;
      bool v = (gm < N) && (gk < P);
      const double* src = v ? (A + gm * lda + gk) : A;
      cp_async16(As + r * BK + (kp ^ ((r & 3) << 2)), src, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < A_ELEMS / THREADS; ++i) {  // 8 x 8-byte copies per thread
      int e = tid + i * THREADS;
      int r = e >> 4, kk = e & 15;
      int64_t gm = m0 + r, gk = k0 + kk;
      bool v = (gm < N) && (gk < P);
      const double* src = v ? (A + gm * lda + gk) : A;
      cp_async8(As + r * BK + (kk ^ ((r & 3) << 2)), src, v);
    }
  }
  // ---- B tile: BK k x BN columns
  if (BV == 2) {
#pragma unroll
    for (int i = 0; i < (B_ELEMS / 2) / THREADS; ++i) {
      int c = tid + i * THREADS;
      int kr = c >> 6, np = (c & 63) * 2;
      int64_t gk = k0 + kr, gn = n0 + np;
      bool v = (gk < P) && (gn < M);
      const double* src = v ? (B + gk * ldb + gn) : B;
      cp_async16(Bs + kr * BN + (np ^ ((kr & 3) << 2)), src, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < B_ELEMS / THREADS; ++i) {
      int e = tid + i * THREADS;
      int kr = e >> 7, nn = e & 127;
      int64_t gk = k0 + kr, gn = n0 + nn;
      bool v = (gk < P) && (gn < M);
      const double* src = v ? (B + gk * ldb + gn) : B;
      cp_async8(Bs + kr * BN + (nn ^ ((kr & 3) << 2)), src, v);
    }
  }
}

template <int AV, int BV, int CV, int STAGES>
__global__ void __launch_bounds__(gemm::THREADS, 1) dgemm_dmma_kernel(GemmProblem pr) {
  using namespace gemm;
  extern __shared__ __align__(128) double smem[];
  double* As_base = smem;
  double* Bs_base = smem + STAGES * A_ELEMS;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;

  // ---- batch and tile coordinates
  const int64_t bidx = int64_t(blockIdx.y) + int64_t(gridDim.y) * blockIdx.z;
  if (bidx >= pr.batch) return;
  const double* __restrict__ A = pr.A + bidx * pr.sA;
  const double* __restrict__ B = pr.B + bidx * pr.sB;
  double* __restrict__ C = pr.C + bidx * pr.sC;
  const int tiles_m = int(cdiv(pr.N, BM)), tiles_n = int(cdiv(pr.M, BN));
  const int tile = blockIdx.x;
  const int group = tile / (GROUP_M * tiles_n);
  const int first_m = group * GROUP_M;
  const int gsize = min(tiles_m - first_m, GROUP_M);
  const int in_group = tile - group * GROUP_M * tiles_n;
  const int tm = first_m + in_group % gsize;
  const int tn = in_group / gsize;
  const int64_t m0 = int64_t(tm) * BM, n0 = int64_t(tn) * BN;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = int(cdiv(pr.P, BK));

  // ---- prologue: fill STAGES-1 stages
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT)
      gemm_load_tile<AV, BV>(As_base + s * A_ELEMS, Bs_base + s * B_ELEMS, A, B, pr.lda, pr.ldb, pr.N, pr.P, pr.M,
                             m0, n0, int64_t(s) * BK, tid);
    cp_async_commit();
  }

  // per-thread fragment offsets inside a stage
  const int a_row0 = wm * WM + g;  // + 8*mi
  const int b_col0 = wn * WN + g;  // + 8*nj

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) {
        const int s = nk % STAGES;
        gemm_load_tile<AV, BV>(As_base + s * A_ELEMS, Bs_base + s * B_ELEMS, A, B, pr.lda, pr.ldb, pr.N, pr.P,
                               pr.M, m0, n0, int64_t(nk) * BK, tid);
      }
      cp_async_commit();
    }
    const double* As = As_base + (kt % STAGES) * A_ELEMS;
    const double* Bs = Bs_base + (kt % STAGES) * B_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + t;
      double af[8], bf[4];
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        const int r = a_row0 + 8 * mi;  // r & 3 == g & 3
        af[mi] = As[r * BK + (k ^ ((g & 3) << 2))];
      }
#pragma unroll
      for (int nj = 0; nj < 4; ++nj) {
        const int c = b_col0 + 8 * nj;
        bf[nj] = Bs[k * BN + (c ^ (t << 2))];  // k & 3 == t
      }
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: registers -> global
#pragma unroll
  for (int mi = 0; mi < 8; ++mi) {
    const int64_t row = m0 + a_row0 + 8 * mi;
    if (row >= pr.N) continue;
    double* crow = C + row * pr.ldc;
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) {
      const int64_t col = n0 + b_col0 - g + 8 * nj + 2 * t;
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
constexpr int GEMM_STAGES = 4;

template <int AV, int BV, int CV>
cudaError_t launch_dgemm_t(const GemmProblem& pr, cudaStream_t st) {
  using namespace gemm;
  auto kern = dgemm_dmma_kernel<AV, BV, CV, GEMM_STAGES>;
  const size_t smem = smem_bytes<GEMM_STAGES>();
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t tiles = cdiv(pr.N, BM) * cdiv(pr.M, BN);
  dim3 grid(unsigned(tiles), 1, 1);
  if (pr.batch <= 65535) {
    grid.y = unsigned(pr.batch);
  } else {
    grid.y = 65535;
    grid.z = unsigned(cdiv(pr.batch, 65535));
  }
  kern<<<grid, THREADS, smem, st>>>(pr);
  note_launch();
  return cudaGetLastError();
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// chooses the 16-byte or 8-byte loaders per operand
inline cudaError_t launch_dgemm(const GemmProblem& pr, cudaStream_t st) {
  const bool av = aligned16(pr.A) && (pr.lda % 2 == 0) && (pr.batch == 1 || pr.sA % 2 == 0);
  const bool bv = aligned16(pr.B) && (pr.ldb % 2 == 0) && (pr.batch == 1 || pr.sB % 2 == 0);
  const bool cv = aligned16(pr.C) && (pr.ldc % 2 == 0) && (pr.batch == 1 || pr.sC % 2 == 0);
  if (av && bv && cv) return launch_dgemm_t<2, 2, 2>(pr, st);
  if (av && bv) return launch_dgemm_t<2, 2, 1>(pr, st);
  if (av && cv) return launch_dgemm_t<2, 1, 2>(pr, st);
  if (bv && cv) return launch_dgemm_t<1, 2, 2>(pr, st);
  if (av) return launch_dgemm_t<2, 1, 1>(pr, st);
  if (bv) return launch_dgemm_t<1, 2, 1>(pr, st);
  if (cv) return launch_dgemm_t<1, 1, 2>(pr, st);
  return launch_dgemm_t<1, 1, 1>(pr, st);
}

}  // namespace mmk
