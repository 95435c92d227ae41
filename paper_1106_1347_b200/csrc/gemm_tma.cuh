// gemm_tma.cuh -- K1 with TMA operand staging: FP64 tensor-core GEMM C = A B (P:102-106,
// NaivStandard; also the batched Strassen base alpha_{m,0}) for operands a TMA tensor
// map can describe (16-byte aligned base, even row pitch and batch stride).  Other operands use
// the cp.async kernel of gemm_dmma.cuh.  Both walk k in the same increasing order, 4 per
// DMMA.8x8x4, so their results are bitwise identical (= the oracle's or_naive_fma, reading R2).
//
//  * Operand tiles arrive by TMA (cp.async.bulk.tensor.3d: columns, rows, batch) into a
//    STAGES-deep ring: A as one [BM rows][16 k] box, B as BN/16 boxes of [16 k][16 columns],
//    all with the 128-byte swizzle (16-byte chunk q of box row r stored at chunk q ^ (r % 8)).
//    Ragged edges are zero-filled by the TMA unit.
//  * One thread issues the copies; completion is counted in bytes on a per-stage "full"
//    mbarrier, and each warp releases a stage on its "empty" mbarrier -- no CTA-wide barrier
//    in the main loop.  Tile kt-1's stage is released and refilled at the top of tile kt (after
//    the loop back edge, so every LDS of it has completed), so STAGES-1 tiles are in flight
//    while a tile is multiplied.
//  * Bank-conflict-free fragment loads under the TMA swizzle come from permuting which tile
//    rows / columns a fragment's lanes own (the 8x8 fragment rows g -> rho(g) =
//    0,2,4,6,1,3,5,7 and columns g -> sigma(g) = 0,1,8,9,2,3,10,11 (+4 for the second fragment
//    of a 16-column box)).  The permutation only changes which lane computes which C entry;
//    every entry is still the k-ordered DMMA chain.
#pragma once
#include "gemm_dmma.cuh"
#include "tma.cuh"

namespace mmk {

struct GemmTmaArgs {
  CUtensorMap mapA, mapB;  // 3-D maps {columns, rows, batch}
  GemmProblem pr;
};

template <class CF>
struct TmaLayout {
  static constexpr int A_TILE = CF::BM * CF::BK, B_TILE = CF::BK * CF::BN;  // doubles
  static constexpr unsigned STAGE_BYTES = unsigned(A_TILE + B_TILE) * 8u;
  static constexpr size_t SMEM = 1024 + size_t(CF::STAGES) * STAGE_BYTES + 2 * CF::STAGES * 8;
  static_assert(CF::BK == 16 || CF::BK == 32, "one or two 128-byte swizzle rows of k per tile row");
  static_assert(CF::WTN % 16 == 0, "a warp covers whole 16-column B boxes");
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int rho8(int g) { return g < 4 ? 2 * g : 2 * (g - 4) + 1; }
__device__ __forceinline__ int sigma8(int g) { return (g & 1) + 8 * ((g >> 1) & 1) + 2 * (g >> 2); }

template <class CF, int CV>
__global__ void __launch_bounds__(CF::THREADS, CF::MIN_BLOCKS) dgemm_tma_kernel(const __grid_constant__ GemmTmaArgs args) {
  using LY = TmaLayout<CF>;
  constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES, MI = CF::MI, NJ = CF::NJ;
  constexpr int NWARPS = CF::WARPS_M * CF::WARPS_N;
  const GemmProblem& pr = args.pr;
  extern __shared__ __align__(1024) unsigned char g_raw[];
  double* sm = reinterpret_cast<double*>(g_raw + ((1024 - (smem_u32(g_raw) & 1023)) & 1023));
  double* As_base = sm;
  double* Bs_base = sm + STAGES * LY::A_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs_base + STAGES * LY::B_TILE);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / CF::WARPS_N, wn = warp % CF::WARPS_N;

  const int64_t bidx = int64_t(blockIdx.y) + int64_t(gridDim.y) * blockIdx.z;
  if (bidx >= pr.batch) return;
  double* __restrict__ C = pr.C + bidx * pr.sC;
  const int tiles_m = int(cdiv(pr.N, BM)), tiles_n = int(cdiv(pr.M, BN));
  const int tile = blockIdx.x;
  const int group = tile / (CF::GROUP_M * tiles_n);
  const int first_m = group * CF::GROUP_M;
  const int gsize = min(tiles_m - first_m, CF::GROUP_M);
  const int in_group = tile - group * CF::GROUP_M * tiles_n;
  const int m0 = (first_m + in_group % gsize) * BM, n0 = (in_group / gsize) * BN;
  constexpr int BK = CF::BK;
  const int KT = int(cdiv(pr.P, BK));

  if (tid == 0) {
    tma_prefetch_desc(&args.mapA);
    tma_prefetch_desc(&args.mapB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NWARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int kt, int s) {  // thread 0 only
    mbar_arrive_expect_tx(full + s, LY::STAGE_BYTES);
#pragma unroll
    for (int h = 0; h < BK / 16; ++h)  // A: [BM rows][16 k] boxes
      tma_load_3d(As_base + s * LY::A_TILE + h * (BM * 16), &args.mapA, kt * BK + 16 * h, m0, int(bidx), full + s);
#pragma unroll
    for (int b = 0; b < BN / 16; ++b)  // B: [BK k][16 columns] boxes
      tma_load_3d(Bs_base + s * LY::B_TILE + b * (BK * 16), &args.mapB, n0 + 16 * b, kt * BK, int(bidx), full + s);
  };
  if (tid == 0)
    for (int s = 0; s < STAGES && s < KT; ++s) issue(s, s);

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // fragment addressing (doubles): A row of fragment mi = wm*WTM + 8 mi + rho(g)
  const int rho = rho8(g);
  if (pr.accumulate) {  // continue each entry's chain from C (same mapping as the epilogue)
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int64_t row = int64_t(m0) + wm * CF::WTM + 8 * mi + rho;
      if (row >= pr.N) continue;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) {
        const int64_t col = int64_t(n0) + wn * CF::WTN + 16 * (nj >> 1) + sigma8(2 * t) + 4 * (nj & 1);
        if (col < pr.M) acc[mi][nj][0] = C[row * pr.ldc + col];
        if (col + 1 < pr.M) acc[mi][nj][1] = C[row * pr.ldc + col + 1];
      }
    }
  }
  const int a_base = (wm * CF::WTM + rho) * 16;
  const int sig0 = sigma8(g), sig1 = sig0 + 4;
  const int b_box0 = (wn * CF::WTN) / 16;

#pragma unroll 1
  for (int kt = 0; kt < KT; ++kt) {
    if (kt >= 1) {
      // Release tile kt-1's stage HERE, after the loop back edge: every DMMA of tile kt-1 has been
      // issued, so every LDS feeding it has returned its data (operand scoreboards).  Releasing at
      // the end of iteration kt-1 instead lets ptxas hoist the arrive above DMMAs whose LDS are
      // still in flight, and the TMA refill can then overwrite the stage under them (a
      // write-after-read race, observed as sporadic wrong 32x32 blocks).
      const int sp = (kt - 1) % STAGES;
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + sp);
      const int kp = kt - 1 + STAGES;
      if (tid == 0 && kp < KT) {  // refill it once every warp has released it
        mbar_wait(empty + sp, unsigned(((kt - 1) / STAGES) & 1));
        issue(kp, sp);
      }
      __syncwarp();
    }
    const int s = kt % STAGES;
    mbar_wait(full + s, unsigned((kt / STAGES) & 1));
    const double* As = As_base + s * LY::A_TILE;
    const double* Bs = Bs_base + s * LY::B_TILE;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + t;
      const int a_off = (k >> 4) * (BM * 16) + (((((k & 15) >> 1) ^ rho)) << 1) + (k & 1);
      const int k8 = k & 7;
      double af[MI], bf[NJ];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = As[a_base + mi * 8 * 16 + a_off];
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) {
        const int sg = (nj & 1) ? sig1 : sig0;
        bf[nj] = Bs[(b_box0 + (nj >> 1)) * (BK * 16) + k * 16 + ((((sg >> 1) ^ k8)) << 1) + (sg & 1)];
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
    }
  }

  // epilogue: fragment (mi, nj) holds C[row][col], C[row][col + 1] with
  // row = m0 + wm*WTM + 8 mi + rho(g), col = n0 + wn*WTN + 16 (nj/2) + sigma_{nj%2}(2t)
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t row = int64_t(m0) + wm * CF::WTM + 8 * mi + rho;
    if (row >= pr.N) continue;
    double* crow = C + row * pr.ldc;
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj) {
      const int64_t col = int64_t(n0) + wn * CF::WTN + 16 * (nj >> 1) + sigma8(2 * t) + 4 * (nj & 1);
      if (CV == 2 && col + 1 < pr.M) {
        *reinterpret_cast<double2*>(crow + col) = make_double2(acc[mi][nj][0], acc[mi][nj][1]);
      } else {
        if (col < pr.M) crow[col] = acc[mi][nj][0];
        if (col + 1 < pr.M) crow[col + 1] = acc[mi][nj][1];
      }
    }
  }
}

// can the operands of pr be described by TMA maps?
inline bool gemm_tma_ok(const GemmProblem& pr) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!tma_encoder()) return false;
  if (!al(pr.A) || !al(pr.B) || pr.lda % 2 || pr.ldb % 2) return false;
  if (pr.batch > 1 && (pr.sA % 2 || pr.sB % 2)) return false;
  if (pr.N > INT32_MAX || pr.P > INT32_MAX || pr.M > INT32_MAX || pr.batch > INT32_MAX) return false;
  return true;
}

template <auto KERN, int THREADS, size_t SMEM>
inline cudaError_t launch_tma_t(const GemmTmaArgs& args, dim3 grid, cudaStream_t st) {
  cudaError_t e = smem_attr_once<KERN>(SMEM);
  if (e != cudaSuccess) return e;
  KERN<<<grid, THREADS, SMEM, st>>>(args);
  note_launch();
  return cudaGetLastError();
}

template <class CF>
inline cudaError_t launch_dgemm_tma(const GemmProblem& pr, cudaStream_t st) {
  using LY = TmaLayout<CF>;
  GemmTmaArgs args;
  args.pr = pr;
  if (!tma_encode_3d(&args.mapA, pr.A, pr.N, pr.P, pr.lda, pr.batch, pr.sA, CF::BM) ||
      !tma_encode_3d(&args.mapB, pr.B, pr.P, pr.M, pr.ldb, pr.batch, pr.sB, CF::BK))
    return cudaErrorInvalidValue;
  const bool cv = (reinterpret_cast<uintptr_t>(pr.C) & 15) == 0 && pr.ldc % 2 == 0 && (pr.batch == 1 || pr.sC % 2 == 0);
  const int64_t tiles = cdiv(pr.N, CF::BM) * cdiv(pr.M, CF::BN);
  dim3 grid(unsigned(tiles), 1, 1);
  if (pr.batch <= 65535) {
    grid.y = unsigned(pr.batch);
  } else {
    grid.y = 65535;
    grid.z = unsigned(cdiv(pr.batch, 65535));
  }
  return cv ? launch_tma_t<dgemm_tma_kernel<CF, 2>, CF::THREADS, LY::SMEM>(args, grid, st)
            : launch_tma_t<dgemm_tma_kernel<CF, 1>, CF::THREADS, LY::SMEM>(args, grid, st);
}

#ifndef GEMM_TMA_GROUP_M
#define GEMM_TMA_GROUP_M 8
#endif
// the production configuration of the TMA path: 64 x 64 x 32 tiles, 4 warps of 32 x 32, double
// buffered, 3 CTAs (12 warps) per SM -- 36.3 TF at 8192^3, 34.4 at 2048^3 on B200 (16-deep tiles,
// 4 stages: 36.26 / 33.8; tools/tune/gemm_tune.cu, profiles/r01/gemm_tune_tma.jsonl,
// gemm_tune_bk32.jsonl; cuBLAS DGEMM: 35.5 at 8192^3)
using GemmTma = GemmCfg<64, 64, 2, 2, 2, 3, 32, GEMM_TMA_GROUP_M>;
// fewer than two waves of 64 x 64 tiles (e.g. 1024^3): 64 x 32 tiles, 2 warps of 32 x 32, 6 CTAs
// per SM -- 28.2 vs 26.6 TF at 1024^3 (profiles/r01/gemm_tune_small.jsonl)
using GemmTmaSmall = GemmCfg<64, 32, 2, 1, 4, 6, 16, GEMM_TMA_GROUP_M>;

// K1 entry: TMA-staged kernel when the operands allow a tensor map, else the cp.async kernel
// (same k order, bitwise the same result)
// tiny problems (each at most 32 x 32 outputs: the leaves of the paper's Strassen plan, orders
// 17..32) batched by the thousand: one warp per 32 x 32 tile instead of a 64 x 64 CTA
// that would leave three quarters of its DMMAs padding
using GemmTmaTiny = GemmCfg<32, 32, 1, 1, 2, 8, 32, GEMM_TMA_GROUP_M>;

inline cudaError_t launch_dgemm(const GemmProblem& pr, cudaStream_t st, int sms = 148) {
  if (gemm_tma_ok(pr)) {
    if (pr.N <= 32 && pr.M <= 32 && pr.batch > 1) return launch_dgemm_tma<GemmTmaTiny>(pr, st);
    const int64_t tiles = cdiv(pr.N, GemmTma::BM) * cdiv(pr.M, GemmTma::BN) * pr.batch;
    if (tiles < 2 * 3 * int64_t(sms)) return launch_dgemm_tma<GemmTmaSmall>(pr, st);
    return launch_dgemm_tma<GemmTma>(pr, st);
  }
  return launch_dgemm_cpasync(pr, st, sms);
}

}  // namespace mmk
