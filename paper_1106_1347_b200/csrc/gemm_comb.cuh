// gemm_comb.cuh -- SURVEY 8(f) NEXT-1 (half of it): the deepest Strassen-Winograd combination
// fused into the epilogue of the batched leaf GEMM.
//
// A CTA owns one output tile position of one parent node q at depth d - 1 and computes the tile
// of its seven children's leaf products H_1 .. H_7 (batch 7q + t) one after the other, the TMA
// ring running on across the child boundaries.  After each child the epilogue folds the tile into
// the parent's four quadrants with exactly the operations and order of comb4:
//   t = 0: r1 = H1                    t = 4: C22 = r2 + H5, r1 = r1 + H5   (= (H8 + H5))
//   t = 1: C11 = r1 + H2              t = 5: C12 = r2 + H6
//   t = 2: r1 = r1 + H3   (= H8)      t = 6: C21 = r1 + H7
//   t = 3: r2 = r1 + H4   (= H9)
// so level d - 1 is written directly (bitwise the separate combination pass) and the 7^d leaf
// products never reach HBM.  The two running tiles r1, r2 (64 doubles per thread) live in TENSOR
// MEMORY, which the FP64 DMMA path leaves idle: each warp parks them in its own 32-lane quadrant
// (tcgen05.st / tcgen05.ld, 32x32b shape, 128 columns per CTA), so the registers hold only the
// 32 accumulators and K1's 3 CTAs per SM are kept.  StrassenNaiv's chains need three
// running tiles in any child order, so only the 15-addition variant is fused.
#pragma once
#include "gemm_tma.cuh"

namespace mmk {

// ---- tensor memory as per-thread scratch (32x32b: thread = TMEM lane, 16 x 32-bit columns)
__device__ __forceinline__ void tm_st16(uint32_t taddr, const double (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};\n" ::"r"(taddr),
      "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])), "r"(__double2hiint(v[1])),
      "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])), "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])),
      "r"(__double2loint(v[4])), "r"(__double2hiint(v[4])), "r"(__double2loint(v[5])), "r"(__double2hiint(v[5])),
      "r"(__double2loint(v[6])), "r"(__double2hiint(v[6])), "r"(__double2loint(v[7])), "r"(__double2hiint(v[7]))
      : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, double (&v)[8]) {
  uint32_t w[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
        "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __hiloint2double(int(w[2 * i + 1]), int(w[2 * i]));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
constexpr uint32_t COMB_TMEM_COLS = 128;  // r1: columns 0..63, r2: 64..127 (64 x 32 bits = 32 doubles each)

struct CombStore {
  double* dst;                      // parent level: node q at dst + q * stride
  int64_t pitch, stride;            // row pitch of a parent node, distance between nodes (elements)
  int64_t rows_valid, cols_valid;   // stored region of a parent (the extraction at level 0)
};

struct GemmCombArgs {
  CUtensorMap mapA, mapB;  // 3-D maps {columns, rows, batch = 7^d}
  GemmProblem pr;          // one leaf problem: N x P times P x M, batch = 7^d
  CombStore out;
};

template <class CF, int CV>
__global__ void __launch_bounds__(CF::THREADS, CF::MIN_BLOCKS) dgemm_tma_comb_kernel(
    const __grid_constant__ GemmCombArgs args) {
  using LY = TmaLayout<CF>;
  constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES, MI = CF::MI, NJ = CF::NJ, BK = CF::BK;
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
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp / CF::WARPS_N, wn = warp % CF::WARPS_N;

  const int64_t q = int64_t(blockIdx.y) + int64_t(gridDim.y) * blockIdx.z;  // parent node
  if (7 * q >= pr.batch) return;
  const int tiles_m = int(cdiv(pr.N, BM)), tiles_n = int(cdiv(pr.M, BN));
  const int tile = blockIdx.x;
  const int group = tile / (CF::GROUP_M * tiles_n);
  const int first_m = group * CF::GROUP_M;
  const int gsize = min(tiles_m - first_m, CF::GROUP_M);
  const int in_group = tile - group * CF::GROUP_M * tiles_n;
  const int m0 = (first_m + in_group % gsize) * BM, n0 = (in_group / gsize) * BN;
  const int KT = int(cdiv(pr.P, BK));
  const int IT = 7 * KT;  // seven children, one k-loop each, one continuous TMA ring

  static_assert(NWARPS == 4 && MI * NJ * 2 == 32, "one TMEM lane quadrant per warp, 32 doubles per tile");
  __shared__ uint32_t tmem_base;
  if (warp == 0) {  // one warp allocates the CTA's 128 TMEM columns and later frees them
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(COMB_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    tma_prefetch_desc(&args.mapA);
    tma_prefetch_desc(&args.mapB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NWARPS);
    }
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // this warp's lane quadrant; r1 of fragment row mi at column 16 mi, r2 at 64 + 16 mi
  const uint32_t tm = tmem_base + (uint32_t(32 * (warp & 3)) << 16);

  auto issue = [&](int it, int s) {  // thread 0 only
    const int kt = it % KT, b = int(7 * q) + it / KT;
    mbar_arrive_expect_tx(full + s, LY::STAGE_BYTES);
#pragma unroll
    for (int h = 0; h < BK / 16; ++h)
      tma_load_3d(As_base + s * LY::A_TILE + h * (BM * 16), &args.mapA, kt * BK + 16 * h, m0, b, full + s);
#pragma unroll
    for (int bb = 0; bb < BN / 16; ++bb)
      tma_load_3d(Bs_base + s * LY::B_TILE + bb * (BK * 16), &args.mapB, n0 + 16 * bb, kt * BK, b, full + s);
  };
  if (tid == 0)
    for (int s = 0; s < STAGES && s < IT; ++s) issue(s, s);

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int rho = rho8(g);
  const int a_base = (wm * CF::WTM + rho) * 16;
  const int sig0 = sigma8(g), sig1 = sig0 + 4;
  const int b_box0 = (wn * CF::WTN) / 16;
  const CombStore& o = args.out;
  double* node = o.dst + q * o.stride;

  // one quadrant value of the parent: quadrant (qa, qb), leaf-tile element (row, col)
  auto put = [&](int qa, int qb, int64_t row, int64_t col, double v0, double v1) {
    const int64_t R = row + qa * pr.N, Cc = col + qb * pr.M;
    if (R >= o.rows_valid) return;
    double* p = node + R * o.pitch + Cc;
    if (CV == 2 && Cc + 1 < o.cols_valid) {
      *reinterpret_cast<double2*>(p) = make_double2(v0, v1);
    } else {
      if (Cc < o.cols_valid) p[0] = v0;
      if (Cc + 1 < o.cols_valid) p[1] = v1;
    }
  };

#pragma unroll 1
  for (int it = 0; it < IT; ++it) {
    if (it >= 1) {  // release / refill it-1's stage after the loop back edge (see gemm_tma.cuh)
      const int sp = (it - 1) % STAGES;
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + sp);
      const int ip = it - 1 + STAGES;
      if (tid == 0 && ip < IT) {
        mbar_wait(empty + sp, unsigned(((it - 1) / STAGES) & 1));
        issue(ip, sp);
      }
      __syncwarp();
    }
    const int s = it % STAGES;
    mbar_wait(full + s, unsigned((it / STAGES) & 1));
    const double* As = As_base + s * LY::A_TILE;
    const double* Bs = Bs_base + s * LY::B_TILE;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + t4;
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
    if ((it + 1) % KT != 0) continue;
    // child t's tile is complete: fold it into the parent's quadrants (comb4's order)
    const int t = it / KT;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int64_t row = int64_t(m0) + wm * CF::WTM + 8 * mi + rho;
      const uint32_t c1 = tm + 16 * mi, c2 = tm + 64 + 16 * mi;
      double h[8], x[8], y[8];
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) {
        h[2 * nj] = acc[mi][nj][0];
        h[2 * nj + 1] = acc[mi][nj][1];
        acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
      }
      auto store = [&](int qa, int qb, const double (&v)[8]) {
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) {
          const int64_t col = int64_t(n0) + wn * CF::WTN + 16 * (nj >> 1) + sigma8(2 * t4) + 4 * (nj & 1);
          if (row < pr.N && col < pr.M) put(qa, qb, row, col, v[2 * nj], v[2 * nj + 1]);
        }
      };
      auto add = [](double (&o)[8], const double (&a)[8], const double (&b)[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = dadd(a[i], b[i]);
      };
      switch (t) {
        case 0: tm_st16(c1, h); break;                                            // r1 = H1
        case 1: tm_ld16(c1, x); add(x, x, h); store(0, 0, x); break;              // C11 = H1 + H2
        case 2: tm_ld16(c1, x); add(x, x, h); tm_st16(c1, x); break;              // r1 = H8 = H1 + H3
        case 3: tm_ld16(c1, x); add(y, x, h); tm_st16(c2, y); break;              // r2 = H9 = H8 + H4
        case 4:
          tm_ld16(c2, y); add(y, y, h); store(1, 1, y);                           // C22 = H9 + H5
          tm_ld16(c1, x); add(x, x, h); tm_st16(c1, x);                           // r1 = H8 + H5
          break;
        case 5: tm_ld16(c2, y); add(y, y, h); store(0, 1, y); break;              // C12 = H9 + H6
        default: tm_ld16(c1, x); add(x, x, h); store(1, 0, x);                    // C21 = (H8 + H5) + H7
      }
    }
    tm_wait_st();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(COMB_TMEM_COLS)
                 : "memory");
  }
}

// the fused configuration: K1's 64 x 64 x 32 tiles, 4 warps, 2 stages, 3 CTAs per SM
using GemmComb = GemmCfg<64, 64, 2, 2, 2, 3, 32, GEMM_TMA_GROUP_M>;

// Leaf products of depth d (pr.batch = 7^d problems N x P x M, operands TMA-describable, M even)
// combined into their 7^(d-1) parents.  Returns cudaErrorNotSupported when the operands do not
// qualify (the caller then runs the separate leaf GEMM and combination pass).
inline cudaError_t launch_dgemm_comb(const GemmProblem& pr, const CombStore& out, cudaStream_t st) {
  using CF = GemmComb;
  using LY = TmaLayout<CF>;
  if (!gemm_tma_ok(pr) || pr.M % 2 != 0 || pr.batch % 7 != 0) return cudaErrorNotSupported;
  GemmCombArgs args;
  args.pr = pr;
  args.out = out;
  if (!tma_encode_3d(&args.mapA, pr.A, pr.N, pr.P, pr.lda, pr.batch, pr.sA, CF::BM) ||
      !tma_encode_3d(&args.mapB, pr.B, pr.P, pr.M, pr.ldb, pr.batch, pr.sB, CF::BK))
    return cudaErrorInvalidValue;
  const bool cv = (reinterpret_cast<uintptr_t>(out.dst) & 15) == 0 && out.pitch % 2 == 0 && out.stride % 2 == 0;
  const int64_t tiles = cdiv(pr.N, CF::BM) * cdiv(pr.M, CF::BN);
  const int64_t nodes = pr.batch / 7;
  dim3 grid(unsigned(tiles), 1, 1);
  if (nodes <= 65535) {
    grid.y = unsigned(nodes);
  } else {
    grid.y = 65535;
    grid.z = unsigned(cdiv(nodes, 65535));
  }
  cudaError_t e;
  if (cv) {
    constexpr auto k = dgemm_tma_comb_kernel<CF, 2>;
    if ((e = smem_attr_once<k>(LY::SMEM)) != cudaSuccess) return e;
    k<<<grid, CF::THREADS, LY::SMEM, st>>>(args);
  } else {
    constexpr auto k = dgemm_tma_comb_kernel<CF, 1>;
    if ((e = smem_attr_once<k>(LY::SMEM)) != cudaSuccess) return e;
    k<<<grid, CF::THREADS, LY::SMEM, st>>>(args);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace mmk
