// simt_tma.cuh -- TMA-fed main loops of the FP64 SIMT kernels: K2 Kahan and
// K3 Winograd pair sums, for operands a tensor map can describe (16-byte aligned,
// even pitches: P and M even).  Other operands use the cp.async kernels of kahan.cuh /
// winograd.cuh.  Measured at 8192^3 with 32-deep k tiles (profiles/r01/simt_tune_tma_bk32.jsonl):
// Winograd 65.1 ms vs 67.4 ms with cp.async, Kahan 157.0 ms vs 157.5 ms.  (With 16-deep tiles
// the TMA Kahan lost, 161.7 vs 157.8 ms: the swizzled addressing cost more than the barriers it
// removed; profiles/r01/simt_tune_tma.jsonl.)
// Per output entry the arithmetic and its order are exactly those kernels' (and the
// oracle's): only the operand staging differs, so results are bitwise identical.
//
//  * A tile = BK/16 TMA boxes [BM rows][16 k], B tile = BN/16 boxes [BK k][16 columns], 128-byte
//    swizzle (16-byte chunk q of box row r at chunk q ^ (r % 8)).  Thread (ty, tx) reads rows
//    ty + TYM i of A (4 consecutive rows per warp -> 4 distinct chunks, broadcast over tx) and
//    the column pairs 2 tx + 16 c of B (box c, chunk tx -> 8 distinct chunks): conflict free.
//  * One thread issues the copies into a STAGES-deep ring with per-stage full (expect_tx) and
//    empty (one arrival per warp) mbarriers: no CTA-wide barrier in the main loop; a stage is
//    released at the top of the next tile (after every read of it has completed).
//  * TMA zero-fills out-of-range rows/columns; the Kahan k-loop still stops exactly at P (a
//    zero term is not a no-op for the compensated update) and Winograd's pair loop ends at
//    gamma = P/2 (P is even on this path).
#pragma once
#include "simt_tile.cuh"
#include "tma.cuh"

#ifndef MMK_WINO_SCHED  // inner-loop order of K3 (tools/tune/simt_tune.cu compares them)
#define MMK_WINO_SCHED 0
#endif
#ifndef MMK_KAHAN_UNROLL
#define MMK_KAHAN_UNROLL 4
#endif
#ifndef MMK_WINO_UNROLL
#define MMK_WINO_UNROLL 8
#endif
#ifndef MMK_WINO_UNROLL_EX
#define MMK_WINO_UNROLL_EX 4
#endif

namespace mmk {

constexpr int kWinoUnroll = MMK_WINO_UNROLL, kWinoUnrollEx = MMK_WINO_UNROLL_EX, kKahanUnroll = MMK_KAHAN_UNROLL;

struct SimtTmaArgs {
  CUtensorMap mapA, mapB;
  const double* A;  // for Winograd's epilogue (odd P never takes this path, kept for symmetry)
  const double* B;
  double* C;
  const double* y;
  const double* z;
  int64_t N, P, M;
  // k-panel continuation (mm_kahan_ex / mm_winograd_ex): SIMT_EX_ACC starts
  // every entry's running state from C (and Kahan's err from E) instead of +0; SIMT_EX_KEEP
  // stores the running state (Kahan: err into E; Winograd: the raw pair sum, no epilogue)
  double* E;
  int flags;
  // WinogradScaled with odd P on its even-pitch copies: the pair loop covers the P - 1 columns
  // the maps describe (P here), the epilogue adds A[i][P] B[P][k] read at pitches lda / ldb
  int odd;
  int64_t lda, ldb;
};
constexpr int SIMT_EX_ACC = 1, SIMT_EX_KEEP = 2;

template <class CF>
struct SimtTmaLayout {
  static constexpr int A_TILE = CF::BM * CF::BK, B_TILE = CF::BK * CF::BN;
  static constexpr unsigned STAGE_BYTES = unsigned(A_TILE + B_TILE) * 8u;
  static constexpr size_t SMEM = 1024 + size_t(CF::STAGES) * STAGE_BYTES + 2 * CF::STAGES * 8;
  static_assert(CF::TXN == 8, "a warp's 8 column pairs must fill one 16-column TMA box row");
  static_assert(CF::BK == 16 || CF::BK == 32, "tiles of 16 or 32 k (one or two 128-byte swizzle rows)");
};

// A[row][k] in the swizzled boxes [k/16][BM][16]
template <class CF>
__device__ __forceinline__ int sw_a(int row, int k) {
  return (k >> 4) * (CF::BM * 16) + row * 16 + (((((k & 15) >> 1) ^ (row & 7))) << 1) + (k & 1);
}
// B[k][2 tx + 16 c .. +1] (a 16-byte pair) in box c of [BK][16]
template <class CF>
__device__ __forceinline__ int sw_b(int k, int tx, int c) {
  return c * (CF::BK * 16) + k * 16 + ((tx ^ (k & 7)) << 1);
}

template <class CF>
struct SimtPipe {
  using LY = SimtTmaLayout<CF>;
  double* As_base;
  double* Bs_base;
  uint64_t* full;
  uint64_t* empty;
  int m0, n0, KT;

  __device__ __forceinline__ void init(unsigned char* raw, int m0_, int n0_, int KT_) {
    double* sm = reinterpret_cast<double*>(raw + ((1024 - (smem_u32(raw) & 1023)) & 1023));
    As_base = sm;
    Bs_base = sm + CF::STAGES * LY::A_TILE;
    full = reinterpret_cast<uint64_t*>(Bs_base + CF::STAGES * LY::B_TILE);
    empty = full + CF::STAGES;
    m0 = m0_;
    n0 = n0_;
    KT = KT_;
  }
  __device__ __forceinline__ void issue(const SimtTmaArgs& a, int kt, int s) {
    mbar_arrive_expect_tx(full + s, LY::STAGE_BYTES);
#pragma unroll
    for (int h = 0; h < CF::BK / 16; ++h)
      tma_load_2d(As_base + s * LY::A_TILE + h * (CF::BM * 16), &a.mapA, kt * CF::BK + 16 * h, m0, full + s);
#pragma unroll
    for (int c = 0; c < CF::BN / 16; ++c)
      tma_load_2d(Bs_base + s * LY::B_TILE + c * (CF::BK * 16), &a.mapB, n0 + 16 * c, kt * CF::BK, full + s);
  }
  // barriers + prologue; every thread calls it
  __device__ __forceinline__ void start(const SimtTmaArgs& a) {
    if (threadIdx.x == 0) {
      tma_prefetch_desc(&a.mapA);
      tma_prefetch_desc(&a.mapB);
      for (int s = 0; s < CF::STAGES; ++s) {
        mbar_init(full + s, 1);
        mbar_init(empty + s, CF::THREADS / 32);
      }
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int s = 0; s < CF::STAGES && s < KT; ++s) issue(a, s, s);
  }
  // top of tile kt: release tile kt-1's stage (after the loop back edge every FP64 op reading
  // its LDS results has issued, so the loads have completed -- see gemm_tma.cuh), refill it
  // once every warp released it, then wait for tile kt; returns its stage
  __device__ __forceinline__ int acquire(const SimtTmaArgs& a, int kt) {
    if (kt >= 1) {
      const int sp = (kt - 1) % CF::STAGES;
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(empty + sp);
      const int kp = kt - 1 + CF::STAGES;
      if (threadIdx.x == 0 && kp < KT) {
        mbar_wait(empty + sp, unsigned(((kt - 1) / CF::STAGES) & 1));
        issue(a, kp, sp);
      }
      __syncwarp();  // reconverge warp 0 before the tile's math (else lanes 1-31 run it apart)
    }
    const int s = kt % CF::STAGES;
    mbar_wait(full + s, unsigned((kt / CF::STAGES) & 1));
    return s;
  }
};

// ---------------------------------------------------------------- K2 Kahan, TMA-fed
template <class CF, int CV, bool FUSED>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB) kahan_tma_kernel(const __grid_constant__ SimtTmaArgs a) {
  using LY = SimtTmaLayout<CF>;
  extern __shared__ __align__(1024) unsigned char k_raw[];
  const int tid = threadIdx.x, tx = tid % CF::TXN, ty = tid / CF::TXN;
  int64_t m0, n0;
  simt_tile_coords(a.N, a.M, CF::BM, CF::BN, m0, n0);
  SimtPipe<CF> pp;
  pp.init(k_raw, int(m0), int(n0), int(cdiv(a.P, CF::BK)));
  pp.start(a);

  double sum[CF::TM][CF::TN], err[CF::TM][CF::TN];
#pragma unroll
  for (int i = 0; i < CF::TM; ++i)
#pragma unroll
    for (int j = 0; j < CF::TN; ++j) sum[i][j] = err[i][j] = 0.0;
  if (a.flags & SIMT_EX_ACC) {  // continue each entry's (sum, err) from the previous k-panel
#pragma unroll
    for (int i = 0; i < CF::TM; ++i) {
      const int64_t row = m0 + simt_row<CF>(ty, i);
#pragma unroll
      for (int j = 0; j < CF::TN; ++j) {
        const int64_t col = n0 + 2 * tx + 2 * CF::TXN * (j / 2) + (j & 1);
        if (row < a.N && col < a.M) {
          sum[i][j] = a.C[row * a.M + col];
          err[i][j] = a.E[row * a.M + col];
        }
      }
    }
  }

  // per k: B's TN values stay in registers, A's value of row i is read just before its TN
  // updates (156.5 vs 156.7 ms with all of A's values loaded up front; kahan_sched.log)
  auto step = [&](const double* As, const double* Bs, int kk) {
    double bv[CF::TN];
#pragma unroll
    for (int c = 0; c < CF::TN / 2; ++c) {
      const double2 v = *reinterpret_cast<const double2*>(Bs + sw_b<CF>(kk, tx, c));
      bv[2 * c] = v.x;
      bv[2 * c + 1] = v.y;
    }
#pragma unroll
    for (int i = 0; i < CF::TM; ++i) {
      const double ai = As[sw_a<CF>(simt_row<CF>(ty, i), kk)];
#pragma unroll
      for (int j = 0; j < CF::TN; ++j) {  // the update of P:122-132, every op separately rounded
        // (FUSED, NEXT-3 / reading R22: err = fma(a, b, err))
        double e = FUSED ? __fma_rn(ai, bv[j], err[i][j]) : dadd(err[i][j], dmul(ai, bv[j]));
        const double t = dadd(sum[i][j], e);
        e = dadd(dsub(sum[i][j], t), e);
        sum[i][j] = t;
        err[i][j] = e;
      }
    }
  };

#pragma unroll 1
  for (int kt = 0; kt < pp.KT; ++kt) {
    const int s = pp.acquire(a, kt);
    const double* As = pp.As_base + s * LY::A_TILE;
    const double* Bs = pp.Bs_base + s * LY::B_TILE;
    const int64_t k0 = int64_t(kt) * CF::BK;
    if (k0 + CF::BK <= a.P) {
#pragma unroll kKahanUnroll
      for (int kk = 0; kk < CF::BK; ++kk) step(As, Bs, kk);
    } else {
      const int kmax = int(a.P - k0);  // stop exactly at P
      for (int kk = 0; kk < kmax; ++kk) step(As, Bs, kk);
    }
  }

#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    const int64_t row = m0 + simt_row<CF>(ty, i);
    if (row >= a.N) continue;
#pragma unroll
    for (int c = 0; c < CF::TN / 2; ++c) {
      const int64_t col = n0 + 2 * tx + 2 * CF::TXN * c;
      if (CV == 2 && col + 1 < a.M) {
        *reinterpret_cast<double2*>(a.C + row * a.M + col) = make_double2(sum[i][2 * c], sum[i][2 * c + 1]);
      } else {
        if (col < a.M) a.C[row * a.M + col] = sum[i][2 * c];
        if (col + 1 < a.M) a.C[row * a.M + col + 1] = sum[i][2 * c + 1];
      }
      if (a.flags & SIMT_EX_KEEP) {
        if (col < a.M) a.E[row * a.M + col] = err[i][2 * c];
        if (col + 1 < a.M) a.E[row * a.M + col + 1] = err[i][2 * c + 1];
      }
    }
  }
}

// ---------------------------------------------------------------- K3 Winograd pair sums, TMA-fed (P even)
template <class CF, int CV, bool FUSED, bool EX = false>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB) winograd_tma_kernel(const __grid_constant__ SimtTmaArgs a) {
  using LY = SimtTmaLayout<CF>;
  constexpr int TM = CF::TM, TN = CF::TN;
  extern __shared__ __align__(1024) unsigned char w_raw[];
  const int tid = threadIdx.x, tx = tid % CF::TXN, ty = tid / CF::TXN;
  int64_t m0, n0;
  simt_tile_coords(a.N, a.M, CF::BM, CF::BN, m0, n0);
  SimtPipe<CF> pp;
  pp.init(w_raw, int(m0), int(n0), int(cdiv(a.P, CF::BK)));  // P even: 2 gamma = P
  pp.start(a);

  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
  if (EX && (a.flags & SIMT_EX_ACC)) {  // continue each entry's pair sum from the previous k-panel
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t row = m0 + simt_row<CF>(ty, i);
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t col = n0 + 2 * tx + 2 * CF::TXN * (j / 2) + (j & 1);
        if (row < a.N && col < a.M) acc[i][j] = a.C[row * a.M + col];
      }
    }
  }

#pragma unroll 1
  for (int kt = 0; kt < pp.KT; ++kt) {
    const int s = pp.acquire(a, kt);
    const double* As = pp.As_base + s * LY::A_TILE;
    const double* Bs = pp.Bs_base + s * LY::B_TILE;
    // a zero-filled pair past P adds (0+0)(0+0) = +0 to acc, which leaves acc unchanged
    // (acc starts at +0 and can never become -0), so the last tile needs no guard
    // per pair: B's TN column pairs stay in registers, A's pair of row i is read just before its
    // TN entries (64.70 vs 65.02 ms with all of A's pairs loaded up front; winograd_sched.log)
    // 8 pairs per unrolled body on the 2-CTA tiles: 63.9 vs 64.7 ms at 8192^3 with 2
    // (tools/tune/simt_tune.cu x, profiles/r02/winograd_unroll.log); the 3-CTA tiles keep 2.  The
    // k-panel variant (EX) takes 4: the g = 8 c4 shard's four 2048-deep panels 8.19 vs 8.50 ms with
    // 8, 32.20 vs 32.58 at 4096 rows, equal at 8192 (simt_tune e, profiles/r02/winograd_unroll_ex.jsonl)
    constexpr int UNR = CF::MINB >= 3 ? 2 : (EX ? kWinoUnrollEx : kWinoUnroll);
#pragma unroll UNR
    for (int jp = 0; jp < CF::BK / 2; ++jp) {
      double b0[TN], b1[TN];
#pragma unroll
      for (int c = 0; c < TN / 2; ++c) {
        const double2 u = *reinterpret_cast<const double2*>(Bs + sw_b<CF>(2 * jp, tx, c));
        const double2 w = *reinterpret_cast<const double2*>(Bs + sw_b<CF>(2 * jp + 1, tx, c));
        b0[2 * c] = u.x;
        b0[2 * c + 1] = u.y;
        b1[2 * c] = w.x;
        b1[2 * c + 1] = w.y;
      }
#if MMK_WINO_SCHED == 1
      // per row: the 2 TN sums first, then the TN products, then the TN accumulations
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const double2 v = *reinterpret_cast<const double2*>(As + sw_a<CF>(simt_row<CF>(ty, i), 2 * jp));
        double s1[TN], s2[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j) s1[j] = dadd(v.x, b1[j]);
#pragma unroll
        for (int j = 0; j < TN; ++j) s2[j] = dadd(v.y, b0[j]);
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          if (FUSED) acc[i][j] = __fma_rn(s1[j], s2[j], acc[i][j]);
          else s1[j] = dmul(s1[j], s2[j]);
        }
        if (!FUSED) {
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = dadd(acc[i][j], s1[j]);
        }
      }
#elif MMK_WINO_SCHED == 2
      // two rows interleaved: row i's products wait on sums issued a row-pair earlier
#pragma unroll
      for (int i = 0; i < TM; i += 2) {
        const double2 v = *reinterpret_cast<const double2*>(As + sw_a<CF>(simt_row<CF>(ty, i), 2 * jp));
        const double2 w = *reinterpret_cast<const double2*>(As + sw_a<CF>(simt_row<CF>(ty, i + 1), 2 * jp));
        double s1[2][TN], s2[2][TN];
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          s1[0][j] = dadd(v.x, b1[j]);
          s1[1][j] = dadd(w.x, b1[j]);
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          s2[0][j] = dadd(v.y, b0[j]);
          s2[1][j] = dadd(w.y, b0[j]);
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i + r][j] = FUSED ? __fma_rn(s1[r][j], s2[r][j], acc[i + r][j])
                                                              : dadd(acc[i + r][j], dmul(s1[r][j], s2[r][j]));
      }
#else
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const double2 v = *reinterpret_cast<const double2*>(As + sw_a<CF>(simt_row<CF>(ty, i), 2 * jp));
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = wino_pair<FUSED>(acc[i][j], v.x, v.y, b0[j], b1[j]);
      }
#endif
    }
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t row = m0 + simt_row<CF>(ty, i);
    if (row >= a.N) continue;
    const bool keep = EX && (a.flags & SIMT_EX_KEEP);  // raw pair sums for the next k-panel
    const double yi = keep ? 0.0 : a.y[row];
#pragma unroll
    for (int c = 0; c < TN / 2; ++c) {
      const int64_t col = n0 + 2 * tx + 2 * CF::TXN * c;
      double out[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t cc = col + e;
        out[e] = cc >= a.M ? 0.0 : keep ? acc[i][2 * c + e] : dsub(dsub(acc[i][2 * c + e], yi), a.z[cc]);
        if (!EX && a.odd && cc < a.M) {  // + A_{i,P} B_{P,k}, after -y -z
          const double al = a.A[row * a.lda + a.P], bl = a.B[a.P * a.ldb + cc];
          out[e] = FUSED ? __fma_rn(al, bl, out[e]) : dadd(out[e], dmul(al, bl));
        }
      }  // (acc - y_i) - z_k
      if (CV == 2 && col + 1 < a.M) {
        *reinterpret_cast<double2*>(a.C + row * a.M + col) = make_double2(out[0], out[1]);
      } else {
        if (col < a.M) a.C[row * a.M + col] = out[0];
        if (col + 1 < a.M) a.C[row * a.M + col + 1] = out[1];
      }
    }
  }
}

// ---------------------------------------------------------------- launchers
inline bool simt_tma_ok(const double* A, const double* B, int64_t N, int64_t P, int64_t M) {
  return tma_ok(A, P) && tma_ok(B, M) && N <= INT32_MAX && P <= INT32_MAX && M <= INT32_MAX;
}

template <auto KERN, int THREADS, size_t SMEM>
inline cudaError_t launch_simt_tma_t_(const SimtTmaArgs& args, unsigned grid, cudaStream_t st) {
  cudaError_t e = smem_attr_once<KERN>(SMEM);
  if (e != cudaSuccess) return e;
  KERN<<<grid, THREADS, SMEM, st>>>(args);
  note_launch();
  return cudaGetLastError();
}

template <class CF>
inline bool simt_tma_args(SimtTmaArgs& args, const double* A, const double* B, double* C, int64_t N, int64_t P,
                          int64_t M, int64_t lda = 0, int64_t ldb = 0) {
  args.A = A;
  args.B = B;
  args.C = C;
  args.N = N;
  args.P = P;
  args.M = M;
  return tma_encode_2d(&args.mapA, A, N, P, lda ? lda : P, CF::BM, 16, true) &&
         tma_encode_2d(&args.mapB, B, P, M, ldb ? ldb : M, CF::BK, 16, true);
}

template <class CF, bool FUSED = false>
inline cudaError_t launch_kahan_tma(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                                    cudaStream_t st) {
  using LY = SimtTmaLayout<CF>;
  SimtTmaArgs args{};
  if (!simt_tma_args<CF>(args, A, B, C, N, P, M)) return cudaErrorInvalidValue;
  const unsigned grid = unsigned(cdiv(M, CF::BN) * cdiv(N, CF::BM));
  const bool cv = (reinterpret_cast<uintptr_t>(C) & 15) == 0 && M % 2 == 0;
  return cv ? launch_simt_tma_t_<kahan_tma_kernel<CF, 2, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st)
            : launch_simt_tma_t_<kahan_tma_kernel<CF, 1, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st);
}

template <class CF, bool FUSED>
inline cudaError_t launch_winograd_pairs_tma(const double* A, const double* B, double* C, const double* y,
                                             const double* z, int64_t N, int64_t P, int64_t M, cudaStream_t st) {
  using LY = SimtTmaLayout<CF>;
  SimtTmaArgs args{};
  if (!simt_tma_args<CF>(args, A, B, C, N, P, M)) return cudaErrorInvalidValue;
  args.y = y;
  args.z = z;
  const unsigned grid = unsigned(cdiv(M, CF::BN) * cdiv(N, CF::BM));
  const bool cv = (reinterpret_cast<uintptr_t>(C) & 15) == 0 && M % 2 == 0;
  return cv ? launch_simt_tma_t_<winograd_tma_kernel<CF, 2, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st)
            : launch_simt_tma_t_<winograd_tma_kernel<CF, 1, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st);
}

// WinogradScaled, odd P: the pair sums of the even-pitch copies As (pitch lda) and Bs (pitch ldb)
// over their first P - 1 columns / rows, then (acc - y) - z + As[i][P-1] Bs[P-1][k] -- per entry the
// cp.async kernel's operations in its order, so bitwise the same
template <class CF, bool FUSED>
inline cudaError_t launch_winograd_pairs_tma_odd(const double* As, int64_t lda, const double* Bs, int64_t ldb,
                                                 double* C, const double* y, const double* z, int64_t N, int64_t P,
                                                 int64_t M, cudaStream_t st) {
  using LY = SimtTmaLayout<CF>;
  SimtTmaArgs args{};
  if (!simt_tma_args<CF>(args, As, Bs, C, N, P - 1, M, lda, ldb)) return cudaErrorInvalidValue;
  args.y = y;
  args.z = z;
  args.odd = 1;
  args.lda = lda;
  args.ldb = ldb;
  const unsigned grid = unsigned(cdiv(M, CF::BN) * cdiv(N, CF::BM));
  const bool cv = (reinterpret_cast<uintptr_t>(C) & 15) == 0 && M % 2 == 0;
  return cv ? launch_simt_tma_t_<winograd_tma_kernel<CF, 2, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st)
            : launch_simt_tma_t_<winograd_tma_kernel<CF, 1, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st);
}

// k-panel steps (NEXT-4): A (lda) / B (ldb) are panel views of wider operands, C and E dense N x M
inline bool simt_tma_ex_ok(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t N, int64_t P,
                           int64_t M) {
  return tma_ok(A, lda) && tma_ok(B, ldb) && lda >= P && ldb >= M && M % 2 == 0 && N <= INT32_MAX &&
         P <= INT32_MAX && M <= INT32_MAX;
}

template <class CF, bool FUSED>
inline cudaError_t launch_kahan_tma_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                       double* E, int64_t N, int64_t P, int64_t M, int flags, cudaStream_t st) {
  using LY = SimtTmaLayout<CF>;
  SimtTmaArgs args{};
  if (!simt_tma_args<CF>(args, A, B, C, N, P, M, lda, ldb)) return cudaErrorInvalidValue;
  args.E = E;
  args.flags = flags;
  const unsigned grid = unsigned(cdiv(M, CF::BN) * cdiv(N, CF::BM));
  const bool cv = (reinterpret_cast<uintptr_t>(C) & 15) == 0;
  return cv ? launch_simt_tma_t_<kahan_tma_kernel<CF, 2, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st)
            : launch_simt_tma_t_<kahan_tma_kernel<CF, 1, FUSED>, CF::THREADS, LY::SMEM>(args, grid, st);
}

template <class CF, bool FUSED>
inline cudaError_t launch_winograd_tma_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                          const double* y, const double* z, int64_t N, int64_t P, int64_t M,
                                          int flags, cudaStream_t st) {
  using LY = SimtTmaLayout<CF>;
  SimtTmaArgs args{};
  if (!simt_tma_args<CF>(args, A, B, C, N, P, M, lda, ldb)) return cudaErrorInvalidValue;
  args.y = y;
  args.z = z;
  args.flags = flags;
  const unsigned grid = unsigned(cdiv(M, CF::BN) * cdiv(N, CF::BM));
  const bool cv = (reinterpret_cast<uintptr_t>(C) & 15) == 0;
  return cv ? launch_simt_tma_t_<winograd_tma_kernel<CF, 2, FUSED, true>, CF::THREADS, LY::SMEM>(args, grid, st)
            : launch_simt_tma_t_<winograd_tma_kernel<CF, 1, FUSED, true>, CF::THREADS, LY::SMEM>(args, grid, st);
}

}  // namespace mmk
