// lines.cuh -- order-faithful per-line reductions streamed from HBM (product path).
//
// Three steps of the hot path are "one sequential sum per line of a matrix":
//   * NormInf:          s_i = sum_j |X_ij|, left to right; ||X|| = max_i s_i
//   * Winograd y:         y_i = sum_{j<gamma} A[i][2j] A[i][2j+1]           (rows of A)
//   * Winograd z:         z_k = sum_{j<gamma} B[2j][k] B[2j+1][k]           (columns of B)
// and WinogradScaled needs the exact copies 2^lambda A and 2^-lambda B
// (MultiplyWithScalar) whose y/z are the sums above taken on the copies.
//
// The sums must run in index order (reading R1/R17: the oracle's order; on ill-scaled inputs
// a different order changes y by ~50, SURVEY PR-7), so one lane owns one line and there is no
// parallelism inside a line.  The kernel is therefore built to keep HBM busy with few warps:
//   * one warp = 32 lines, one warp per CTA, a shared-memory ring of LN_STAGES (6) to
//     LN_MAX_STAGES (24) stages -- deeper when the grid leaves SMs to spare (a 1024-row shard of
//     A is only 32 warps: each then keeps 24 x 8 KB in flight instead of 6 x 8 KB) -- of
//     32 x LN_TK (32, or LN_TK_LONG = 128 when the launch has few lines) tiles;
//   * operands with a 16-byte aligned base and even pitch arrive by TMA (2-D tensor maps,
//     one elected lane issues the tile's box copies, completion counted in bytes on an
//     mbarrier); 8-byte aligned operands (odd pitch, e.g. P = 1001) fall back to 8-byte
//     cp.async with cp.async.mbarrier.arrive.noinc on the same barrier;
//   * row-line tiles use the 128-byte TMA swizzle so the lanes' 16-byte reads of their own
//     rows are bank-conflict free;
//   * optional fused scaled copy: the scaled tile is written back coalesced from shared
//     memory, and y/z are accumulated on the scaled values (dmul(s, x) -- the same single
//     rounding as the oracle's copy), so WinogradScaled needs one pass over A and B after
//     the norms instead of copy + y/z passes.
// Up to two jobs (e.g. rows of A and columns of B) share one launch.
//
// K4 norm_inf: one lane per row, the row summed left to right (bitwise the oracle's row sums); the
// max over rows is order-free: each warp reduces its 32 rows and issues one atomicMax on the IEEE
// bit pattern (non-negative doubles order like their uint64 images; a NaN row sum is forced to the
// canonical quiet NaN, whose pattern exceeds +inf's, so it propagates).  K5, the lambda rule
// (lambda_rule below), is evaluated on the device by every block of the scaled pass from the two
// norms K4 left in device memory -- no host round trip and no separate launch.
#pragma once
#include <cstdlib>

#include "tma.cuh"

namespace mmk {

constexpr int LN_LINES = 32, LN_TK = 32, LN_STAGES = 6, LN_MAX_STAGES = 24;
constexpr int LN_TILE = LN_LINES * LN_TK;  // 8 KB per stage
constexpr unsigned LN_TILE_BYTES = LN_TILE * sizeof(double);
inline constexpr size_t ln_smem(int stages, int tk = LN_TK) {
  return 1024 + size_t(stages) * LN_LINES * tk * sizeof(double) + stages * sizeof(uint64_t);
}
// Long tiles (TK = 128) for launches with few lines: a line's chain costs 8 cycles per element
// (FP64 latency, tools/probes/lat_probe.cu) plus a fixed cost per tile (barrier wait, refill,
// fences) that a warp alone on its SM cannot hide; 4x longer tiles amortise it 4x.
constexpr int LN_TK_LONG = 128, LN_TK_MID = 64;
static_assert(LN_TK == 32 && LN_LINES == 32, "one lane per tile column / line");

// LN_PAIRS_FMA: the NEXT-3 fused variant (reading R22), y = fma(x0, x1, y)
enum { LN_ABS = 0, LN_PAIRS = 1, LN_PAIRS_FMA = 2 };

template <int OP>
__device__ __forceinline__ double ln_pair(double acc, double x0, double x1) {
  return OP == LN_PAIRS_FMA ? __fma_rn(x0, x1, acc) : dadd(acc, dmul(x0, x1));
}

struct LineJob {
  const double* X;               // row-major matrix with leading dimension ld
  int64_t ld;
  int64_t nlines;                // rows (by_rows) or columns
  int64_t len;                   // elements streamed per line (columns, or rows)
  int64_t pair_end;              // LN_PAIRS: only elements < pair_end enter the sum (2 floor(P/2))
  double* out;                   // LN_PAIRS: per-line sums
  const double* init;            // LN_PAIRS, optional: per-line start values (a sum continued over a
                                 // later row panel of B -- the multi-GPU scaled Winograd, mm_dist_step)
  unsigned long long* out_max;   // LN_ABS: max over lines, as the bit pattern of a non-negative double
  double* copy;                  // optional scaled copy (same shape as X, row pitch copy_ld)
  int64_t copy_ld;
  int by_rows;
  int op;
  int scale_sel;                 // -1: unscaled; 0: x 2^lambda; 1: x 2^-lambda (lambda from norms)
  int bulk;                      // 1: tiles arrive by TMA (map[job]); 0: 8-byte cp.async fallback
  int cbulk;                     // 1: the scaled copy leaves by TMA store (cmap[job]) from the tile,
                                 //    scaled in place; 0: per-lane global stores
  int blocks;                    // 32-line blocks of this job
};

struct LineLaunch {
  CUtensorMap map[2];               // TMA maps of the jobs' operands (when bulk)
  CUtensorMap cmap[2];              // TMA maps of the jobs' copies (when cbulk)
  LineJob job[2];
  int njobs;
  const unsigned long long* norms;  // {||A||, ||B||} bit patterns (for scale_sel >= 0)
  int stages;                       // ring depth (LN_STAGES .. LN_MAX_STAGES), set by launch_lines
  int* lam_out;                     // optional: lambda, written by block 0
  double* scale_out;                // optional: {2^lambda, 2^-lambda}, written by block 0
};

// The rule of P:206-208 (reading R7): the integer lambda with 1/2 <= 2^(2 lambda) nA/nB <= 2,
// exact via frexp; when both candidates qualify take the larger |lambda|; a zero norm gives 0.
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

// ---- tile layouts (doubles).  Row-line tile: lines = rows r, elements = columns c, stored as two
// TMA boxes of [32 rows][16 columns] with the 128-byte swizzle (16-byte chunk q of row r at chunk
// q ^ (r % 8)), so that lane r reading its own row 16 bytes at a time is conflict free.
// Column-line tile: [32 rows k][32 columns l] plain, lane l reads t[k][l].
__device__ __forceinline__ int ln_rowoff(int r, int c) {
  return (c >> 4) * (LN_LINES * 16) + r * 16 + ((((c & 15) >> 1) ^ (r & 7)) << 1) + (c & 1);
}

// issue the copies of tile kt of block-lines [l0, l0+32) into stage buffer t (barrier bar)
template <int TK>
__device__ __forceinline__ void ln_issue(const LineLaunch& L, int ji, double* t, uint64_t* bar, int64_t l0,
                                         int64_t kt, int lane) {
  const LineJob& jb = L.job[ji];
  const int64_t k0 = kt * TK;
  if (jb.bulk) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bar, unsigned(LN_LINES * TK * sizeof(double)));
      if (jb.by_rows) {
#pragma unroll
        for (int bx = 0; bx < TK / 16; ++bx)  // [32 rows][16 columns] boxes
          tma_load_2d(t + bx * (LN_LINES * 16), &L.map[ji], int(k0 + 16 * bx), int(l0), bar);
      } else {
        tma_load_2d(t, &L.map[ji], int(l0), int(k0), bar);
      }
    }
  } else {
    const int64_t kv = jb.len - k0 < TK ? jb.len - k0 : TK;              // valid elements along the line
    const int64_t lv = jb.nlines - l0 < LN_LINES ? jb.nlines - l0 : LN_LINES;  // valid lines
    if (jb.by_rows) {
#pragma unroll 8
      for (int r = 0; r < LN_LINES; ++r) {
#pragma unroll
        for (int c = lane; c < TK; c += 32) {
          const bool v = r < lv && c < kv;
          cp_async8(t + ln_rowoff(r, c), v ? jb.X + (l0 + r) * jb.ld + k0 + c : jb.X, v);
        }
      }
    } else {
#pragma unroll 8
      for (int k = 0; k < TK; ++k) {
        const bool v = k < kv && lane < lv;
        cp_async8(t + k * LN_LINES + lane, v ? jb.X + (k0 + k) * jb.ld + l0 + lane : jb.X, v);
      }
    }
    cp_async_mbar_arrive_noinc(bar);
  }
}

// SCALED: the jobs carry scale_sel >= 0 (WinogradScaled's copies); a compile-time flag so the
// unscaled y/z pass executes exactly the method's DMUL/DADD (SASS fingerprint, tools/fingerprint.py)
template <int OP, bool SCALED, int TK>
__global__ void __launch_bounds__(LN_LINES) line_kernel(const __grid_constant__ LineLaunch L) {
  extern __shared__ __align__(1024) unsigned char ln_raw[];
  // 1024-byte aligned stage buffers (the 128-byte swizzle pattern repeats every 1024 bytes)
  double* ln_smem = reinterpret_cast<double*>(ln_raw + ((1024 - (smem_u32(ln_raw) & 1023)) & 1023));
  const int S = L.stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ln_smem + S * (LN_LINES * TK));
  const int lane = threadIdx.x;
  int b = blockIdx.x, ji = 0;
  if (L.njobs > 1 && b >= L.job[0].blocks) {
    b -= L.job[0].blocks;
    ji = 1;
  }
  const LineJob& jb = L.job[ji];
  const int64_t l0 = int64_t(b) * LN_LINES;
  const int KT = int(cdiv(jb.len, TK));

  double s = 1.0;
  if (SCALED && jb.scale_sel >= 0) {
    const double nA = __longlong_as_double(static_cast<long long>(L.norms[0]));
    const double nB = __longlong_as_double(static_cast<long long>(L.norms[1]));
    const int lam = lambda_rule(nA, nB);
    s = ldexp(1.0, jb.scale_sel == 0 ? lam : -lam);
    if (blockIdx.x == 0 && lane == 0) {
      if (L.lam_out) L.lam_out[0] = lam;
      if (L.scale_out) {
        L.scale_out[0] = ldexp(1.0, lam);
        L.scale_out[1] = ldexp(1.0, -lam);
      }
    }
  }

  if (lane == 0) {
    if (jb.bulk) tma_prefetch_desc(&L.map[ji]);
    if (jb.cbulk) tma_prefetch_desc(&L.cmap[ji]);
    for (int st = 0; st < S; ++st) mbar_init(bars + st, jb.bulk ? 1 : LN_LINES);
    fence_mbar_init();
  }
  __syncwarp();
#pragma unroll 1
  for (int st = 0; st < S; ++st)
    if (st < KT) ln_issue<TK>(L, ji, ln_smem + st * (LN_LINES * TK), bars + st, l0, st, lane);
  // ring positions kept incrementally (S is a launch parameter: no division per tile)
  int st = 0, rs = 0;  // stage of tile kt, stage of the tile refilled at kt (kt - lag)
  unsigned ph = 0;     // mbarrier phase parity of tile kt

  const bool scaled = SCALED && jb.scale_sel >= 0;
  // with the TMA-stored copy a stage is refilled one tile later (lag 2): the store of the tile just
  // finished may still be reading its stage, the one before it must have finished (wait_group.read 1)
  const bool cbulk = SCALED && jb.cbulk;
  const int lag = cbulk ? 2 : 1;
  double acc = (OP != LN_ABS && jb.init && l0 + lane < jb.nlines) ? jb.init[l0 + lane] : 0.0;
#pragma unroll 1
  for (int kt = 0; kt < KT; ++kt) {
    if (kt >= lag) {
      // refill tile kt-lag's stage with tile kt-lag+STAGES here, after the loop back edge: every op
      // consuming its shared-memory loads has issued, so those loads have completed (refilling
      // at the end of iteration kt-1 would let ptxas hoist the copy above in-flight loads)
      const int nk = kt - lag + S;
      if (jb.bulk) fence_proxy_async_smem();
      __syncwarp();
      if (nk < KT) {
        if (cbulk && lane == 0) bulk_wait_read<1>();
        ln_issue<TK>(L, ji, ln_smem + rs * (LN_LINES * TK), bars + rs, l0, nk, lane);
      }
      rs = rs + 1 == S ? 0 : rs + 1;
      __syncwarp();
    }
    mbar_wait(bars + st, ph);
    const double* t = ln_smem + st * (LN_LINES * TK);
    const int64_t k0 = int64_t(kt) * TK;
    const int kv = int(jb.len - k0 < TK ? jb.len - k0 : TK);
    if (jb.by_rows) {
      // lane = row l0 + lane; its 16-byte chunk q (columns 2q, 2q+1) sits in box q/8 at chunk (q%8)^(lane%8)
      const double* row = t + lane * 16;
      auto chunk = [&](int q) {
        return *reinterpret_cast<const double2*>(row + (q >> 3) * (LN_LINES * 16) + (((q & 7) ^ (lane & 7)) << 1));
      };
      if (OP == LN_ABS) {
        if (kv == TK) {
#pragma unroll
          for (int q = 0; q < TK / 2; ++q) {
            const double2 v = chunk(q);
            acc = dadd(acc, fabs(v.x));  // row sum, left to right
            acc = dadd(acc, fabs(v.y));
          }
        } else {
          for (int j = 0; j < kv; ++j) acc = dadd(acc, fabs(t[ln_rowoff(lane, j)]));
        }
      } else {
        // pairs (2q, 2q+1) of this tile that lie below pair_end
        const int64_t pe = jb.pair_end - k0;
        const int np = int((pe < kv ? pe : kv) / 2);
        if (cbulk) {
          // scale the lane's row of the tile in place (the copy leaves from here by TMA store),
          // then the pairs below pair_end on the scaled values: the same dmul(s, x) roundings
          double* rw = ln_smem + st * (LN_LINES * TK) + lane * 16;
#pragma unroll
          for (int q = 0; q < TK / 2; ++q) {
            double2* p2 = reinterpret_cast<double2*>(rw + (q >> 3) * (LN_LINES * 16) + (((q & 7) ^ (lane & 7)) << 1));
            double2 v = *p2;
            v = make_double2(dmul(s, v.x), dmul(s, v.y));
            *p2 = v;
            if (q < np) acc = ln_pair<OP>(acc, v.x, v.y);
          }
        } else if (np == TK / 2) {
#pragma unroll
          for (int q = 0; q < TK / 2; ++q) {
            double2 v = chunk(q);
            if (scaled) v = make_double2(dmul(s, v.x), dmul(s, v.y));
            acc = ln_pair<OP>(acc, v.x, v.y);  // y_i += A[i][2j] A[i][2j+1]
          }
        } else {
          for (int q = 0; q < np; ++q) {
            double2 v = chunk(q);
            if (scaled) v = make_double2(dmul(s, v.x), dmul(s, v.y));
            acc = ln_pair<OP>(acc, v.x, v.y);
          }
        }
      }
      if (cbulk) {  // the scaled tile leaves by TMA store (two 16-column boxes; the map clips edges)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int bx = 0; bx < TK / 16; ++bx)
            tma_store_2d(&L.cmap[ji], int(k0 + 16 * bx), int(l0), t + bx * (LN_LINES * 16));
          bulk_commit();
        }
      } else if (jb.copy) {  // coalesced write of the scaled tile: lane = column
        const int64_t lv = jb.nlines - l0 < LN_LINES ? jb.nlines - l0 : LN_LINES;
        if (lane < kv)
          for (int r = 0; r < lv; ++r) jb.copy[(l0 + r) * jb.copy_ld + k0 + lane] = dmul(s, t[ln_rowoff(r, lane)]);
      }
    } else {
      // column lines: lane = column l0 + lane, tile row k = element k0 + k of the line
      if (OP == LN_ABS) {
        for (int k = 0; k < kv; ++k) acc = dadd(acc, fabs(t[k * LN_LINES + lane]));
      } else {
        const int64_t pe = jb.pair_end - k0;
        const int np = int((pe < kv ? pe : kv) / 2);
        if (cbulk) {  // scale the lane's column of the tile in place, pairs on the scaled values
          double* cw = ln_smem + st * (LN_LINES * TK) + lane;
#pragma unroll
          for (int j = 0; j < TK / 2; ++j) {
            const double x0 = dmul(s, cw[(2 * j) * LN_LINES]), x1 = dmul(s, cw[(2 * j + 1) * LN_LINES]);
            cw[(2 * j) * LN_LINES] = x0;
            cw[(2 * j + 1) * LN_LINES] = x1;
            if (j < np) acc = ln_pair<OP>(acc, x0, x1);
          }
        } else if (np == TK / 2) {
#pragma unroll
          for (int j = 0; j < TK / 2; ++j) {
            double x0 = t[(2 * j) * LN_LINES + lane], x1 = t[(2 * j + 1) * LN_LINES + lane];
            if (scaled) {
              x0 = dmul(s, x0);
              x1 = dmul(s, x1);
            }
            acc = ln_pair<OP>(acc, x0, x1);  // z_k += B[2j][k] B[2j+1][k]
          }
        } else {
          for (int j = 0; j < np; ++j) {
            double x0 = t[(2 * j) * LN_LINES + lane], x1 = t[(2 * j + 1) * LN_LINES + lane];
            if (scaled) {
              x0 = dmul(s, x0);
              x1 = dmul(s, x1);
            }
            acc = ln_pair<OP>(acc, x0, x1);
          }
        }
      }
      if (cbulk) {  // the scaled tile leaves by TMA store (the map clips the edges)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&L.cmap[ji], int(l0), int(k0), t);
          bulk_commit();
        }
      } else if (jb.copy) {  // lane = column; rows of the panel are 256-byte coalesced stores
        const int64_t lv = jb.nlines - l0 < LN_LINES ? jb.nlines - l0 : LN_LINES;
        if (lane < lv)
          for (int k = 0; k < kv; ++k) jb.copy[(k0 + k) * jb.copy_ld + l0 + lane] = dmul(s, t[k * LN_LINES + lane]);
      }
    }
    if (++st == S) {
      st = 0;
      ph ^= 1u;
    }
  }

  if (cbulk && lane == 0) bulk_wait_all();  // the stores have left shared memory (and landed)
  __syncwarp();
  const bool valid = l0 + lane < jb.nlines;
  if (OP == LN_ABS) {
    double m = valid ? acc : 0.0;  // max is order-free
    const bool any_nan = __any_sync(0xffffffffu, valid && isnan(acc));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const unsigned long long bits =
        any_nan ? 0x7ff8000000000000ull : static_cast<unsigned long long>(__double_as_longlong(m));
    if (lane == 0) atomicMax(jb.out_max, bits);
  } else {
    if (valid) jb.out[l0 + lane] = acc;
  }
}

// fill the derived fields of a job (blocks; TMA map when the operand allows one)
inline void ln_finish_job(LineJob& j, CUtensorMap* map, CUtensorMap* cmap, int tk) {
  j.blocks = int(cdiv(j.nlines, LN_LINES));
  j.bulk = 0;
  j.cbulk = 0;
  if (tma_ok(j.X, j.ld)) {
    const int64_t rows = j.by_rows ? j.nlines : j.len, cols = j.by_rows ? j.len : j.nlines;
    if (j.by_rows)
      j.bulk = tma_encode_2d(map, j.X, rows, cols, j.ld, LN_LINES, 16, true);
    else
      j.bulk = tma_encode_2d(map, j.X, rows, cols, j.ld, tk, LN_LINES, false);
    // the copy has X's shape: the same box geometry stores the (in place scaled) tile
    if (j.bulk && j.copy && j.scale_sel >= 0 && tma_ok(j.copy, j.copy_ld))
      j.cbulk = j.by_rows ? tma_encode_2d(cmap, j.copy, rows, cols, j.copy_ld, LN_LINES, 16, true)
                          : tma_encode_2d(cmap, j.copy, rows, cols, j.copy_ld, tk, LN_LINES, false);
  }
}

template <int OP, bool SCALED, int TK>
inline cudaError_t launch_lines_tk(LineLaunch& L, int blocks, int sms, cudaStream_t st) {
  constexpr auto k = line_kernel<OP, SCALED, TK>;
  constexpr int tile = LN_LINES * TK * int(sizeof(double)) + 8;
  constexpr int smax = (220 * 1024 - 1024) / tile < LN_MAX_STAGES ? (220 * 1024 - 1024) / tile : LN_MAX_STAGES;
  cudaError_t e = smem_attr_once<k>(ln_smem(smax, TK));
  if (e != cudaSuccess) return e;
  // ring depth: the shared memory of an SM (~220 KB usable) shared by the blocks it will hold
  const int per_sm = int((blocks + sms - 1) / sms);
  int stages = int((220 * 1024 / (per_sm > 0 ? per_sm : 1) - 1024) / tile);
  if (stages > smax) stages = smax;
  static const int cap = [] {  // MM_LN_MAX_STAGES: tuning override of the depth cap
    const char* v = std::getenv("MM_LN_MAX_STAGES");
    const int c = v ? std::atoi(v) : LN_MAX_STAGES;
    return c < 2 ? 2 : (c > LN_MAX_STAGES ? LN_MAX_STAGES : c);
  }();
  const int lo = TK == LN_TK ? LN_STAGES : 3;
  L.stages = stages < lo ? lo : (stages > cap ? cap : stages);
  k<<<unsigned(blocks), LN_LINES, ln_smem(L.stages, TK), st>>>(L);
  note_launch();
  return cudaGetLastError();
}

template <int OP, bool SCALED = false>
inline cudaError_t launch_lines(LineLaunch& L, cudaStream_t st) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                   cudaSuccess) {
      cudaGetLastError();
      sms = 148;
    }
  }
  // longer tiles the fewer blocks an SM holds, when every operand streams by TMA: 128-element
  // tiles up to two blocks per SM (3-6 stages of 32 KB), 64-element tiles up to four (3 of 16 KB)
  int blocks = 0;
  bool all_tma = true;
  for (int i = 0; i < L.njobs; ++i) {
    blocks += int(cdiv(L.job[i].nlines, LN_LINES));
    all_tma = all_tma && tma_ok(L.job[i].X, L.job[i].ld);
  }
  const int tk = !all_tma ? LN_TK : blocks <= 2 * sms ? LN_TK_LONG : blocks <= 4 * sms ? LN_TK_MID : LN_TK;
  for (int i = 0; i < L.njobs; ++i) ln_finish_job(L.job[i], &L.map[i], &L.cmap[i], tk);
  if (tk == LN_TK_LONG) return launch_lines_tk<OP, SCALED, LN_TK_LONG>(L, blocks, sms, st);
  if (tk == LN_TK_MID) return launch_lines_tk<OP, SCALED, LN_TK_MID>(L, blocks, sms, st);
  return launch_lines_tk<OP, SCALED, LN_TK>(L, blocks, sms, st);
}

inline LineJob ln_job(const double* X, int64_t ld, int64_t nlines, int64_t len, bool by_rows, int op) {
  LineJob j{};
  j.X = X;
  j.ld = ld;
  j.nlines = nlines;
  j.len = len;
  j.pair_end = 2 * (len / 2);
  j.copy_ld = ld;
  j.by_rows = by_rows ? 1 : 0;
  j.op = op;
  j.scale_sel = -1;
  return j;
}

// ||X||_inf of one or two matrices in one launch; out[i] zeroed here, then max-reduced.
inline cudaError_t launch_norms(const double* X0, int64_t r0, int64_t c0, const double* X1, int64_t r1, int64_t c1,
                                unsigned long long* out, cudaStream_t st) {
  const int n = X1 ? 2 : 1;
  cudaError_t e = cudaMemsetAsync(out, 0, n * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  LineLaunch L{};
  L.njobs = n;
  L.job[0] = ln_job(X0, c0, r0, c0, true, LN_ABS);
  L.job[0].out_max = out;
  if (X1) {
    L.job[1] = ln_job(X1, c1, r1, c1, true, LN_ABS);
    L.job[1].out_max = out + 1;
  }
  return launch_lines<LN_ABS>(L, st);
}

// out: device uint64 slot, zeroed here then max-reduced
inline cudaError_t launch_norm_inf(const double* X, int64_t rows, int64_t cols, unsigned long long* out,
                                   cudaStream_t st) {
  return launch_norms(X, rows, cols, nullptr, 0, 0, out, st);
}

// Winograd y (rows of A) and z (columns of B); optionally on the exact scaled copies
// As = 2^lambda A, Bs = 2^-lambda B, which are written in the same pass (lambda from norms).
inline cudaError_t launch_yz(const double* A, const double* B, double* y, double* z, int64_t N, int64_t P, int64_t M,
                             double* As, double* Bs, const unsigned long long* norms, int* lam_out, double* scale_out,
                             cudaStream_t st, bool fused = false, int64_t as_ld = 0) {
  LineLaunch L{};
  L.njobs = 2;
  L.norms = norms;
  L.lam_out = lam_out;
  L.scale_out = scale_out;
  const bool scaled = As != nullptr;
  // y: rows of A (stream the whole row when the copy needs the odd column too)
  L.job[0] = ln_job(A, P, N, scaled ? P : 2 * (P / 2), true, LN_PAIRS);
  L.job[0].pair_end = 2 * (P / 2);
  L.job[0].out = y;
  // z: columns of B (rows 0 .. 2 gamma - 1, or all P rows for the copy)
  L.job[1] = ln_job(B, M, M, scaled ? P : 2 * (P / 2), false, LN_PAIRS);
  L.job[1].pair_end = 2 * (P / 2);
  L.job[1].out = z;
  if (scaled) {
    L.job[0].copy = As;
    if (as_ld) L.job[0].copy_ld = as_ld;  // an even pitch for odd P: the copy can feed the TMA kernel
    L.job[0].scale_sel = 0;
    L.job[1].copy = Bs;
    L.job[1].scale_sel = 1;
  }
  if (scaled) return fused ? launch_lines<LN_PAIRS_FMA, true>(L, st) : launch_lines<LN_PAIRS, true>(L, st);
  return fused ? launch_lines<LN_PAIRS_FMA, false>(L, st) : launch_lines<LN_PAIRS, false>(L, st);
}

// The two halves of launch_yz's scaled pass, for the multi-GPU WinogradScaled (mm_dist_step):
// MM_OP_SCALE_A: As = 2^lambda A and y' (rows of A); MM_OP_SCALE_B: rows [k0, k1) of Bs = 2^-lambda B
// and z' continued over those rows (k0 even; `chain` = continue z' from its current value, else start
// at 0).  Panels in increasing k0 perform every z'_k's operations in the one-pass order, so y', z'
// and the copies are bitwise those of launch_yz(..., As, Bs, ...).
inline cudaError_t launch_scale_rows(const double* A, double* As, double* y, int64_t N, int64_t P,
                                     const unsigned long long* norms, cudaStream_t st, bool fused) {
  // (the multi-GPU panel path: P even, so the copy keeps A's pitch)
  LineLaunch L{};
  L.njobs = 1;
  L.norms = norms;
  L.job[0] = ln_job(A, P, N, P, true, LN_PAIRS);
  L.job[0].pair_end = 2 * (P / 2);
  L.job[0].out = y;
  L.job[0].copy = As;
  L.job[0].scale_sel = 0;
  return fused ? launch_lines<LN_PAIRS_FMA, true>(L, st) : launch_lines<LN_PAIRS, true>(L, st);
}

inline cudaError_t launch_scale_cols(const double* B, double* Bs, double* z, int64_t P, int64_t M, int64_t k0,
                                     int64_t k1, bool chain, const unsigned long long* norms, cudaStream_t st,
                                     bool fused) {
  LineLaunch L{};
  L.njobs = 1;
  L.norms = norms;
  L.job[0] = ln_job(B + k0 * M, M, M, k1 - k0, false, LN_PAIRS);
  const int64_t pe = 2 * (P / 2) - k0;
  L.job[0].pair_end = pe < k1 - k0 ? pe : k1 - k0;
  L.job[0].out = z;
  L.job[0].init = chain ? z : nullptr;
  L.job[0].copy = Bs + k0 * M;
  L.job[0].scale_sel = 1;
  return fused ? launch_lines<LN_PAIRS_FMA, true>(L, st) : launch_lines<LN_PAIRS, true>(L, st);
}

}  // namespace mmk
