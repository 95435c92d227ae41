// strassen.cuh -- K6/K7/K8: StrassenNaiv and StrassenWinograd as a
// breadth-first recursion over a workspace arena.
//
//  level l holds 7^l nodes; node q's operands are dense [n_l x p_l] / [p_l x m_l] blocks at
//  q * n_l * p_l of the level buffer; child t (t = 0..6 for H_{t+1}) of node q is node 7q + t.
//
//  * form kernel (one launch per level and side, or per two / three levels, below): reads the
//    four quadrants X11, X12, X21, X22 of every node once and writes the seven child operands,
//    fusing the paper's block
//    additions (P:271-277 / P:300-306) in registers with exactly the oracle's per-element
//    operations and order (e.g. A2 = A22 - (A11 - A21)).  At level 0 it reads the caller's A
//    or B with the zero embedding of P:286 applied on the fly (no padded copy).
//  * the 7^d leaf products H = S T run as ONE batched DMMA GEMM launch (gemm_tma.cuh, or
//    gemm_dmma.cuh for operands a tensor map cannot describe).
//  * combine kernel (one launch per level): reads H_1..H_7 of every node once and writes
//    the four C quadrants (P:279-282 / P:307-311, left to right as displayed); at level 0
//    it writes straight into the caller's C, dropping the padding (the "extract" of P:286).
//  * two levels per pass (strassen_form2_kernel / strassen_combine2_kernel) for the deepest
//    pairs of levels: the intermediate level -- 7/4 the data of the one above it -- is never
//    written nor re-read, and a three-level formation pass (strassen_form3_kernel) at odd depth
//    (c4, d = 3: 24.6 -> 22.4 ms per product).
// All add/sub kernels are HBM-bound grid-stride loops with 16-byte vectors where aligned.
#pragma once
#include <cstdlib>

#include "common.cuh"
#include "gemm_comb.cuh"
#include "gemm_tma.cuh"

namespace mmk {

constexpr int SV_NAIV = 0, SV_WINOGRAD = 1;

struct FormArgs {
  const double* src;      // parent level: cnt nodes
  int64_t src_pitch;      // row pitch of a parent node (elements)
  int64_t src_stride;     // distance between parent nodes (elements)
  int64_t rows_valid;     // rows of the parent that hold data (the rest are the zero embedding)
  int64_t cols_valid;
  double* dst;            // child level: 7 cnt dense nodes of h_rows x h_cols
  int64_t h_rows, h_cols; // child (= quadrant) dims
  int64_t cnt;
  int64_t u0, u1;         // row units [u0, u1) of the cnt * h_rows this pass covers (all by default;
                          // a sub-range forms the operands from the rows of B that have already
                          // arrived -- the multi-GPU broadcast overlap, mm_dist_step MM_OP_FORM_B)
};

// ---- vector I/O: V = 4 -> 256-bit LDG/STG (sm_100a), V = 2 -> 128-bit, V = 1 -> scalar
template <int V>
__device__ __forceinline__ void ldv(const double* p, double* v) {
  if (V == 4) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p));
  } else if (V == 2) {
    const double2 w = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = w.x;
    v[1] = w.y;
  } else {
    v[0] = __ldg(p);
  }
}
template <int V>
__device__ __forceinline__ void stv(double* p, const double* v) {
  if (V == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
  } else if (V == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  } else {
    p[0] = v[0];
  }
}

// v[0..V) = parent[r][c .. c+V) with the zero embedding of P:286 outside rows_valid x cols_valid
template <int V>
__device__ __forceinline__ void ld_quad(const FormArgs& a, const double* base, int64_t r, int64_t c, double* v) {
  const double* p = base + r * a.src_pitch + c;
  if (r < a.rows_valid && c + V <= a.cols_valid) {
    ldv<V>(p, v);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) v[e] = (r < a.rows_valid && c + e < a.cols_valid) ? p[e] : 0.0;
  }
}

// Work mapping of the add/sub kernels: a "row unit" is one row of one node's quadrant; 2^TPRS
// threads sweep a row unit with V-wide vectors (consecutive threads -> consecutive vectors,
// so every warp access is a contiguous, fully used run of sectors), 256 >> TPRS row units per
// block, grid-stride over the pass's units [u0, u1) (all cnt * h_rows of them unless a multi-GPU
// panel restricts the first B-side pass).  Index arithmetic is once per row unit.

// the seven child operands of one node at one element position, from its four quadrants'
// values: P:271-277 (StrassenNaiv) / P:300-306 (StrassenWinograd), the oracle's operations in
// the oracle's order
template <int VARIANT, int SIDE>
__device__ __forceinline__ void form7(double x11, double x12, double x21, double x22, double (&o)[7]) {
  if (VARIANT == SV_NAIV) {
    if (SIDE == 0) {              // P:271-277, left factors
      o[0] = dadd(x11, x22);  // H1: A11 + A22
      o[1] = dadd(x21, x22);  // H2: A21 + A22
      o[2] = x11;             // H3: A11
      o[3] = x22;             // H4: A22
      o[4] = dadd(x11, x12);  // H5: A11 + A12
      o[5] = dsub(x21, x11);  // H6: A21 - A11
      o[6] = dsub(x12, x22);  // H7: A12 - A22
    } else {                      // right factors
      o[0] = dadd(x11, x22);  // H1: B11 + B22
      o[1] = x11;             // H2: B11
      o[2] = dsub(x12, x22);  // H3: B12 - B22
      o[3] = dsub(x21, x11);  // H4: B21 - B11
      o[4] = x22;             // H5: B22
      o[5] = dadd(x11, x12);  // H6: B11 + B12
      o[6] = dadd(x21, x22);  // H7: B21 + B22
    }
  } else {
    if (SIDE == 0) {
      const double a1 = dsub(x11, x21);  // A1 = A11 - A21
      const double a2 = dsub(x22, a1);   // A2 = A22 - A1
      o[0] = x11;                        // H1: A11
      o[1] = x12;                        // H2: A12
      o[2] = a2;                         // H3: A2
      o[3] = dadd(x21, x22);             // H4: A21 + A22
      o[4] = a1;                         // H5: A1
      o[5] = dsub(x12, a2);              // H6: A12 - A2
      o[6] = x22;                        // H7: A22
    } else {
      const double b1 = dsub(x22, x12);  // B1 = B22 - B12
      const double b2 = dadd(b1, x11);   // B2 = B1 + B11
      o[0] = x11;                        // H1: B11
      o[1] = x21;                        // H2: B21
      o[2] = b2;                         // H3: B2
      o[3] = dsub(x12, x11);             // H4: B12 - B11
      o[4] = b1;                         // H5: B1
      o[5] = x22;                        // H6: B22
      o[6] = dsub(x21, b2);              // H7: B21 - B2
    }
  }
}

// child c alone (c warp-uniform): the same operations as form7's c-th output
template <int VARIANT, int SIDE>
__device__ __forceinline__ double form1(int c, double x11, double x12, double x21, double x22) {
  double o[7];
  switch (c) {  // each case evaluates only what form7 does for output c
    case 0: { form7<VARIANT, SIDE>(x11, x12, x21, x22, o); return o[0]; }
    case 1: { form7<VARIANT, SIDE>(x11, x12, x21, x22, o); return o[1]; }
    case 2: { form7<VARIANT, SIDE>(x11, x12, x21, x22, o); return o[2]; }
    case 3: { form7<VARIANT, SIDE>(x11, x12, x21, x22, o); return o[3]; }
    case 4: { form7<VARIANT, SIDE>(x11, x12, x21, x22, o); return o[4]; }
    case 5: { form7<VARIANT, SIDE>(x11, x12, x21, x22, o); return o[5]; }
    default: { form7<VARIANT, SIDE>(x11, x12, x21, x22, o); return o[6]; }
  }
}

// SIDE 0 = left operands (from A), SIDE 1 = right operands (from B)
template <int VARIANT, int SIDE, int V>
__global__ void __launch_bounds__(256) strassen_form_kernel(FormArgs a, int tprs) {
  const int sub = threadIdx.x >> tprs, lt = threadIdx.x & ((1 << tprs) - 1);
  const int64_t rpb = 256 >> tprs, step = int64_t(V) << tprs;
  const int64_t child_elems = a.h_rows * a.h_cols;
  for (int64_t u = a.u0 + int64_t(blockIdx.x) * rpb + sub; u < a.u1; u += int64_t(gridDim.x) * rpb) {
    const int64_t q = u / a.h_rows, i = u - q * a.h_rows;
    const double* base = a.src + q * a.src_stride;
    double* d0 = a.dst + (7 * q) * child_elems + i * a.h_cols;
    for (int64_t j = int64_t(lt) * V; j < a.h_cols; j += step) {
      double x11[V], x12[V], x21[V], x22[V];
      ld_quad<V>(a, base, i, j, x11);
      ld_quad<V>(a, base, i, j + a.h_cols, x12);
      ld_quad<V>(a, base, i + a.h_rows, j, x21);
      ld_quad<V>(a, base, i + a.h_rows, j + a.h_cols, x22);
      double o[7][V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        double r7[7];
        form7<VARIANT, SIDE>(x11[e], x12[e], x21[e], x22[e], r7);
#pragma unroll
        for (int t = 0; t < 7; ++t) o[t][e] = r7[t];
      }
#pragma unroll
      for (int t = 0; t < 7; ++t) stv<V>(d0 + t * child_elems + j, o[t]);
    }
  }
}

// One child of each node (the alternative partition, mm_s7_step MM_OP_S7_FORM): child `child`'s
// operand alone, form1 -- form7's output `child` with exactly its operations -- into cnt dense
// nodes of h_rows x h_cols.
template <int VARIANT, int SIDE, int V>
__global__ void __launch_bounds__(256) strassen_form_child_kernel(FormArgs a, int child, int tprs) {
  const int sub = threadIdx.x >> tprs, lt = threadIdx.x & ((1 << tprs) - 1);
  const int64_t rpb = 256 >> tprs, step = int64_t(V) << tprs;
  const int64_t child_elems = a.h_rows * a.h_cols;
  for (int64_t u = a.u0 + int64_t(blockIdx.x) * rpb + sub; u < a.u1; u += int64_t(gridDim.x) * rpb) {
    const int64_t q = u / a.h_rows, i = u - q * a.h_rows;
    const double* base = a.src + q * a.src_stride;
    double* d0 = a.dst + q * child_elems + i * a.h_cols;
    for (int64_t j = int64_t(lt) * V; j < a.h_cols; j += step) {
      double x11[V], x12[V], x21[V], x22[V], o[V];
      ld_quad<V>(a, base, i, j, x11);
      ld_quad<V>(a, base, i, j + a.h_cols, x12);
      ld_quad<V>(a, base, i + a.h_rows, j, x21);
      ld_quad<V>(a, base, i + a.h_rows, j + a.h_cols, x22);
#pragma unroll
      for (int e = 0; e < V; ++e) o[e] = form1<VARIANT, SIDE>(child, x11[e], x12[e], x21[e], x22[e]);
      stv<V>(d0 + j, o);
    }
  }
}

// Two recursion levels in one pass (l -> l + 2): each thread reads the 16 sub-blocks' values of
// a node at one position, forms its 7 children's 4 quadrant values (form7 per quadrant) and
// from those the 49 grandchildren -- the same per-element operations and order as two
// single-level passes (bitwise the same operands), without writing and re-reading level l + 1
// (the deepest two levels carry most of the formation traffic: 7/4 more data per level).
// FormArgs: h_rows / h_cols are the GRANDCHILD dims (a quarter of the parent's), dst holds
// 49 cnt nodes.
template <int VARIANT, int SIDE, int V>
__global__ void __launch_bounds__(256) strassen_form2_kernel(FormArgs a, int tprs) {
  const int sub = threadIdx.x >> tprs, lt = threadIdx.x & ((1 << tprs) - 1);
  const int64_t rpb = 256 >> tprs, step = int64_t(V) << tprs;
  const int64_t gelems = a.h_rows * a.h_cols;
  for (int64_t u = a.u0 + int64_t(blockIdx.x) * rpb + sub; u < a.u1; u += int64_t(gridDim.x) * rpb) {
    const int64_t q = u / a.h_rows, i = u - q * a.h_rows;
    const double* base = a.src + q * a.src_stride;
    double* d0 = a.dst + (49 * q) * gelems + i * a.h_cols;
    for (int64_t j = int64_t(lt) * V; j < a.h_cols; j += step) {
      double x[4][4][V];  // x[row sub-block][col sub-block]
#pragma unroll
      for (int pr = 0; pr < 4; ++pr)
#pragma unroll
        for (int pc = 0; pc < 4; ++pc) ld_quad<V>(a, base, i + pr * a.h_rows, j + pc * a.h_cols, x[pr][pc]);
      // child c (a warp-uniform loop, not unrolled: keeps the register count low enough for
      // two blocks per SM), its quadrant (qa, qb) = child c of the parent quadrants' (qa, qb)
      // sub-blocks, then its 7 children
      double* p = d0 + j;
#pragma unroll 1
      for (int c = 0; c < 7; ++c) {
        double g[7][V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
          double cq[2][2];
#pragma unroll
          for (int qa = 0; qa < 2; ++qa)
#pragma unroll
            for (int qb = 0; qb < 2; ++qb)
              cq[qa][qb] = form1<VARIANT, SIDE>(c, x[qa][qb][e], x[qa][2 + qb][e], x[2 + qa][qb][e],
                                                x[2 + qa][2 + qb][e]);
          double r7[7];
          form7<VARIANT, SIDE>(cq[0][0], cq[0][1], cq[1][0], cq[1][1], r7);
#pragma unroll
          for (int t = 0; t < 7; ++t) g[t][e] = r7[t];
        }
#pragma unroll
        for (int t = 0; t < 7; ++t) {
          stv<V>(p, g[t]);
          p += gelems;
        }
      }
    }
  }
}

// Three recursion levels in one pass (l -> l + 3, scalar): a thread reads a node's 64 sub-block
// values (8 x 8 grid) at one position; for each child c its 16 sub-block values, for each
// grandchild g its 4 quadrant values, then the 7 great-grandchildren -- again exactly the
// single-level operations in their order.  h_rows / h_cols: the great-grandchild dims (an
// eighth of the parent's); dst holds 343 cnt nodes.  At d = 3 this is the whole formation.
// The 64 inputs are staged in a THREAD-PRIVATE slice of shared memory (slot k of thread t at
// k * F3_THREADS + t: conflict-free, no barrier -- no thread reads another's values) instead of
// registers: a child's sub-block value needs only 4 of them, so a thread keeps 16 child values
// live instead of 64 inputs (255 registers with spills and one 256-thread block per SM before;
// ~100 registers and three 128-thread blocks per SM now).
constexpr int F3_THREADS = 128;
constexpr size_t F3_SMEM = size_t(64) * F3_THREADS * sizeof(double);  // 64 KB

template <int VARIANT, int SIDE>
__global__ void __launch_bounds__(F3_THREADS) strassen_form3_kernel(FormArgs a, int tprs) {
  extern __shared__ double f3_x[];
  double* xs = f3_x + threadIdx.x;  // this thread's 64 slots, stride F3_THREADS
  const int sub = threadIdx.x >> tprs, lt = threadIdx.x & ((1 << tprs) - 1);
  const int64_t rpb = F3_THREADS >> tprs, step = int64_t(1) << tprs;
  const int64_t gelems = a.h_rows * a.h_cols;
  for (int64_t u = a.u0 + int64_t(blockIdx.x) * rpb + sub; u < a.u1; u += int64_t(gridDim.x) * rpb) {
    const int64_t q = u / a.h_rows, i = u - q * a.h_rows;
    const double* base = a.src + q * a.src_stride;
    double* d0 = a.dst + (343 * q) * gelems + i * a.h_cols;
    for (int64_t j = lt; j < a.h_cols; j += step) {
#pragma unroll 1
      for (int pr0 = 0; pr0 < 8; pr0 += 2) {  // 16 loads in flight per thread, then parked
        double v[16];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int pc = 0; pc < 8; ++pc)
            ld_quad<1>(a, base, i + (pr0 + r) * a.h_rows, j + pc * a.h_cols, &v[r * 8 + pc]);
#pragma unroll
        for (int k = 0; k < 16; ++k) xs[(pr0 * 8 + k) * F3_THREADS] = v[k];
      }
      // volatile: read from shared memory where used, not hoisted back into 64 registers
      const volatile double* xv = xs;
      auto x = [&](int pr, int pc) { return xv[(pr * 8 + pc) * F3_THREADS]; };
      double* p = d0 + j;
#pragma unroll 1
      for (int c = 0; c < 7; ++c) {
        double ch[4][4];  // child c's 4 x 4 sub-blocks: child c of the parent quadrants' sub-blocks
#pragma unroll
        for (int ra = 0; ra < 4; ++ra)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb)
            ch[ra][cb] = form1<VARIANT, SIDE>(c, x(ra, cb), x(ra, 4 + cb), x(4 + ra, cb), x(4 + ra, 4 + cb));
#pragma unroll 1
        for (int g = 0; g < 7; ++g) {
          double gq[2][2];
#pragma unroll
          for (int ra = 0; ra < 2; ++ra)
#pragma unroll
            for (int cb = 0; cb < 2; ++cb)
              gq[ra][cb] = form1<VARIANT, SIDE>(g, ch[ra][cb], ch[ra][2 + cb], ch[2 + ra][cb], ch[2 + ra][2 + cb]);
          double o[7];
          form7<VARIANT, SIDE>(gq[0][0], gq[0][1], gq[1][0], gq[1][1], o);
#pragma unroll
          for (int t = 0; t < 7; ++t) {
            *p = o[t];
            p += gelems;
          }
        }
      }
    }
  }
}

struct CombineArgs {
  const double* H;         // 7 cnt dense nodes of h_rows x h_cols
  double* dst;             // cnt parent nodes
  int64_t dst_pitch, dst_stride;
  int64_t rows_valid, cols_valid;  // parent region that is stored (extraction at level 0)
  int64_t h_rows, h_cols, cnt;
};

template <int V>
__device__ __forceinline__ void st_quad(const CombineArgs& a, double* base, int64_t r, int64_t c, const double* v) {
  double* p = base + r * a.dst_pitch + c;
  if (r < a.rows_valid && c + V <= a.cols_valid) {
    stv<V>(p, v);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e)
      if (r < a.rows_valid && c + e < a.cols_valid) p[e] = v[e];
  }
}

// the four quadrants C11, C12, C21, C22 of one node at one element position from its seven
// products: P:279-282 (StrassenNaiv) / P:308-311 (StrassenWinograd), left to right as displayed
template <int VARIANT>
__device__ __forceinline__ void comb4(double H1, double H2, double H3, double H4, double H5, double H6, double H7,
                                      double (&c)[4]) {
  if (VARIANT == SV_NAIV) {  // P:279-282, left to right
    c[0] = dadd(dsub(dadd(H1, H4), H5), H7);
    c[1] = dadd(H3, H5);
    c[2] = dadd(H2, H4);
    c[3] = dadd(dsub(dadd(H1, H3), H2), H6);
  } else {
    const double H8 = dadd(H1, H3);
    const double H9 = dadd(H8, H4);
    c[0] = dadd(H1, H2);
    c[1] = dadd(H9, H6);
    c[2] = dadd(dadd(H8, H5), H7);
    c[3] = dadd(H9, H5);
  }
}

template <int VARIANT, int V>
__global__ void __launch_bounds__(256) strassen_combine_kernel(CombineArgs a, int tprs) {
  const int sub = threadIdx.x >> tprs, lt = threadIdx.x & ((1 << tprs) - 1);
  const int64_t rpb = 256 >> tprs, step = int64_t(V) << tprs;
  const int64_t units = a.cnt * a.h_rows;
  const int64_t child_elems = a.h_rows * a.h_cols;
  for (int64_t u = int64_t(blockIdx.x) * rpb + sub; u < units; u += int64_t(gridDim.x) * rpb) {
    const int64_t q = u / a.h_rows, i = u - q * a.h_rows;
    const double* h0 = a.H + (7 * q) * child_elems + i * a.h_cols;
    double* base = a.dst + q * a.dst_stride;
    for (int64_t j = int64_t(lt) * V; j < a.h_cols; j += step) {
      double h[7][V];
#pragma unroll
      for (int t = 0; t < 7; ++t) ldv<V>(h0 + t * child_elems + j, h[t]);
      double c11[V], c12[V], c21[V], c22[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        double q4[4];
        comb4<VARIANT>(h[0][e], h[1][e], h[2][e], h[3][e], h[4][e], h[5][e], h[6][e], q4);
        c11[e] = q4[0];
        c12[e] = q4[1];
        c21[e] = q4[2];
        c22[e] = q4[3];
      }
      st_quad<V>(a, base, i, j, c11);
      st_quad<V>(a, base, i, j + a.h_cols, c12);
      st_quad<V>(a, base, i + a.h_rows, j, c21);
      st_quad<V>(a, base, i + a.h_rows, j + a.h_cols, c22);
    }
  }
}

// Two recursion levels in one pass (level l + 2 products -> level l node): per position, the 49
// grandchild products of a node give its 7 children's 4 quadrant values (comb4 per child), and
// those give the node's 16 sub-blocks (comb4 per child quadrant) -- the same operations and order
// as two single-level passes (bitwise), without writing and re-reading level l + 1.
// CombineArgs: H holds 49 cnt grandchild products of h_rows x h_cols (a quarter of the node).
template <int VARIANT, int V>
__global__ void __launch_bounds__(256) strassen_combine2_kernel(CombineArgs a, int tprs) {
  const int sub = threadIdx.x >> tprs, lt = threadIdx.x & ((1 << tprs) - 1);
  const int64_t rpb = 256 >> tprs, step = int64_t(V) << tprs;
  const int64_t units = a.cnt * a.h_rows;
  const int64_t gelems = a.h_rows * a.h_cols;
  for (int64_t u = int64_t(blockIdx.x) * rpb + sub; u < units; u += int64_t(gridDim.x) * rpb) {
    const int64_t q = u / a.h_rows, i = u - q * a.h_rows;
    const double* h0 = a.H + (49 * q) * gelems + i * a.h_cols;
    double* base = a.dst + q * a.dst_stride;
    for (int64_t j = int64_t(lt) * V; j < a.h_cols; j += step) {
      double cq[7][4][V];  // child c's quadrant (0 = 11, 1 = 12, 2 = 21, 3 = 22) at this position
      const double* hp = h0 + j;
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        double h[7][V];
#pragma unroll
        for (int t = 0; t < 7; ++t) {
          ldv<V>(hp, h[t]);
          hp += gelems;
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
          double q4[4];
          comb4<VARIANT>(h[0][e], h[1][e], h[2][e], h[3][e], h[4][e], h[5][e], h[6][e], q4);
#pragma unroll
          for (int k = 0; k < 4; ++k) cq[c][k][e] = q4[k];
        }
      }
      // node quadrant QK at child-quadrant k: comb4 over the children's quadrant-k values
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double o[4][V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
          double q4[4];
          comb4<VARIANT>(cq[0][k][e], cq[1][k][e], cq[2][k][e], cq[3][k][e], cq[4][k][e], cq[5][k][e], cq[6][k][e],
                         q4);
#pragma unroll
          for (int QK = 0; QK < 4; ++QK) o[QK][e] = q4[QK];
        }
        const int64_t sr = (k >> 1) * a.h_rows, sc = (k & 1) * a.h_cols;  // sub-block inside a quadrant
#pragma unroll
        for (int QK = 0; QK < 4; ++QK)
          st_quad<V>(a, base, i + sr + (QK >> 1) * 2 * a.h_rows, j + sc + (QK & 1) * 2 * a.h_cols, o[QK]);
      }
    }
  }
}

// ---------------------------------------------------------------- plan + arena
struct StrassenPlan {
  int depth;
  int64_t Np, Pp, Mp;
  // arena offsets (bytes)
  size_t offS[2], offT[2], offH, offC[2], total;
};

inline int64_t ipow7(int d) {
  int64_t r = 1;
  for (int i = 0; i < d; ++i) r *= 7;
  return r;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Formation schedule (levels from -> to per pass): an odd remaining depth >= 3 starts with a
// three-level pass, then two levels per pass, a single level only when d = 1.  The produced
// levels alternate between two buffers, the last (level d, read by the leaf GEMM) in buffer 0:
// pass k writes buffer (ns - 1 - k) % 2.
inline int form_schedule(int d, int (*steps)[2]) {
  int ns = 0;
  for (int l = 0; l < d;) {
    const int r = d - l;
    const int to = (r % 2 == 1 && r >= 3) ? l + 3 : (r >= 2 ? l + 2 : l + 1);
    steps[ns][0] = l;
    steps[ns][1] = to;
    ++ns;
    l = to;
  }
  return ns;
}
// Combination schedule: two levels per pass from the deepest level down, a single level last
// when one remains; the k-th pass writing an intermediate level (> 0) uses buffer k % 2.
inline int combine_schedule(int d, int (*steps)[2]) {
  int ns = 0;
  for (int l_from = d; l_from > 0;) {
    const int l = l_from >= 2 ? l_from - 2 : l_from - 1;
    steps[ns][0] = l_from;
    steps[ns][1] = l;
    ++ns;
    l_from = l;
  }
  return ns;
}

// levels >= 0: pad each dim to a multiple of 2^(levels+1) (keeps every level's row pitch
// even, so 16-byte vectors apply); levels == -1: the paper's square plan.
inline bool make_strassen_plan(int64_t N, int64_t P, int64_t M, int levels, StrassenPlan* pl) {
  if (N < 1 || P < 1 || M < 1 || levels < -1 || levels > 8) return false;
  if (levels == -1) {
    int64_t X = N > P ? N : P;
    X = X > M ? X : M;
    int lg = 0;
    while ((int64_t(1) << (lg + 1)) <= X) ++lg;
    int k = lg - 4;
    if (k < 0) k = 0;
    const int64_t m = (X >> k) + 1;
    const int64_t Y = m << k;
    pl->depth = k;
    pl->Np = pl->Pp = pl->Mp = Y;
    if (k > 8) return false;
  } else {
    const int64_t q = int64_t(2) << levels;
    pl->depth = levels;
    pl->Np = cdiv(N, q) * q;
    pl->Pp = cdiv(P, q) * q;
    pl->Mp = cdiv(M, q) * q;
  }
  const int d = pl->depth;
  auto lvl = [&](int l, int64_t r, int64_t c) -> size_t {  // bytes of level l for an r x c root
    if (l <= 0) return 0;
    return size_t(ipow7(l)) * size_t(r >> l) * size_t(c >> l) * sizeof(double);
  };
  // buffers sized for exactly the levels the schedules write into them
  int fs[16][2], cs[16][2];
  const int nf = form_schedule(d, fs), nc = combine_schedule(d, cs);
  size_t s0 = 0, s1 = 0, t0 = 0, t1 = 0, c0 = 0, c1 = 0;
  for (int k = 0; k < nf; ++k) {
    const int l = fs[k][1];
    size_t& sb = ((nf - 1 - k) % 2) ? s1 : s0;
    size_t& tb = ((nf - 1 - k) % 2) ? t1 : t0;
    sb = sb > lvl(l, pl->Np, pl->Pp) ? sb : lvl(l, pl->Np, pl->Pp);
    tb = tb > lvl(l, pl->Pp, pl->Mp) ? tb : lvl(l, pl->Pp, pl->Mp);
  }
  for (int k = 0, produced = 0; k < nc; ++k) {
    const int l = cs[k][1];
    if (l == 0) continue;
    size_t& cb = (produced % 2) ? c1 : c0;
    cb = cb > lvl(l, pl->Np, pl->Mp) ? cb : lvl(l, pl->Np, pl->Mp);
    ++produced;
  }
  const size_t h = lvl(d, pl->Np, pl->Mp);
  size_t off = 0;
  pl->offS[0] = off; off = align256(off + s0);
  pl->offS[1] = off; off = align256(off + s1);
  pl->offT[0] = off; off = align256(off + t0);
  pl->offT[1] = off; off = align256(off + t1);
  pl->offH = off;    off = align256(off + h);
  pl->offC[0] = off; off = align256(off + c0);
  pl->offC[1] = off; off = align256(off + c1);
  pl->total = (d == 0) ? 0 : off;
  return true;
}

// threads per row unit: the smallest power of two (32 .. 256) covering the row's vectors
inline int tpr_shift(int64_t h_cols, int v) {
  const int64_t vecs = cdiv(h_cols, v);
  int s = 5;
  while (s < 8 && (int64_t(1) << s) < vecs) ++s;
  return s;
}

// vector width usable by every access of a launch: base pointers 8 V-byte aligned, row pitches,
// node strides and quadrant widths multiples of V
inline int pick_vec(const void* p0, const void* p1, int64_t pitch, int64_t stride, int64_t h_cols) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p0) | reinterpret_cast<uintptr_t>(p1);
  for (int v = 4; v > 1; v >>= 1)
    if ((a & (8 * v - 1)) == 0 && pitch % v == 0 && stride % v == 0 && h_cols % v == 0) return v;
  return 1;
}

template <auto KERN>
inline unsigned grid_for(int64_t units, int tprs, int sms) {
  static int per_sm = 0;  // resident blocks per SM of this kernel
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, KERN, 256, 0) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      per_sm = 4;
    }
  }
  int64_t b = cdiv(units, int64_t(256 >> tprs));
  const int64_t cap = int64_t(sms) * per_sm;  // one full wave, grid-stride beyond it
  if (b > cap) b = cap;
  return unsigned(b < 1 ? 1 : b);
}

template <int VARIANT, int SIDE>
cudaError_t launch_form_side(const FormArgs& fa, int v, int sms, cudaStream_t st) {
  const int64_t units = fa.u1 - fa.u0;
  const int tprs = tpr_shift(fa.h_cols, v);
  if (v == 4) {
    constexpr auto k = strassen_form_kernel<VARIANT, SIDE, 4>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, tprs);
  } else if (v == 2) {
    constexpr auto k = strassen_form_kernel<VARIANT, SIDE, 2>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, tprs);
  } else {
    constexpr auto k = strassen_form_kernel<VARIANT, SIDE, 1>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, tprs);
  }
  note_launch();
  return cudaGetLastError();
}

template <int VARIANT, int SIDE>
cudaError_t launch_form_child_side(const FormArgs& fa, int child, int v, int sms, cudaStream_t st) {
  const int64_t units = fa.u1 - fa.u0;
  const int tprs = tpr_shift(fa.h_cols, v);
  if (v == 4) {
    constexpr auto k = strassen_form_child_kernel<VARIANT, SIDE, 4>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, child, tprs);
  } else if (v == 2) {
    constexpr auto k = strassen_form_child_kernel<VARIANT, SIDE, 2>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, child, tprs);
  } else {
    constexpr auto k = strassen_form_child_kernel<VARIANT, SIDE, 1>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, child, tprs);
  }
  note_launch();
  return cudaGetLastError();
}

template <int VARIANT>
cudaError_t launch_form_child(int side, const FormArgs& fa, int child, int v, int sms, cudaStream_t st) {
  return side == 0 ? launch_form_child_side<VARIANT, 0>(fa, child, v, sms, st)
                   : launch_form_child_side<VARIANT, 1>(fa, child, v, sms, st);
}

template <int VARIANT>
cudaError_t launch_form_level(int side, const FormArgs& fa, int v, int sms, cudaStream_t st) {
  return side == 0 ? launch_form_side<VARIANT, 0>(fa, v, sms, st) : launch_form_side<VARIANT, 1>(fa, v, sms, st);
}

template <int VARIANT, int SIDE>
cudaError_t launch_form2_side(const FormArgs& fa, int v, int sms, cudaStream_t st) {
  if (v > 2) v = 2;  // 16 inputs x V live per thread: V = 4 would spill (V = 1: same time)
  const int64_t units = fa.u1 - fa.u0;
  const int tprs = tpr_shift(fa.h_cols, v);
  if (v == 2) {
    constexpr auto k = strassen_form2_kernel<VARIANT, SIDE, 2>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, tprs);
  } else {
    constexpr auto k = strassen_form2_kernel<VARIANT, SIDE, 1>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(fa, tprs);
  }
  note_launch();
  return cudaGetLastError();
}

template <int VARIANT, int SIDE>
cudaError_t launch_form3_side(const FormArgs& fa, int sms, cudaStream_t st) {
  constexpr auto k = strassen_form3_kernel<VARIANT, SIDE>;
  cudaError_t e = smem_attr_once<k>(F3_SMEM);
  if (e != cudaSuccess) return e;
  static int per_sm = 0;  // resident blocks per SM (shared memory bound: 3 x 64 KB)
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, F3_THREADS, F3_SMEM) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      per_sm = 2;
    }
  }
  const int64_t units = fa.u1 - fa.u0;
  int tprs = tpr_shift(fa.h_cols, 1);
  if (tprs > 7) tprs = 7;  // at most one row unit per 128-thread block
  int64_t b = cdiv(units, int64_t(F3_THREADS >> tprs));
  const int64_t cap = int64_t(sms) * per_sm;
  if (b > cap) b = cap;
  k<<<unsigned(b < 1 ? 1 : b), F3_THREADS, F3_SMEM, st>>>(fa, tprs);
  note_launch();
  return cudaGetLastError();
}

template <int VARIANT>
cudaError_t launch_form3_level(int side, const FormArgs& fa, int sms, cudaStream_t st) {
  return side == 0 ? launch_form3_side<VARIANT, 0>(fa, sms, st) : launch_form3_side<VARIANT, 1>(fa, sms, st);
}

template <int VARIANT>
cudaError_t launch_form2_level(int side, const FormArgs& fa, int v, int sms, cudaStream_t st) {
  return side == 0 ? launch_form2_side<VARIANT, 0>(fa, v, sms, st) : launch_form2_side<VARIANT, 1>(fa, v, sms, st);
}

template <int VARIANT>
cudaError_t launch_combine_level(const CombineArgs& ca, int v, int sms, cudaStream_t st) {
  const int64_t units = ca.cnt * ca.h_rows;
  const int tprs = tpr_shift(ca.h_cols, v);
  if (v == 4) {
    constexpr auto k = strassen_combine_kernel<VARIANT, 4>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(ca, tprs);
  } else if (v == 2) {
    constexpr auto k = strassen_combine_kernel<VARIANT, 2>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(ca, tprs);
  } else {
    constexpr auto k = strassen_combine_kernel<VARIANT, 1>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(ca, tprs);
  }
  note_launch();
  return cudaGetLastError();
}

template <int VARIANT>
cudaError_t launch_combine2_level(const CombineArgs& ca, int v, int sms, cudaStream_t st) {
  if (v > 2) v = 2;  // 28 child-quadrant values x V live per thread
  const int64_t units = ca.cnt * ca.h_rows;
  const int tprs = tpr_shift(ca.h_cols, v);
  if (v == 2) {
    constexpr auto k = strassen_combine2_kernel<VARIANT, 2>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(ca, tprs);
  } else {
    constexpr auto k = strassen_combine2_kernel<VARIANT, 1>;
    k<<<grid_for<k>(units, tprs, sms), 256, 0, st>>>(ca, tprs);
  }
  note_launch();
  return cudaGetLastError();
}

// Phases of one product (mm_dist_step runs them separately so the first B-side formation pass
// can follow the broadcast of B panel by panel; mm_strassen runs SP_ALL):
enum { SP_FORM_A = 1, SP_FORM_B_FIRST = 2, SP_FORM_B_REST = 4, SP_LEAF_COMBINE = 8, SP_ALL = 15 };

// Span (levels) of the first formation pass at depth d >= 1, and its row units: the first pass on
// the B side reads B rows {u + r * (Pp >> span) : r < 2^span} for unit u in [0, Pp >> span).
inline int first_form_span(int d) {
  int steps[16][2];
  form_schedule(d, steps);
  return steps[0][1] - steps[0][0];
}

template <int VARIANT>
cudaError_t run_strassen(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                         const StrassenPlan& pl, char* ws, int sms, cudaStream_t st, int phases = SP_ALL,
                         int64_t b_u0 = 0, int64_t b_u1 = INT64_MAX) {
  const int d = pl.depth;
  if (d == 0) {
    if (!(phases & SP_LEAF_COMBINE)) return cudaSuccess;
    GemmProblem pr{A, B, C, N, P, M, P, M, M, 0, 0, 0, 1};
    return launch_dgemm(pr, st, sms);
  }
  cudaError_t e;
  double* S[2] = {reinterpret_cast<double*>(ws + pl.offS[0]), reinterpret_cast<double*>(ws + pl.offS[1])};
  double* T[2] = {reinterpret_cast<double*>(ws + pl.offT[0]), reinterpret_cast<double*>(ws + pl.offT[1])};
  double* Hb = reinterpret_cast<double*>(ws + pl.offH);
  double* Cb[2] = {reinterpret_cast<double*>(ws + pl.offC[0]), reinterpret_cast<double*>(ws + pl.offC[1])};
  // Formation schedule (form_schedule): an odd remaining depth >= 3 starts with a three-level pass
  // (strassen_form3_kernel), then two levels per pass (strassen_form2_kernel), a single level only
  // when d = 1, so the deepest -- largest -- intermediate levels are never written.  Pass k writes
  // buffer (ns - 1 - k) % 2 (the last pass, level d read by the leaf GEMM, writes buffer 0) and
  // reads what pass k - 1 wrote; make_strassen_plan sizes each buffer for the levels written to it.
  int steps[16][2];
  const int ns = form_schedule(d, steps);
  for (int side = 0; side < 2; ++side) {
    const int want = side == 0 ? SP_FORM_A : (SP_FORM_B_FIRST | SP_FORM_B_REST);
    if (!(phases & want)) continue;
    NvtxRange nvtx(side == 0 ? "strassen form (A side)" : "strassen form (B side)");
    const int64_t R = side == 0 ? pl.Np : pl.Pp, Ccols = side == 0 ? pl.Pp : pl.Mp;
    double** buf = side == 0 ? S : T;
    for (int k = 0; k < ns; ++k) {
      if (side == 1 && !(phases & (k == 0 ? SP_FORM_B_FIRST : SP_FORM_B_REST))) continue;
      const int l = steps[k][0], span = steps[k][1] - l, two = span == 2;
      FormArgs fa;
      const int64_t r_l = R >> l, c_l = Ccols >> l;
      if (l == 0) {
        fa.src = side == 0 ? A : B;
        fa.src_pitch = side == 0 ? P : M;
        fa.src_stride = 0;
        fa.rows_valid = side == 0 ? N : P;
        fa.cols_valid = side == 0 ? P : M;
      } else {
        fa.src = buf[(ns - k) % 2];  // level l was produced by step k - 1: buffer (ns - 1 - (k - 1)) % 2
        fa.src_pitch = c_l;
        fa.src_stride = r_l * c_l;
        fa.rows_valid = r_l;
        fa.cols_valid = c_l;
      }
      fa.dst = buf[(ns - 1 - k) % 2];
      fa.h_rows = r_l >> span;
      fa.h_cols = c_l >> span;
      fa.cnt = ipow7(l);
      fa.u0 = 0;
      fa.u1 = fa.cnt * fa.h_rows;
      if (side == 1 && k == 0) {  // the B rows of this unit range are the ones that have arrived
        fa.u0 = b_u0 < fa.u1 ? b_u0 : fa.u1;
        fa.u1 = b_u1 < fa.u1 ? b_u1 : fa.u1;
        if (fa.u0 >= fa.u1) continue;
      }
      const int v = pick_vec(fa.src, fa.dst, fa.src_pitch, fa.src_stride, fa.h_cols);
      e = span == 3 ? launch_form3_level<VARIANT>(side, fa, sms, st)
          : two     ? launch_form2_level<VARIANT>(side, fa, v, sms, st)
                    : launch_form_level<VARIANT>(side, fa, v, sms, st);
      if (e != cudaSuccess) return e;
    }
  }
  if (!(phases & SP_LEAF_COMBINE)) return cudaSuccess;
  // the 7^d leaf products, one batched DMMA launch -- for Strassen-Winograd at depth >= 3 with
  // the deepest combination fused into its epilogue (NEXT-1, gemm_comb.cuh: level d - 1 written
  // straight into Hb, or into C at d = 1).  Measured at 8192^3 (profiles/r02/next1_comb.log):
  // d = 3 22.38 -> 22.17 ms; d = 2 24.28 -> 24.65 ms (the seven children of a parent then span
  // 7 x 64 MB of operands, more than L2 holds), hence the depth rule; it also needs >= 4 waves of
  // CTAs (a CTA computes seven products).  MM_STRASSEN_FUSED_COMBINE=0 / 1 forces it off / on.
  int dc = d;  // the level the combination passes start from
  {
    NvtxRange nvtx("strassen leaf products");
    const int64_t n = pl.Np >> d, p = pl.Pp >> d, m = pl.Mp >> d;
    GemmProblem pr{S[0], T[0], Hb, n, p, m, p, m, m, n * p, p * m, n * m, ipow7(d)};
    static const int force = [] {
      const char* v = std::getenv("MM_STRASSEN_FUSED_COMBINE");
      return v ? (v[0] == '1' ? 1 : 0) : -1;
    }();
    const int64_t ctas = cdiv(n, int64_t(GemmComb::BM)) * cdiv(m, int64_t(GemmComb::BN)) * ipow7(d - 1);
    const bool fuse = force == 1 || (force == -1 && d >= 3 && ctas >= 4 * 3 * int64_t(sms));
    e = cudaErrorNotSupported;
    if (VARIANT == SV_WINOGRAD && fuse) {
      CombStore o;
      if (d == 1) {
        o = CombStore{C, M, 0, N, M};
      } else {
        const int64_t rl = pl.Np >> (d - 1), cl = pl.Mp >> (d - 1);
        o = CombStore{Hb, cl, rl * cl, rl, cl};
      }
      e = launch_dgemm_comb(pr, o, st);
      if (e == cudaSuccess) dc = d - 1;
      else if (e == cudaErrorNotSupported) cudaGetLastError();
      else return e;
    }
    if (dc == d) {
      e = launch_dgemm(pr, st, sms);
      if (e != cudaSuccess) return e;
    }
  }
  NvtxRange nvtx_combine("strassen combination");
  // Combination schedule (combine_schedule): two levels per pass from the deepest (largest) level
  // down, a single level last when one remains; the j-th intermediate level produced (> 0) is
  // written to Cb[j % 2] and read by the next pass.  At d = 3 the passes are 3 -> 1 (into Cb[0])
  // and 1 -> 0 (into C), so Cb[1] is never used and make_strassen_plan gives it no bytes.
  const double* Hsrc = Hb;
  int produced = 0;
  int csteps[16][2];
  const int ncs = combine_schedule(dc, csteps);
  for (int k = 0; k < ncs; ++k) {
    const int l_from = csteps[k][0], l = csteps[k][1];  // this pass reads level l_from, writes level l
    const bool two = l_from - l == 2;
    CombineArgs ca;
    const int64_t r_l = pl.Np >> l, c_l = pl.Mp >> l;
    ca.H = Hsrc;
    if (l == 0) {
      ca.dst = C;
      ca.dst_pitch = M;
      ca.dst_stride = 0;
      ca.rows_valid = N;
      ca.cols_valid = M;
    } else {
      ca.dst = Cb[produced % 2];
      ca.dst_pitch = c_l;
      ca.dst_stride = r_l * c_l;
      ca.rows_valid = r_l;
      ca.cols_valid = c_l;
    }
    ca.h_rows = two ? r_l / 4 : r_l / 2;
    ca.h_cols = two ? c_l / 4 : c_l / 2;
    ca.cnt = ipow7(l);
    const int v = pick_vec(ca.dst, ca.H, ca.dst_pitch, ca.dst_stride, ca.h_cols);
    e = two ? launch_combine2_level<VARIANT>(ca, v, sms, st) : launch_combine_level<VARIANT>(ca, v, sms, st);
    if (e != cudaSuccess) return e;
    if (l > 0) Hsrc = ca.dst, ++produced;
  }
  return cudaSuccess;
}

}  // namespace mmk
