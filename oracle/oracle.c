/*
 * oracle.c -- CPU oracle for Hedtke, "Methods of Matrix Multiplication" (arXiv 1106.1347).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): loaded by tests/, __graft_entry__.smoke()
 * and bench.py's CPU legs; never by the product path.  Shares no code with csrc/.
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fPIC -shared -o liboracle.so oracle.c -lm
 * (no -march=native: SSE2 binary64 arithmetic, FLT_EVAL_METHOD == 0).
 *
 * Every function follows the paper's text step by step; "P:L" cites
 * /root/reference/PAPER.md line L.
 */
#define _POSIX_C_SOURCE 199309L
#include "oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#if !defined(FLT_EVAL_METHOD) || FLT_EVAL_METHOD != 0
#error "oracle needs FLT_EVAL_METHOD == 0 (plain binary64 arithmetic)"
#endif

#define IDX(i, j, ld) ((int64_t)(i) * (int64_t)(ld) + (int64_t)(j))

static int bad_dims(const void* A, const void* B, const void* C, int64_t N, int64_t P, int64_t M) {
  return A == NULL || B == NULL || C == NULL || N < 1 || P < 1 || M < 1;
}

/* ------------------------------------------------------------------ self check */
int or_selfcheck(void) {
  /* contraction detector: a*b rounds to 1.0, so a*b + c == 0 exactly; fused gives -2^-60 */
  volatile double a = 1.0 + ldexp(1.0, -30), b = 1.0 - ldexp(1.0, -30), c = -1.0;
  double r = a * b + c;
  if (r != 0.0) return -1;
  /* Kahan pin: [2^53, 1, 1] sums to 2^53 + 2; plain summation gives 2^53 */
  {
    volatile double x[3];
    double sum = 0.0, err = 0.0, t;
    int i;
    x[0] = ldexp(1.0, 53); x[1] = 1.0; x[2] = 1.0;
    for (i = 0; i < 3; i++) {
      err = err + x[i];
      t = sum + err;
      err = (sum - t) + err;
      sum = t;
    }
    if (sum != ldexp(1.0, 53) + 2.0) return -2;
  }
  return 0;
}

/* ------------------------------------------------------------------ Section 1 */
void or_plus(const double* X, const double* Y, double* Z, int64_t r, int64_t c) {
  int64_t i, j;
  for (i = 0; i < r; i++)
    for (j = 0; j < c; j++) Z[IDX(i, j, c)] = X[IDX(i, j, c)] + Y[IDX(i, j, c)];
}

void or_minus(const double* X, const double* Y, double* Z, int64_t r, int64_t c) {
  int64_t i, j;
  for (i = 0; i < r; i++)
    for (j = 0; j < c; j++) Z[IDX(i, j, c)] = X[IDX(i, j, c)] - Y[IDX(i, j, c)];
}

double or_max_d(double x, double y) { return (x >= y) ? x : y; }
int64_t or_max_i(int64_t x, int64_t y) { return (x >= y) ? x : y; }

double or_norm_inf(const double* X, int64_t r, int64_t c) {
  /* max over rows of the row sum of |X_ij|, row sums left to right */
  double res = 0.0;
  int64_t i, j;
  for (i = 0; i < r; i++) {
    double s = 0.0;
    for (j = 0; j < c; j++) s = s + fabs(X[IDX(i, j, c)]);
    res = or_max_d(s, res);
  }
  return res;
}

void or_scalar_mul(double alpha, const double* X, double* Z, int64_t r, int64_t c) {
  int64_t i, j;
  for (i = 0; i < r; i++)
    for (j = 0; j < c; j++) Z[IDX(i, j, c)] = alpha * X[IDX(i, j, c)];
}

/* ------------------------------------------------------------------ Section 2.1 / 2.2 */
static double entry_standard(const double* A, const double* B, int64_t P, int64_t M, int64_t i, int64_t j) {
  double aux = 0.0;
  int64_t k;
  for (k = 0; k < P; k++) aux = aux + A[IDX(i, k, P)] * B[IDX(k, j, M)];
  return aux;
}

static double entry_fma(const double* A, const double* B, int64_t P, int64_t M, int64_t i, int64_t j) {
  double aux = 0.0;
  int64_t k;
  for (k = 0; k < P; k++) aux = fma(A[IDX(i, k, P)], B[IDX(k, j, M)], aux);
  return aux;
}

static double entry_kahan(const double* A, const double* B, int64_t P, int64_t M, int64_t i, int64_t j) {
  /* P:122-132, with x_k = A_ik * B_kj */
  double t, sum = 0.0, err = 0.0;
  int64_t k;
  for (k = 0; k < P; k++) {
    double x = A[IDX(i, k, P)] * B[IDX(k, j, M)];
    err = err + x;
    t = sum + err;
    err = (sum - t) + err;
    sum = t;
  }
  return sum;
}

static double entry_unroll(int u, const double* A, const double* B, int64_t P, int64_t M, int64_t i, int64_t j) {
  double aux = 0.0;
  int64_t g, k, groups = P / u;
  for (g = 0; g < groups; g++) {
    int64_t k0 = g * u;
    double s = A[IDX(i, k0, P)] * B[IDX(k0, j, M)] + A[IDX(i, k0 + 1, P)] * B[IDX(k0 + 1, j, M)];
    if (u >= 3) s = s + A[IDX(i, k0 + 2, P)] * B[IDX(k0 + 2, j, M)];
    if (u >= 4) s = s + A[IDX(i, k0 + 3, P)] * B[IDX(k0 + 3, j, M)];
    aux = aux + s;
  }
  for (k = groups * u; k < P; k++) aux = aux + A[IDX(i, k, P)] * B[IDX(k, j, M)];
  return aux;
}

int or_naive_standard(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, j;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) C[IDX(i, j, M)] = entry_standard(A, B, P, M, i, j);
  return 0;
}

int or_naive_on_array(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, j, k;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) {
      C[IDX(i, j, M)] = 0.0;
      for (k = 0; k < P; k++) C[IDX(i, j, M)] = C[IDX(i, j, M)] + A[IDX(i, k, P)] * B[IDX(k, j, M)];
    }
  return 0;
}

int or_naive_kahan(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, j;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) C[IDX(i, j, M)] = entry_kahan(A, B, P, M, i, j);
  return 0;
}

int or_naive_unroll(int u, const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, j;
  if (bad_dims(A, B, C, N, P, M) || u < 2 || u > 4) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) C[IDX(i, j, M)] = entry_unroll(u, A, B, P, M, i, j);
  return 0;
}

int or_naive_fma(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, j;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) C[IDX(i, j, M)] = entry_fma(A, B, P, M, i, j);
  return 0;
}

/* Reading R2 continued: the chain of or_naive_fma started from C's current value,
 * C_ij = fma(A_i,K-1 B_K-1,j, ... fma(A_i0 B_0j, C_ij)), strided operands.  Consecutive k-panels
 * therefore compose to or_naive_fma (SURVEY 8(f) NEXT-4's panelised product). */
int or_naive_fma_acc(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                     int64_t N, int64_t K, int64_t M) {
  int64_t i, j, k;
  if (!A || !B || !C || N < 1 || K < 1 || M < 1 || lda < K || ldb < M || ldc < M) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) {
      double aux = C[i * ldc + j];
      for (k = 0; k < K; k++) aux = fma(A[i * lda + k], B[k * ldb + j], aux);
      C[i * ldc + j] = aux;
    }
  return 0;
}

/* NEXT-4 for NaivKahan: the loop of P:122-132 (fused: err = fma(a, b, err), reading R22) resumed
 * from a given state -- sum = S_ij, err = E_ij -- over k = 0..K-1 of strided panels; the state is
 * written back.  Consecutive k-panels started from (0, 0) therefore compose to or_naive_kahan. */
int or_naive_kahan_acc(const double* A, int64_t lda, const double* B, int64_t ldb, double* S, double* E,
                       int64_t N, int64_t K, int64_t M, int fused) {
  int64_t i, j, k;
  if (!A || !B || !S || !E || N < 1 || K < 1 || M < 1 || lda < K || ldb < M) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) {
      double t, sum = S[i * M + j], err = E[i * M + j];
      for (k = 0; k < K; k++) {
        if (fused) {
          err = fma(A[i * lda + k], B[k * ldb + j], err);
        } else {
          double x = A[i * lda + k] * B[k * ldb + j];
          err = err + x;
        }
        t = sum + err;
        err = (sum - t) + err;
        sum = t;
      }
      S[i * M + j] = sum;
      E[i * M + j] = err;
    }
  return 0;
}

/* ------------------------------------------------------------------ Section 2.3 */
static double winograd_y(const double* A, int64_t P, int64_t i) {
  double y = 0.0;
  int64_t j, gamma = P / 2;
  for (j = 0; j < gamma; j++) y = y + A[IDX(i, 2 * j, P)] * A[IDX(i, 2 * j + 1, P)];
  return y;
}

static double winograd_z(const double* B, int64_t P, int64_t M, int64_t k) {
  double z = 0.0;
  int64_t j, gamma = P / 2;
  for (j = 0; j < gamma; j++) z = z + B[IDX(2 * j, k, M)] * B[IDX(2 * j + 1, k, M)];
  return z;
}

static double winograd_entry_yz(const double* A, const double* B, int64_t P, int64_t M, int64_t i, int64_t k,
                                double yi, double zk) {
  /* (acc - y_i) - z_k, then + A_{i,P} B_{P,k} if P odd ("B_{B,k}" read as B_{P,k}) */
  double acc = 0.0, c;
  int64_t j, gamma = P / 2;
  for (j = 0; j < gamma; j++)
    acc = acc + (A[IDX(i, 2 * j, P)] + B[IDX(2 * j + 1, k, M)]) * (A[IDX(i, 2 * j + 1, P)] + B[IDX(2 * j, k, M)]);
  c = (acc - yi) - zk;
  if (P % 2 == 1) c = c + A[IDX(i, P - 1, P)] * B[IDX(P - 1, k, M)];
  return c;
}

int or_winograd_yz(const double* A, const double* B, double* y, double* z, int64_t N, int64_t P, int64_t M) {
  int64_t i, k;
  if (bad_dims(A, B, y, N, P, M) || z == NULL) return -1;
  for (i = 0; i < N; i++) y[i] = winograd_y(A, P, i);
  for (k = 0; k < M; k++) z[k] = winograd_z(B, P, M, k);
  return 0;
}

int or_winograd_original(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, k;
  double *y, *z;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  y = (double*)malloc(sizeof(double) * (size_t)N);
  z = (double*)malloc(sizeof(double) * (size_t)M);
  if (!y || !z) { free(y); free(z); return -2; }
  or_winograd_yz(A, B, y, z, N, P, M);
  for (i = 0; i < N; i++)
    for (k = 0; k < M; k++) C[IDX(i, k, M)] = winograd_entry_yz(A, B, P, M, i, k, y[i], z[k]);
  free(y);
  free(z);
  return 0;
}

/* NEXT-4 for WinogradOriginal: the pair sum of P:189-192 (fused: acc = fma(.., .., acc)) resumed
 * from Acc_ik over the K/2 pairs of a strided k-panel (K even), written back; and the epilogue
 * C = (acc - y_i) - z_k of an even-P product. */
int or_winograd_pairs_acc(const double* A, int64_t lda, const double* B, int64_t ldb, double* Acc, int64_t N,
                          int64_t K, int64_t M, int fused) {
  int64_t i, k, j;
  if (!A || !B || !Acc || N < 1 || K < 2 || K % 2 || M < 1 || lda < K || ldb < M) return -1;
  for (i = 0; i < N; i++)
    for (k = 0; k < M; k++) {
      double acc = Acc[i * M + k];
      for (j = 0; j < K / 2; j++) {
        double u = A[i * lda + 2 * j] + B[(2 * j + 1) * ldb + k];
        double v = A[i * lda + 2 * j + 1] + B[(2 * j) * ldb + k];
        acc = fused ? fma(u, v, acc) : acc + u * v;
      }
      Acc[i * M + k] = acc;
    }
  return 0;
}

int or_winograd_finish(const double* Acc, const double* y, const double* z, double* C, int64_t N, int64_t M) {
  int64_t i, k;
  if (!Acc || !y || !z || !C || N < 1 || M < 1) return -1;
  for (i = 0; i < N; i++)
    for (k = 0; k < M; k++) C[i * M + k] = (Acc[i * M + k] - y[i]) - z[k];
  return 0;
}

int or_lambda(double nA, double nB) {
  /* find integer lambda with 1/2 <= 2^(2 lambda) nA / nB <= 2.
   * nA = mA 2^eA, nB = mB 2^eB with m in [1/2, 1); d = eB - eA.
   * ratio = 2^(2 lambda - d) * (mA / mB), and mA / mB lies in (1/2, 2).
   * d even: lambda = d/2 is the only solution.
   * d odd:  lambda = (d+1)/2 valid iff mA <= mB; lambda = (d-1)/2 valid iff mA >= mB;
   *         both valid iff mA == mB -> take the larger |lambda| (reading R7). */
  int eA, eB, d;
  double mA, mB;
  if (nA == 0.0 || nB == 0.0) return 0;
  mA = frexp(nA, &eA);
  mB = frexp(nB, &eB);
  d = eB - eA;
  if (d % 2 == 0) return d / 2;
  if (mA < mB) return (d + 1) / 2;
  if (mA > mB) return (d - 1) / 2;
  return (d > 0) ? (d + 1) / 2 : (d - 1) / 2;
}

int or_winograd_scaled(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                       int32_t* lambda_out) {
  double nA, nB, *As, *Bs;
  int lambda, rc;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  nA = or_norm_inf(A, N, P);
  nB = or_norm_inf(B, P, M);
  lambda = or_lambda(nA, nB);
  As = (double*)malloc(sizeof(double) * (size_t)(N * P));
  Bs = (double*)malloc(sizeof(double) * (size_t)(P * M));
  if (!As || !Bs) { free(As); free(Bs); return -2; }
  or_scalar_mul(ldexp(1.0, lambda), A, As, N, P);  /* 2^lambda A */
  or_scalar_mul(ldexp(1.0, -lambda), B, Bs, P, M); /*        2^-lambda B */
  rc = or_winograd_original(As, Bs, C, N, P, M);   /* result is not rescaled */
  free(As);
  free(Bs);
  if (lambda_out) *lambda_out = lambda;
  return rc;
}

/* ------------------------------------------------------------------ Section 2.4 */
static int64_t g_base_products = 0, g_block_ops = 0;
static double* g_trace = NULL;
static int64_t g_trace_cap = 0, g_trace_len = 0;

void or_strassen_trace(double* buf, int64_t cap) {
  g_trace = buf;
  g_trace_cap = cap;
  g_trace_len = 0;
}
int64_t or_strassen_trace_len(void) { return g_trace_len; }

void or_strassen_counters(int64_t* base_products, int64_t* block_ops) {
  if (base_products) *base_products = g_base_products;
  if (block_ops) *block_ops = g_block_ops;
}

void or_strassen_plan_paper(int64_t N, int64_t P, int64_t M, int32_t* k, int64_t* m, int64_t* Y) {
  /* P:286 */
  int64_t X = or_max_i(N, or_max_i(P, M));
  int32_t lg = 0, kk;
  while (((int64_t)1 << (lg + 1)) <= X) lg++; /* floor(log2 X) */
  kk = lg - 4;
  if (kk < 0) kk = 0; /* reading R8 */
  *k = kk;
  *m = (X >> kk) + 1; /* floor(X 2^-k) + 1 */
  *Y = (*m) << kk;
}

void or_strassen_plan_levels(int64_t N, int64_t P, int64_t M, int32_t levels, int64_t align,
                             int64_t* Np, int64_t* Pp, int64_t* Mp) {
  int64_t q = align << levels;
  *Np = (N + q - 1) / q * q;
  *Pp = (P + q - 1) / q * q;
  *Mp = (M + q - 1) / q * q;
}

/* strided dense helpers: Z (ldz) = X (ldx) +/- Y (ldy), r x c */
static void blk_add(const double* X, int64_t ldx, const double* Y, int64_t ldy, double* Z, int64_t ldz,
                    int64_t r, int64_t c) {
  int64_t i, j;
  for (i = 0; i < r; i++)
    for (j = 0; j < c; j++) Z[IDX(i, j, ldz)] = X[IDX(i, j, ldx)] + Y[IDX(i, j, ldy)];
  g_block_ops++;
}
static void blk_sub(const double* X, int64_t ldx, const double* Y, int64_t ldy, double* Z, int64_t ldz,
                    int64_t r, int64_t c) {
  int64_t i, j;
  for (i = 0; i < r; i++)
    for (j = 0; j < c; j++) Z[IDX(i, j, ldz)] = X[IDX(i, j, ldx)] - Y[IDX(i, j, ldy)];
  g_block_ops++;
}

static void base_product(int base, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t n, int64_t p, int64_t m) {
  /* alpha_{m,0}: the naive algorithm */
  int64_t i, j, k;
  for (i = 0; i < n; i++)
    for (j = 0; j < m; j++) {
      double aux = 0.0;
      if (base == OR_BASE_FMA)
        for (k = 0; k < p; k++) aux = fma(A[IDX(i, k, lda)], B[IDX(k, j, ldb)], aux);
      else
        for (k = 0; k < p; k++) aux = aux + A[IDX(i, k, lda)] * B[IDX(k, j, ldb)];
      C[IDX(i, j, ldc)] = aux;
    }
  /* 1x1 base products are recorded in call order (H_1..H_7 per node) when tracing */
  if (g_trace != NULL && n == 1 && m == 1 && g_trace_len < g_trace_cap) g_trace[g_trace_len++] = C[0];
  g_base_products++;
}

static double* dalloc(int64_t n) { return (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1)); }

/* C (n x m, ldc) = A (n x p, lda) * B (p x m, ldb), `levels` recursion levels */
static void strassen_rec(int variant, int base, const double* A, int64_t lda, const double* B, int64_t ldb,
                         double* C, int64_t ldc, int64_t n, int64_t p, int64_t m, int32_t levels) {
  int64_t n2, p2, m2;
  const double *A11, *A12, *A21, *A22, *B11, *B12, *B21, *B22;
  double *C11, *C12, *C21, *C22;
  if (levels == 0) {
    base_product(base, A, lda, B, ldb, C, ldc, n, p, m);
    return;
  }
  /* Eq. (1): 2 x 2 block decomposition */
  n2 = n / 2; p2 = p / 2; m2 = m / 2;
  A11 = A; A12 = A + p2; A21 = A + n2 * lda; A22 = A21 + p2;
  B11 = B; B12 = B + m2; B21 = B + p2 * ldb; B22 = B21 + m2;
  C11 = C; C12 = C + m2; C21 = C + n2 * ldc; C22 = C21 + m2;
  if (variant == OR_STRASSEN_NAIV) {
    /* P:271-282 */
    double *S = dalloc(n2 * p2), *T = dalloc(p2 * m2);
    double *H1 = dalloc(n2 * m2), *H2 = dalloc(n2 * m2), *H3 = dalloc(n2 * m2), *H4 = dalloc(n2 * m2);
    double *H5 = dalloc(n2 * m2), *H6 = dalloc(n2 * m2), *H7 = dalloc(n2 * m2), *W = dalloc(n2 * m2);
    /* H1 = (A11 + A22)(B11 + B22) */
    blk_add(A11, lda, A22, lda, S, p2, n2, p2);
    blk_add(B11, ldb, B22, ldb, T, m2, p2, m2);
    strassen_rec(variant, base, S, p2, T, m2, H1, m2, n2, p2, m2, levels - 1);
    /* H2 = (A21 + A22) B11 */
    blk_add(A21, lda, A22, lda, S, p2, n2, p2);
    strassen_rec(variant, base, S, p2, B11, ldb, H2, m2, n2, p2, m2, levels - 1);
    /* H3 = A11 (B12 - B22) */
    blk_sub(B12, ldb, B22, ldb, T, m2, p2, m2);
    strassen_rec(variant, base, A11, lda, T, m2, H3, m2, n2, p2, m2, levels - 1);
    /* H4 = A22 (B21 - B11) */
    blk_sub(B21, ldb, B11, ldb, T, m2, p2, m2);
    strassen_rec(variant, base, A22, lda, T, m2, H4, m2, n2, p2, m2, levels - 1);
    /* H5 = (A11 + A12) B22 */
    blk_add(A11, lda, A12, lda, S, p2, n2, p2);
    strassen_rec(variant, base, S, p2, B22, ldb, H5, m2, n2, p2, m2, levels - 1);
    /* H6 = (A21 - A11)(B11 + B12) */
    blk_sub(A21, lda, A11, lda, S, p2, n2, p2);
    blk_add(B11, ldb, B12, ldb, T, m2, p2, m2);
    strassen_rec(variant, base, S, p2, T, m2, H6, m2, n2, p2, m2, levels - 1);
    /* H7 = (A12 - A22)(B21 + B22) */
    blk_sub(A12, lda, A22, lda, S, p2, n2, p2);
    blk_add(B21, ldb, B22, ldb, T, m2, p2, m2);
    strassen_rec(variant, base, S, p2, T, m2, H7, m2, n2, p2, m2, levels - 1);
    /* C11 = H1 + H4 - H5 + H7 (left to right) */
    blk_add(H1, m2, H4, m2, W, m2, n2, m2);
    blk_sub(W, m2, H5, m2, W, m2, n2, m2);
    blk_add(W, m2, H7, m2, C11, ldc, n2, m2);
    /* C12 = H3 + H5 */
    blk_add(H3, m2, H5, m2, C12, ldc, n2, m2);
    /* C21 = H2 + H4 */
    blk_add(H2, m2, H4, m2, C21, ldc, n2, m2);
    /* C22 = H1 + H3 - H2 + H6 (left to right) */
    blk_add(H1, m2, H3, m2, W, m2, n2, m2);
    blk_sub(W, m2, H2, m2, W, m2, n2, m2);
    blk_add(W, m2, H6, m2, C22, ldc, n2, m2);
    free(S); free(T); free(H1); free(H2); free(H3); free(H4); free(H5); free(H6); free(H7); free(W);
  } else {
    /* P:299-312 */
    double *A1 = dalloc(n2 * p2), *A2 = dalloc(n2 * p2), *S = dalloc(n2 * p2);
    double *B1 = dalloc(p2 * m2), *B2 = dalloc(p2 * m2), *T = dalloc(p2 * m2);
    double *H1 = dalloc(n2 * m2), *H2 = dalloc(n2 * m2), *H3 = dalloc(n2 * m2), *H4 = dalloc(n2 * m2);
    double *H5 = dalloc(n2 * m2), *H6 = dalloc(n2 * m2), *H7 = dalloc(n2 * m2);
    double *H8 = dalloc(n2 * m2), *H9 = dalloc(n2 * m2), *W = dalloc(n2 * m2);
    blk_sub(A11, lda, A21, lda, A1, p2, n2, p2); /* A1 = A11 - A21 */
    blk_sub(B22, ldb, B12, ldb, B1, m2, p2, m2); /* B1 = B22 - B12 */
    blk_sub(A22, lda, A1, p2, A2, p2, n2, p2);   /* A2 = A22 - A1 */
    blk_add(B1, m2, B11, ldb, B2, m2, p2, m2);   /* B2 = B1 + B11 */
    strassen_rec(variant, base, A11, lda, B11, ldb, H1, m2, n2, p2, m2, levels - 1); /* H1 = A11 B11 */
    strassen_rec(variant, base, A12, lda, B21, ldb, H2, m2, n2, p2, m2, levels - 1); /* H2 = A12 B21 */
    strassen_rec(variant, base, A2, p2, B2, m2, H3, m2, n2, p2, m2, levels - 1);     /* H3 = A2 B2 */
    blk_add(A21, lda, A22, lda, S, p2, n2, p2);
    blk_sub(B12, ldb, B11, ldb, T, m2, p2, m2);
    strassen_rec(variant, base, S, p2, T, m2, H4, m2, n2, p2, m2, levels - 1);       /* H4 = (A21+A22)(B12-B11) */
    strassen_rec(variant, base, A1, p2, B1, m2, H5, m2, n2, p2, m2, levels - 1);     /* H5 = A1 B1 */
    blk_sub(A12, lda, A2, p2, S, p2, n2, p2);
    strassen_rec(variant, base, S, p2, B22, ldb, H6, m2, n2, p2, m2, levels - 1);    /* H6 = (A12-A2) B22 */
    blk_sub(B21, ldb, B2, m2, T, m2, p2, m2);
    strassen_rec(variant, base, A22, lda, T, m2, H7, m2, n2, p2, m2, levels - 1);    /* H7 = A22 (B21-B2) */
    blk_add(H1, m2, H3, m2, H8, m2, n2, m2);     /* H8 = H1 + H3 */
    blk_add(H8, m2, H4, m2, H9, m2, n2, m2);     /* H9 = H8 + H4 */
    blk_add(H1, m2, H2, m2, C11, ldc, n2, m2);   /* C11 = H1 + H2 */
    blk_add(H9, m2, H6, m2, C12, ldc, n2, m2);   /* C12 = H9 + H6 */
    blk_add(H8, m2, H5, m2, W, m2, n2, m2);      /* C21 = (H8 + H5) + H7 */
    blk_add(W, m2, H7, m2, C21, ldc, n2, m2);
    blk_add(H9, m2, H5, m2, C22, ldc, n2, m2);   /* C22 = H9 + H5 */
    free(A1); free(A2); free(S); free(B1); free(B2); free(T);
    free(H1); free(H2); free(H3); free(H4); free(H5); free(H6); free(H7); free(H8); free(H9); free(W);
  }
}

static int strassen_plan_ok(int64_t N, int64_t P, int64_t M, int32_t levels, int64_t Np, int64_t Pp, int64_t Mp) {
  int64_t q;
  if (levels < 0 || levels > 20) return 0;
  q = (int64_t)1 << levels;
  return Np >= N && Pp >= P && Mp >= M && Np % q == 0 && Pp % q == 0 && Mp % q == 0;
}

int or_strassen(int variant, int base, const double* A, const double* B, double* C,
                int64_t N, int64_t P, int64_t M, int32_t levels, int64_t Np, int64_t Pp, int64_t Mp) {
  double *At, *Bt, *Ct;
  int64_t i, j;
  if (bad_dims(A, B, C, N, P, M) || !strassen_plan_ok(N, P, M, levels, Np, Pp, Mp)) return -1;
  if (variant != OR_STRASSEN_NAIV && variant != OR_STRASSEN_WINOGRAD) return -1;
  g_base_products = 0;
  g_block_ops = 0;
  /* embed A, B into zero matrices */
  At = (double*)calloc((size_t)(Np * Pp), sizeof(double));
  Bt = (double*)calloc((size_t)(Pp * Mp), sizeof(double));
  Ct = (double*)calloc((size_t)(Np * Mp), sizeof(double));
  if (!At || !Bt || !Ct) { free(At); free(Bt); free(Ct); return -2; }
  for (i = 0; i < N; i++)
    for (j = 0; j < P; j++) At[IDX(i, j, Pp)] = A[IDX(i, j, P)];
  for (i = 0; i < P; i++)
    for (j = 0; j < M; j++) Bt[IDX(i, j, Mp)] = B[IDX(i, j, M)];
  strassen_rec(variant, base, At, Pp, Bt, Mp, Ct, Mp, Np, Pp, Mp, levels);
  /* extract the N x M block */
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) C[IDX(i, j, M)] = Ct[IDX(i, j, Mp)];
  free(At); free(Bt); free(Ct);
  return 0;
}

/* ------------------------------------------------------------------ exact integers */
int or_int64_gemm(const int64_t* A, const int64_t* B, int64_t* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, j, k;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) {
      int64_t s = 0;
      for (k = 0; k < P; k++) s += A[IDX(i, k, P)] * B[IDX(k, j, M)];
      C[IDX(i, j, M)] = s;
    }
  return 0;
}

/* ------------------------------------------------------------------ NEXT-3: fused variants
 * Not methods of the paper (its C99 rounds every product separately): SURVEY.md 8(f)
 * NEXT-3 variants in which every "s + x*y" of a method is contracted into ONE C99 fma(x, y, s)
 * (reading R22 in DESIGN.md); every other operation, and every order, is the method's own. */

/* NaivKahan with x_k = A_ik B_kj folded into the first update: err = fma(A_ik, B_kj, err) */
static double entry_kahan_fused(const double* A, const double* B, int64_t P, int64_t M, int64_t i, int64_t j) {
  double t, sum = 0.0, err = 0.0;
  int64_t k;
  for (k = 0; k < P; k++) {
    err = fma(A[IDX(i, k, P)], B[IDX(k, j, M)], err);
    t = sum + err;
    err = (sum - t) + err;
    sum = t;
  }
  return sum;
}

/* P:189 y_i, z_k with y = fma(A[i][2j], A[i][2j+1], y), z = fma(B[2j][k], B[2j+1][k], z) */
static double winograd_y_fused(const double* A, int64_t P, int64_t i) {
  double y = 0.0;
  int64_t j, gamma = P / 2;
  for (j = 0; j < gamma; j++) y = fma(A[IDX(i, 2 * j, P)], A[IDX(i, 2 * j + 1, P)], y);
  return y;
}

static double winograd_z_fused(const double* B, int64_t P, int64_t M, int64_t k) {
  double z = 0.0;
  int64_t j, gamma = P / 2;
  for (j = 0; j < gamma; j++) z = fma(B[IDX(2 * j, k, M)], B[IDX(2 * j + 1, k, M)], z);
  return z;
}

/* P:189-192 with acc = fma(A[i][2j] + B[2j+1][k], A[i][2j+1] + B[2j][k], acc) and the odd-P
 * term c = fma(A[i][P-1], B[P-1][k], c); (acc - y_i) - z_k unchanged */
static double winograd_entry_yz_fused(const double* A, const double* B, int64_t P, int64_t M, int64_t i, int64_t k,
                                      double yi, double zk) {
  double acc = 0.0, c;
  int64_t j, gamma = P / 2;
  for (j = 0; j < gamma; j++)
    acc = fma(A[IDX(i, 2 * j, P)] + B[IDX(2 * j + 1, k, M)], A[IDX(i, 2 * j + 1, P)] + B[IDX(2 * j, k, M)], acc);
  c = (acc - yi) - zk;
  if (P % 2 == 1) c = fma(A[IDX(i, P - 1, P)], B[IDX(P - 1, k, M)], c);
  return c;
}

int or_winograd_yz_fused(const double* A, const double* B, double* y, double* z, int64_t N, int64_t P, int64_t M) {
  int64_t i, k;
  if (bad_dims(A, B, y, N, P, M) || z == NULL) return -1;
  for (i = 0; i < N; i++) y[i] = winograd_y_fused(A, P, i);
  for (k = 0; k < M; k++) z[k] = winograd_z_fused(B, P, M, k);
  return 0;
}

int or_naive_kahan_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, j;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  for (i = 0; i < N; i++)
    for (j = 0; j < M; j++) C[IDX(i, j, M)] = entry_kahan_fused(A, B, P, M, i, j);
  return 0;
}

int or_winograd_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M) {
  int64_t i, k;
  double *y, *z;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  y = (double*)malloc(sizeof(double) * (size_t)N);
  z = (double*)malloc(sizeof(double) * (size_t)M);
  if (!y || !z) { free(y); free(z); return -2; }
  for (i = 0; i < N; i++) y[i] = winograd_y_fused(A, P, i);
  for (k = 0; k < M; k++) z[k] = winograd_z_fused(B, P, M, k);
  for (i = 0; i < N; i++)
    for (k = 0; k < M; k++) C[IDX(i, k, M)] = winograd_entry_yz_fused(A, B, P, M, i, k, y[i], z[k]);
  free(y);
  free(z);
  return 0;
}

/* WinogradScaled with the fused WinogradOriginal: same lambda, same exact copies */
int or_winograd_scaled_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                             int32_t* lambda_out) {
  double nA, nB, *As, *Bs;
  int lambda, rc;
  if (bad_dims(A, B, C, N, P, M)) return -1;
  nA = or_norm_inf(A, N, P);
  nB = or_norm_inf(B, P, M);
  lambda = or_lambda(nA, nB);
  As = (double*)malloc(sizeof(double) * (size_t)(N * P));
  Bs = (double*)malloc(sizeof(double) * (size_t)(P * M));
  if (!As || !Bs) { free(As); free(Bs); return -2; }
  or_scalar_mul(ldexp(1.0, lambda), A, As, N, P);
  or_scalar_mul(ldexp(1.0, -lambda), B, Bs, P, M);
  rc = or_winograd_fused(As, Bs, C, N, P, M);
  free(As);
  free(Bs);
  if (lambda_out) *lambda_out = lambda;
  return rc;
}

/* ------------------------------------------------------------------ per entry */
double or_entry(int method, const double* A, const double* B, int64_t N, int64_t P, int64_t M,
                int64_t i, int64_t j, int32_t lambda) {
  (void)N;
  switch (method) {
    case OR_M_STANDARD: return entry_standard(A, B, P, M, i, j);
    case OR_M_ON_ARRAY: {
      double c = 0.0;
      int64_t k;
      for (k = 0; k < P; k++) c = c + A[IDX(i, k, P)] * B[IDX(k, j, M)];
      return c;
    }
    case OR_M_KAHAN: return entry_kahan(A, B, P, M, i, j);
    case OR_M_UNROLL2: return entry_unroll(2, A, B, P, M, i, j);
    case OR_M_UNROLL3: return entry_unroll(3, A, B, P, M, i, j);
    case OR_M_UNROLL4: return entry_unroll(4, A, B, P, M, i, j);
    case OR_M_FMA: return entry_fma(A, B, P, M, i, j);
    case OR_M_WINOGRAD: return winograd_entry_yz(A, B, P, M, i, j, winograd_y(A, P, i), winograd_z(B, P, M, j));
    case OR_M_KAHAN_FUSED: return entry_kahan_fused(A, B, P, M, i, j);
    case OR_M_WINOGRAD_FUSED:
      return winograd_entry_yz_fused(A, B, P, M, i, j, winograd_y_fused(A, P, i), winograd_z_fused(B, P, M, j));
    case OR_M_WINOGRAD_SCALED_FUSED: {
      /* row i of 2^lambda A and column j of 2^-lambda B (exact copies, N = 1 and M = 1 views) */
      double sa = ldexp(1.0, lambda), sb = ldexp(1.0, -lambda), c;
      int64_t q;
      double* a = dalloc(P);
      double* b = dalloc(P);
      for (q = 0; q < P; q++) { a[q] = sa * A[IDX(i, q, P)]; b[q] = sb * B[IDX(q, j, M)]; }
      c = winograd_entry_yz_fused(a, b, P, 1, 0, 0, winograd_y_fused(a, P, 0), winograd_z_fused(b, P, 1, 0));
      free(a);
      free(b);
      return c;
    }
    case OR_M_WINOGRAD_SCALED: {
      /* the row i of 2^lambda A and the column j of 2^-lambda B, then WinogradOriginal's entry */
      double sa = ldexp(1.0, lambda), sb = ldexp(1.0, -lambda), y = 0.0, z = 0.0, acc = 0.0, c;
      int64_t q, gamma = P / 2;
      double* a = dalloc(P);
      double* b = dalloc(P);
      for (q = 0; q < P; q++) { a[q] = sa * A[IDX(i, q, P)]; b[q] = sb * B[IDX(q, j, M)]; }
      for (q = 0; q < gamma; q++) y = y + a[2 * q] * a[2 * q + 1];
      for (q = 0; q < gamma; q++) z = z + b[2 * q] * b[2 * q + 1];
      for (q = 0; q < gamma; q++) acc = acc + (a[2 * q] + b[2 * q + 1]) * (a[2 * q + 1] + b[2 * q]);
      c = (acc - y) - z;
      if (P % 2 == 1) c = c + a[P - 1] * b[P - 1];
      free(a);
      free(b);
      return c;
    }
    default: return NAN;
  }
}

/* Lazy Strassen entry.
 * rows: 2^h rows of the node's left operand X (n x p), row a = node row (i0 + a n/2^h), dense, length p.
 * cols: 2^h columns of the node's right operand Y (p x m), col b = node column (j0 + b m/2^h), length p.
 * Returns entry (i0 + as n/2^h, j0 + bs m/2^h) of X Y computed exactly as strassen_rec computes it. */
static double lz_dot(int base, const double* x, const double* y, int64_t p) {
  double aux = 0.0;
  int64_t k;
  if (base == OR_BASE_FMA)
    for (k = 0; k < p; k++) aux = fma(x[k], y[k], aux);
  else
    for (k = 0; k < p; k++) aux = aux + x[k] * y[k];
  return aux;
}

/* Z[a][k] = X[a][k] op Y[a][k] over `cnt` vectors of length p2, with per-operand row strides */
static void lz_op(double* Z, const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t cnt, int64_t p2,
                  int sub) {
  int64_t a, k;
  for (a = 0; a < cnt; a++)
    for (k = 0; k < p2; k++)
      Z[a * p2 + k] = sub ? X[a * ldx + k] - Y[a * ldy + k] : X[a * ldx + k] + Y[a * ldy + k];
}
static void lz_copy(double* Z, const double* X, int64_t ldx, int64_t cnt, int64_t p2) {
  int64_t a, k;
  for (a = 0; a < cnt; a++)
    for (k = 0; k < p2; k++) Z[a * p2 + k] = X[a * ldx + k];
}

static double lz_rec(int variant, int base, const double* rows, const double* cols, int32_t h, int64_t p,
                     int64_t as, int64_t bs);

/* the H_t entry: product of child operands given as vector sets (each cnt x p2, dense) */
static double lz_child(int variant, int base, const double* S, const double* T, int32_t h, int64_t p2, int64_t a,
                       int64_t b) {
  return lz_rec(variant, base, S, T, h - 1, p2, a, b);
}

static double lz_rec(int variant, int base, const double* rows, const double* cols, int32_t h, int64_t p,
                     int64_t as, int64_t bs) {
  int64_t half, p2, a, b, cnt;
  int qi, qj;
  /* quadrant vector sets (row stride p inside `rows`/`cols`) */
  const double *X11, *X12, *X21, *X22, *Y11, *Y12, *Y21, *Y22;
  double *S, *T, *U, *V;
  double H[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  double r;
  if (h == 0) return lz_dot(base, rows, cols, p);
  half = (int64_t)1 << (h - 1);
  cnt = half;
  p2 = p / 2;
  qi = as >= half; qj = bs >= half;
  a = as - qi * half; b = bs - qj * half;
  X11 = rows; X12 = rows + p2; X21 = rows + half * p; X22 = X21 + p2;
  /* column b of Y11 = top half of cols[b]; Y21 = bottom half of cols[b];
   * Y12 = top half of cols[b + half]; Y22 = bottom half of cols[b + half] */
  Y11 = cols; Y21 = cols + p2; Y12 = cols + half * p; Y22 = Y12 + p2;
  S = dalloc(cnt * p2); T = dalloc(cnt * p2); U = dalloc(cnt * p2); V = dalloc(cnt * p2);
  if (variant == OR_STRASSEN_NAIV) {
    int need[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (!qi && !qj) { need[1] = need[4] = need[5] = need[7] = 1; }
    if (!qi && qj) { need[3] = need[5] = 1; }
    if (qi && !qj) { need[2] = need[4] = 1; }
    if (qi && qj) { need[1] = need[3] = need[2] = need[6] = 1; }
    if (need[1]) { lz_op(S, X11, p, X22, p, cnt, p2, 0); lz_op(T, Y11, p, Y22, p, cnt, p2, 0);
                   H[1] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[2]) { lz_op(S, X21, p, X22, p, cnt, p2, 0); lz_copy(T, Y11, p, cnt, p2);
                   H[2] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[3]) { lz_copy(S, X11, p, cnt, p2); lz_op(T, Y12, p, Y22, p, cnt, p2, 1);
                   H[3] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[4]) { lz_copy(S, X22, p, cnt, p2); lz_op(T, Y21, p, Y11, p, cnt, p2, 1);
                   H[4] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[5]) { lz_op(S, X11, p, X12, p, cnt, p2, 0); lz_copy(T, Y22, p, cnt, p2);
                   H[5] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[6]) { lz_op(S, X21, p, X11, p, cnt, p2, 1); lz_op(T, Y11, p, Y12, p, cnt, p2, 0);
                   H[6] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[7]) { lz_op(S, X12, p, X22, p, cnt, p2, 1); lz_op(T, Y21, p, Y22, p, cnt, p2, 0);
                   H[7] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (!qi && !qj) r = ((H[1] + H[4]) - H[5]) + H[7];
    else if (!qi && qj) r = H[3] + H[5];
    else if (qi && !qj) r = H[2] + H[4];
    else r = ((H[1] + H[3]) - H[2]) + H[6];
  } else {
    /* A1 = A11 - A21 (U), A2 = A22 - A1 (S_A2), B1 = B22 - B12 (V), B2 = B1 + B11 */
    double *A2 = dalloc(cnt * p2), *B2 = dalloc(cnt * p2);
    int need[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    lz_op(U, X11, p, X21, p, cnt, p2, 1);  /* A1 */
    lz_op(A2, X22, p, U, p2, cnt, p2, 1);  /* A2 */
    lz_op(V, Y22, p, Y12, p, cnt, p2, 1);  /* B1 */
    lz_op(B2, V, p2, Y11, p, cnt, p2, 0);  /* B2 */
    if (!qi && !qj) { need[1] = need[2] = 1; }
    if (!qi && qj) { need[1] = need[3] = need[4] = need[6] = 1; }
    if (qi && !qj) { need[1] = need[3] = need[5] = need[7] = 1; }
    if (qi && qj) { need[1] = need[3] = need[4] = need[5] = 1; }
    if (need[1]) { lz_copy(S, X11, p, cnt, p2); lz_copy(T, Y11, p, cnt, p2);
                   H[1] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[2]) { lz_copy(S, X12, p, cnt, p2); lz_copy(T, Y21, p, cnt, p2);
                   H[2] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[3]) { H[3] = lz_child(variant, base, A2, B2, h, p2, a, b); }
    if (need[4]) { lz_op(S, X21, p, X22, p, cnt, p2, 0); lz_op(T, Y12, p, Y11, p, cnt, p2, 1);
                   H[4] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[5]) { H[5] = lz_child(variant, base, U, V, h, p2, a, b); }
    if (need[6]) { lz_op(S, X12, p, A2, p2, cnt, p2, 1); lz_copy(T, Y22, p, cnt, p2);
                   H[6] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (need[7]) { lz_copy(S, X22, p, cnt, p2); lz_op(T, Y21, p, B2, p2, cnt, p2, 1);
                   H[7] = lz_child(variant, base, S, T, h, p2, a, b); }
    if (!qi && !qj) r = H[1] + H[2];
    else if (!qi && qj) { double h8 = H[1] + H[3]; double h9 = h8 + H[4]; r = h9 + H[6]; }
    else if (qi && !qj) { double h8 = H[1] + H[3]; r = (h8 + H[5]) + H[7]; }
    else { double h8 = H[1] + H[3]; double h9 = h8 + H[4]; r = h9 + H[5]; }
    free(A2); free(B2);
  }
  free(S); free(T); free(U); free(V);
  return r;
}

double or_entry_strassen(int variant, int base, const double* A, const double* B,
                         int64_t N, int64_t P, int64_t M, int32_t levels,
                         int64_t Np, int64_t Pp, int64_t Mp, int64_t i, int64_t j) {
  int64_t R, nb, mb, i0, j0, a, k;
  double *rows, *cols, r;
  if (!strassen_plan_ok(N, P, M, levels, Np, Pp, Mp) || i < 0 || j < 0 || i >= N || j >= M) return NAN;
  R = (int64_t)1 << levels;
  nb = Np / R; mb = Mp / R;
  i0 = i % nb; j0 = j % mb;
  rows = (double*)calloc((size_t)(R * Pp), sizeof(double));
  cols = (double*)calloc((size_t)(R * Pp), sizeof(double));
  /* embedded (zero padded) rows i0 + a nb of A~ and columns j0 + a mb of B~ */
  for (a = 0; a < R; a++) {
    int64_t ri = i0 + a * nb, cj = j0 + a * mb;
    for (k = 0; k < Pp; k++) {
      rows[a * Pp + k] = (ri < N && k < P) ? A[IDX(ri, k, P)] : 0.0;
      cols[a * Pp + k] = (cj < M && k < P) ? B[IDX(k, cj, M)] : 0.0;
    }
  }
  r = lz_rec(variant, base, rows, cols, levels, Pp, i / nb, j / mb);
  free(rows);
  free(cols);
  return r;
}

/* ------------------------------------------------------------------ batched per-entry calls */
void or_entries(int method, const double* A, const double* B, int64_t N, int64_t P, int64_t M,
                const int64_t* ij, int64_t count, int32_t lambda, double* out) {
  int64_t q;
  for (q = 0; q < count; q++) out[q] = or_entry(method, A, B, N, P, M, ij[2 * q], ij[2 * q + 1], lambda);
}

void or_entries_strassen(int variant, int base, const double* A, const double* B, int64_t N, int64_t P,
                         int64_t M, int32_t levels, int64_t Np, int64_t Pp, int64_t Mp, const int64_t* ij,
                         int64_t count, double* out) {
  int64_t q;
  for (q = 0; q < count; q++)
    out[q] = or_entry_strassen(variant, base, A, B, N, P, M, levels, Np, Pp, Mp, ij[2 * q], ij[2 * q + 1]);
}
