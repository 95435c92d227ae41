/*
 * oracle.h -- CPU oracle for Hedtke, "Methods of Matrix Multiplication" (arXiv 1106.1347).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1106_1347_b200/, include/, csrc/) never includes, links or calls it, and
 * this file includes nothing from there.
 *
 * Plain, slow, obviously-correct C99 written from the paper's text.  Citations are
 * "P:L" = /root/reference/PAPER.md line L (section / equation in brackets).
 *
 * Conventions:
 *  - 0-based indices, dense row-major storage: X[i][j] = X[i*cols + j].
 *  - A is N x P, B is P x M, C is N x M ("A denotes a N x P matrix and B
 *    denotes a P x M matrix with entries of type double").
 *  - Every loop runs in increasing index order; every "x + y*z" is a separately
 *    rounded product followed by a separately rounded sum (built with
 *    -ffp-contract=off), the only reading consistent with an unoptimised C99
 *    build.  The one exception is or_naive_fma / base==OR_BASE_FMA,
 *    which call C99 fma() explicitly (reading R2 in DESIGN.md).
 *  - Functions returning int return 0 on success and a negative value on bad
 *    arguments (NULL pointers, non-positive sizes, malformed plans).
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py except
 * where its comment says "parity unpinned".
 */
#ifndef MM_ORACLE_H
#define MM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- load-time self checks: IEEE binary64, no contraction, Kahan pin. 0 = ok ---- */
int or_selfcheck(void);

/* ---- Section 1: auxiliary routines ---- */
/* P:28-33 (Plus):  Z_ij = X_ij + Y_ij */
void or_plus(const double* X, const double* Y, double* Z, int64_t r, int64_t c);
/* P:35-39 (Minus): Z_ij = X_ij - Y_ij */
void or_minus(const double* X, const double* Y, double* Z, int64_t r, int64_t c);
/* P:41-49 (max): x if x >= y else y */
double or_max_d(double x, double y);
int64_t or_max_i(int64_t x, int64_t y);
/* P:51-56 (NormInf): max_i sum_j |X_ij|, sums left to right */
double or_norm_inf(const double* X, int64_t r, int64_t c);
/* P:58-62 (MultiplyWithScalar): Z_ij = alpha * X_ij */
void or_scalar_mul(double alpha, const double* X, double* Z, int64_t r, int64_t c);

/* ---- Section 2.1 / 2.2: naive family ---- */
/* P:102-106 (NaivStandard): aux = 0; aux = aux + A_ik*B_kj; C_ij = aux */
int or_naive_standard(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);
/* P:108-109 (NaivOnArray): accumulate directly into C_ij */
int or_naive_on_array(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);
/* P:111-134 (NaivKahan): compensated sum of the products, update of P:122-132 */
int or_naive_kahan(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);
/* P:136-168 (NaivLoopUnrolling{Two,Three,Four}), u in {2,3,4}: groups of u
 * products summed left to right, added to aux; the P mod u tail terms appended
 * in increasing k (P:146-150, P:156 with the 2k->3k typo read as 3k). */
int or_naive_unroll(int u, const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);
/* Reading R2: NaivStandard with the multiply-add contracted, aux = fma(A_ik, B_kj, aux),
 * k increasing.  This is what one FP64 tensor-core DMMA chain computes (probe P3). */
int or_naive_fma(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);

/* Reading R2 continued: C = A B + C where every entry's fma chain starts
 * from C's current value; A N x K (pitch lda), B K x M (pitch ldb), C N x M (pitch ldc). */
int or_naive_fma_acc(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                     int64_t N, int64_t K, int64_t M);

/* NEXT-4: NaivKahan's update (fused != 0: err = fma(a, b, err)) resumed from the state
 * (S = sum, E = err, both N x M dense) over a strided k-panel; writes the state back. */
int or_naive_kahan_acc(const double* A, int64_t lda, const double* B, int64_t ldb, double* S, double* E,
                       int64_t N, int64_t K, int64_t M, int fused);

/* ---- Section 2.3: Winograd ---- */
/* gamma = floor(P/2); y_i = sum_{j<gamma} A[i][2j]*A[i][2j+1];
 * z_k = sum_{j<gamma} B[2j][k]*B[2j+1][k]  (0-based form of A_{i,2j-1}A_{i,2j}) */
int or_winograd_yz(const double* A, const double* B, double* y, double* z, int64_t N, int64_t P, int64_t M);
/* P:187-195 (WinogradOriginal): C_ik = (acc - y_i) - z_k  [+ A[i][P-1]*B[P-1][k] if P odd],
 * acc = sum_{j<gamma} (A[i][2j] + B[2j+1][k]) * (A[i][2j+1] + B[2j][k]) */
int or_winograd_original(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);
/* NEXT-4: WinogradOriginal's pair sum resumed from Acc (N x M) over the K/2 pairs of a
 * strided k-panel (K even); fused != 0: acc = fma(u, v, acc).  or_winograd_finish: the even-P
 * epilogue C = (acc - y_i) - z_k. */
int or_winograd_pairs_acc(const double* A, int64_t lda, const double* B, int64_t ldb, double* Acc, int64_t N,
                          int64_t K, int64_t M, int fused);
int or_winograd_finish(const double* Acc, const double* y, const double* z, double* C, int64_t N, int64_t M);
/* the integer lambda with 1/2 <= 2^lambda nA / (2^-lambda nB) <= 2,
 * exact (frexp); ties (both lambdas valid) -> the larger |lambda|; nA or nB == 0 -> 0. */
int or_lambda(double nA, double nB);
/* P:197-217 (WinogradScaled): lambda from the two norms, WinogradOriginal on
 * (2^lambda A, 2^-lambda B); C not rescaled.  Writes lambda to *lambda_out. */
int or_winograd_scaled(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                       int32_t* lambda_out);

/* ---- fused-multiply-add variants (reading R22; NOT the paper's methods,
 * whose C99 rounds every product separately).  Every "s + x*y" of the method becomes one C99
 * fma(x, y, s); all other operations and all orders are the method's own. ---- */
/* NaivKahan with err = fma(A_ik, B_kj, err) */
int or_naive_kahan_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);
/* y, z of P:189 accumulated by fma (the y/z of or_winograd_fused) */
int or_winograd_yz_fused(const double* A, const double* B, double* y, double* z, int64_t N, int64_t P, int64_t M);
/* WinogradOriginal with y, z, acc and the odd-P term accumulated by fma */
int or_winograd_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M);
/* WinogradScaled on top of or_winograd_fused */
int or_winograd_scaled_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                             int32_t* lambda_out);

/* ---- Section 2.4: Strassen ---- */
#define OR_STRASSEN_NAIV 0     /* P:251-291, 18 block additions per level */
#define OR_STRASSEN_WINOGRAD 1 /* P:294-315, 15 block additions per level */
#define OR_BASE_LITERAL 0      /* alpha_{m,0} = NaivStandard */
#define OR_BASE_FMA 1          /* alpha_{m,0} = or_naive_fma (reading R2) */
/* X = max{N,P,M}; k = floor(log2 X) - 4 (clamped to >= 0, reading R8);
 * m = floor(X 2^-k) + 1; Y = m 2^k. */
void or_strassen_plan_paper(int64_t N, int64_t P, int64_t M, int32_t* k, int64_t* m, int64_t* Y);
/* Levels plan (reading R10): each dim padded to the next multiple of align*2^levels. */
void or_strassen_plan_levels(int64_t N, int64_t P, int64_t M, int32_t levels, int64_t align,
                             int64_t* Np, int64_t* Pp, int64_t* Mp);
/* Embed A, B with zeros into Np x Pp and Pp x Mp, recurse `levels` times
 * (P:254-284 or P:299-312), base alpha_{m,0} per `base`, extract the N x M block.
 * Np, Pp, Mp must be >= N, P, M and divisible by 2^levels. */
int or_strassen(int variant, int base, const double* A, const double* B, double* C,
                int64_t N, int64_t P, int64_t M, int32_t levels, int64_t Np, int64_t Pp, int64_t Mp);
/* counters of the last or_strassen call: base products and block add/sub ops */
void or_strassen_counters(int64_t* base_products, int64_t* block_ops);
/* record the value of every 1 x 1 base product (in call order) into buf; NULL stops */
void or_strassen_trace(double* buf, int64_t cap);
int64_t or_strassen_trace_len(void);

/* ---- exact integer product: an independent arithmetic domain ---- */
int or_int64_gemm(const int64_t* A, const int64_t* B, int64_t* C, int64_t N, int64_t P, int64_t M);

/* ---- per-entry replicas (bit-identical to the full functions) for sampled checks ---- */
#define OR_M_STANDARD 0
#define OR_M_ON_ARRAY 1
#define OR_M_KAHAN 2
#define OR_M_UNROLL2 3
#define OR_M_UNROLL3 4
#define OR_M_UNROLL4 5
#define OR_M_FMA 6
#define OR_M_WINOGRAD 7
#define OR_M_WINOGRAD_SCALED 8 /* uses the lambda argument (global norms needed) */
#define OR_M_KAHAN_FUSED 9
#define OR_M_WINOGRAD_FUSED 10
#define OR_M_WINOGRAD_SCALED_FUSED 11 /* uses the lambda argument */
double or_entry(int method, const double* A, const double* B, int64_t N, int64_t P, int64_t M,
                int64_t i, int64_t j, int32_t lambda);
/* Entry (i,j) of or_strassen(...) computed lazily: only the 2^levels rows of A and
 * columns of B congruent to (i, j) are materialised.  Bit-identical to or_strassen. */
double or_entry_strassen(int variant, int base, const double* A, const double* B,
                         int64_t N, int64_t P, int64_t M, int32_t levels,
                         int64_t Np, int64_t Pp, int64_t Mp, int64_t i, int64_t j);

/* the same, over `count` (i, j) pairs stored as ij[2q], ij[2q+1] */
void or_entries(int method, const double* A, const double* B, int64_t N, int64_t P, int64_t M,
                const int64_t* ij, int64_t count, int32_t lambda, double* out);
void or_entries_strassen(int variant, int base, const double* A, const double* B, int64_t N, int64_t P,
                         int64_t M, int32_t levels, int64_t Np, int64_t Pp, int64_t Mp, const int64_t* ij,
                         int64_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif
