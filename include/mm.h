/*
 * mm.h -- C ABI of the B200 (sm_100a) FP64 matrix-multiplication library implementing the
 * methods of Hedtke, "Methods of Matrix Multiplication" (arXiv 1106.1347).
 *
 * Citations "P:L" refer to /root/reference/PAPER.md line L.
 *
 * Problem statement: "A denotes a N x P matrix and B denotes a P x M matrix with
 * entries of type double".  Every entry point below computes C = A B, C being N x M.
 *
 * Conventions shared by every function:
 *  - Layout: A, B, C are DENSE ROW-MAJOR float64 buffers with leading dimensions P, M and M
 *    (A[i][k] = A[i*P + k]).  All pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *    tensors) on the current CUDA device unless a parameter says "host".
 *  - Ownership: the caller owns A, B, C and the workspace; the library never allocates or
 *    frees on these paths and keeps no reference after the call returns.  The library's
 *    only persistent state is per-process kernel attributes.
 *  - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    stream-ordered and return after enqueue (asynchronous), except where a host output
 *    pointer is given (documented per function), which synchronises the stream.
 *  - Errors: return MM_OK (0) or a negative mm_status.  MM_ERR_ARG: NULL pointer,
 *    N, P or M < 1, or an element count overflowing int64.  MM_ERR_ALIAS: C overlaps A or B.
 *    MM_ERR_WORKSPACE: ws_bytes < mm_workspace_size(...).  MM_ERR_UNSUPPORTED: the current
 *    device is not compute capability 10.0 (sm_100a) -- there is no fallback of any kind.
 *    MM_ERR_CUDA: a launch or CUDA runtime call failed (device faults surface at the
 *    caller's next synchronisation).  MM_ERR_NCCL: the multi-GPU layer could not load NCCL or a
 *    collective failed.  On error nothing is enqueued unless MM_ERR_CUDA / MM_ERR_NCCL.
 *  - Arithmetic is IEEE binary64 round-to-nearest-even throughout; DESIGN.md lists, per
 *    method, which oracle function each kernel reproduces bit for bit.  The paper defines the
 *    methods on finite inputs only; with NaN/Inf operands the IEEE propagation of each operation
 *    applies (norm_inf then returns a NaN if any row sum is NaN), and no result is guaranteed.
 */
#ifndef MM_B200_H
#define MM_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MM_OK = 0,
  MM_ERR_ARG = -1,
  MM_ERR_ALIAS = -2,
  MM_ERR_WORKSPACE = -3,
  MM_ERR_CUDA = -4,
  MM_ERR_NCCL = -5,
  MM_ERR_UNSUPPORTED = -6
} mm_status;

/* method ids for mm_workspace_size / mm_gemm */
typedef enum {
  MM_NAIVE = 0,            /* P:102-106 NaivStandard (also NaivOnArray, unrolled variants) */
  MM_KAHAN = 1,            /* P:111-134 NaivKahan */
  MM_WINOGRAD = 2,         /* P:186-195 WinogradOriginal */
  MM_WINOGRAD_SCALED = 3,  /* P:197-217 WinogradScaled */
  MM_STRASSEN = 4,         /* P:251-291 StrassenNaiv */
  MM_STRASSEN_WINOGRAD = 5, /* P:294-315 StrassenWinograd */
  /* SURVEY.md 8(f) NEXT-3 fused variants (reading R22) -- not the paper's methods */
  MM_KAHAN_FUSED = 6,
  MM_WINOGRAD_FUSED = 7,
  MM_WINOGRAD_SCALED_FUSED = 8
} mm_method;

/* Library version string and a human-readable message for a status code. */
const char* mm_version(void);
const char* mm_status_string(int status);

/*
 * mm_naive -- (AB)_ij = sum_k A_ik B_kj (NaivStandard P:105-106).
 * FP64 tensor-core (DMMA) GEMM; k is walked in increasing order as one fused
 * multiply-add chain per entry (reading R2).  No workspace.
 */
int mm_naive(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* stream);

/*
 * mm_naive_ex -- the mm_naive kernel on strided operands, optionally accumulating:
 *   C = A B          (accumulate == 0)
 *   C = A B + C      (accumulate != 0)   with A N x K (row pitch lda >= K), B K x M (ldb >= M),
 *                                        C N x M (ldc >= M), all device pointers.
 * With accumulate the fma chain of every entry STARTS from C's current value and continues over
 * k = 0..K-1 in order (reading R2), so splitting P into consecutive column panels of A /
 * row panels of B, in increasing k, reproduces mm_naive bit for bit (up to the sign of zero):
 *   mm_naive_ex(A, P, B, M, C, M, N, k1, M, 0); mm_naive_ex(A + k1, P, B + k1*M, M, C, M, N, P-k1, M, 1)
 * -- the building block of the multi-GPU broadcast/compute overlap.
 * Errors as mm_naive (MM_ERR_ARG also for a pitch smaller than its row); no workspace.
 */
int mm_naive_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int64_t N,
                int64_t K, int64_t M, int32_t accumulate, void* stream);

/*
 * k-panel steps of NaivKahan and WinogradOriginal (B broadcast in row panels
 * overlapped with the products; mm_dist_gemm uses them).  A is N x K with row pitch lda >= K, B is
 * K x M with pitch ldb >= M (panel views of wider operands), C (and E) dense N x M.  Flags:
 *   MM_EX_ACCUMULATE  each entry's running state starts from the previous panel's (C, and E for
 *                     Kahan) instead of +0, and continues over k = 0..K-1 in order;
 *   MM_EX_KEEP_STATE  the running state is stored for a later panel: Kahan writes `sum` into C and
 *                     `err` into E; Winograd writes the raw pair sum into C (no epilogue);
 *   MM_EX_FUSED       the NEXT-3 variant (reading R22).
 * Running the panels of P in increasing k -- the first without ACCUMULATE, all but the last with
 * KEEP_STATE -- performs every entry's operations in exactly the one-shot order, so the result is
 * bit for bit mm_kahan / mm_winograd (or the fused variants).  Requirements (else MM_ERR_ARG):
 * A and B 16-byte aligned, lda, ldb and M even (the TMA-fed kernels), and for Winograd K even
 * (whole pairs per panel) and y, z (mm_winograd_yz of the FULL operands) unless KEEP_STATE.
 * No workspace; E is caller-owned (N x M doubles) and required with ACCUMULATE or KEEP_STATE.
 */
#define MM_EX_ACCUMULATE 1
#define MM_EX_KEEP_STATE 2
#define MM_EX_FUSED 4
int mm_kahan_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, double* E, int64_t N,
                int64_t K, int64_t M, int32_t flags, void* stream);
int mm_winograd_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, const double* y,
                   const double* z, int64_t N, int64_t K, int64_t M, int32_t flags, void* stream);
/* y_i and z_k of P:189 (sums in increasing j; fma when flags & MM_EX_FUSED) of dense A (N x P) and
 * B (P x M) into device vectors y (N) and z (M).  MM_ERR_ALIAS if y or z overlaps A, B or each
 * other (mm_winograd_ex likewise if C overlaps y or z). */
int mm_winograd_yz(const double* A, const double* B, int64_t N, int64_t P, int64_t M, double* y, double* z,
                   int32_t flags, void* stream);

/*
 * mm_kahan -- NaivKahan: each entry is the compensated sum of the products
 * A_ik B_kj, k increasing, with the update of P:122-132
 * (err = err + x; t = sum + err; err = (sum - t) + err; sum = t), result `sum`.
 * Separately rounded FP64 operations, no contraction.  No workspace.
 */
int mm_kahan(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* stream);

/*
 * mm_winograd -- WinogradOriginal: y_i = sum_j A_{i,2j-1}A_{i,2j},
 * z_k = sum_j B_{2j-1,k}B_{2j,k}, C_ik = (sum_j (A_{i,2j-1}+B_{2j,k})(A_{i,2j}+B_{2j-1,k}) - y_i) - z_k,
 * plus A_{i,P}B_{P,k} when P is odd.  Sums in increasing j, separately rounded.
 * workspace: device buffer of at least mm_workspace_size(MM_WINOGRAD, N, P, M, 0) bytes
 * (holds y and z), 256-byte aligned.
 */
int mm_winograd(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                void* workspace, size_t ws_bytes, void* stream);

/*
 * mm_winograd_scaled -- WinogradScaled: lambda is the integer with
 * 1/2 <= 2^lambda ||A||_inf / (2^-lambda ||B||_inf) <= 2 (tie -> larger |lambda|,
 * zero norm -> 0), then WinogradOriginal on (2^lambda A, 2^-lambda B); C is not rescaled
 * (P:216).  Norms and lambda are computed on the device (no host sync).
 * workspace: >= mm_workspace_size(MM_WINOGRAD_SCALED, N, P, M, 0) bytes.
 * lambda_out: HOST int32 pointer or NULL; when non-NULL the call synchronises `stream`
 * and stores lambda there.
 */
int mm_winograd_scaled(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                       void* workspace, size_t ws_bytes, int32_t* lambda_out, void* stream);

/*
 * mm_strassen / mm_strassen_winograd -- StrassenNaiv (H_1..H_7 of P:271-277,
 * C blocks of P:279-282) and StrassenWinograd.  `levels` >= 0 recursion levels
 * with each dimension zero-padded to the next multiple of 2^(levels+1) (DESIGN.md reading
 * R10; mm_strassen_plan reports the padded dims); levels == -1 selects the paper's plan
 * (X = max{N,P,M}, k = floor(log2 X) - 4 clamped at 0, m = floor(X 2^-k) + 1,
 * embed in Y x Y with Y = m 2^k, k levels).  The base case alpha_{m,0} is the DMMA GEMM of
 * mm_naive, batched over all 7^levels products.  levels in [-1, 8].
 * workspace: >= mm_workspace_size(MM_STRASSEN[_WINOGRAD], N, P, M, levels) bytes.
 */
int mm_strassen(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, int32_t levels,
                void* workspace, size_t ws_bytes, void* stream);
int mm_strassen_winograd(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                         int32_t levels, void* workspace, size_t ws_bytes, void* stream);

/*
 * mm_strassen_plan -- the recursion depth and padded dimensions mm_strassen uses for
 * (N, P, M, levels): HOST output pointers.  Returns MM_ERR_ARG on bad sizes/levels.
 */
int mm_strassen_plan(int64_t N, int64_t P, int64_t M, int32_t levels, int32_t* depth_out, int64_t* Np_out,
                     int64_t* Pp_out, int64_t* Mp_out);

/* Workspace bytes the given method needs; 0 on bad arguments.  MM_NAIVE and MM_KAHAN[_FUSED] need
 * none with even P; with odd P they report N (P + 1) doubles, which mm_gemm uses (when given) to copy
 * A to an even row pitch so the TMA-fed kernels apply (a tiled TMA box cannot start on an 8-byte
 * boundary) -- same result bit for bit; MM_WINOGRAD[_FUSED] likewise add that room to y | z. */
size_t mm_workspace_size(int method, int64_t N, int64_t P, int64_t M, int32_t levels);

/*
 * mm_gemm -- dispatch by mm_method id (levels only used by the Strassen methods,
 * lambda_out only by MM_WINOGRAD_SCALED[_FUSED]; both may be 0/NULL otherwise).
 */
int mm_gemm(int method, const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
            int32_t levels, void* workspace, size_t ws_bytes, int32_t* lambda_out, void* stream);

/*
 * mm_methods_host -- the paper's test program from HOST memory: C_host[i] = A B by
 * methods[i], i < n, all on the same operands.  A_host (N x P), B_host (P x M) and every C_host[i]
 * (N x M) are HOST pointers, row-major float64 (page-locked memory lets the copies overlap the
 * kernels; pageable memory works but the copies then serialise).  A and B are copied to the device
 * once; the methods run in turn on `stream`; each product is copied back on a library-owned copy
 * stream while the next method computes.  A first NaivStandard multiplies k-panels of A and B as
 * they land (mm_naive_ex accumulation, bitwise the one-shot product); a first row-local method
 * (NaivKahan, WinogradOriginal and their fused variants) starts on each of `row_blocks` row blocks
 * of A as it lands; a last row-local method returns its product by row blocks of halving height.
 * Every C_host[i] equals the device entry point's result bit for bit.  levels: for the Strassen
 * methods (as mm_strassen).  dev_ws: DEVICE workspace of at least
 * mm_methods_host_workspace_size(methods, n, N, P, M, levels) bytes (device copies of A and B,
 * min(n, 3) product buffers, the largest method workspace).  SYNCHRONOUS: returns once every product has
 * landed in host memory.  The library keeps two copy streams per device for these calls.
 * Errors as mm_gemm; MM_ERR_ARG for a NULL C_host[i] or an unknown method id.
 */
size_t mm_methods_host_workspace_size(const int* methods, int32_t n, int64_t N, int64_t P, int64_t M,
                                      int32_t levels);
int mm_methods_host(const int* methods, int32_t n, const double* A_host, const double* B_host, double* const* C_host,
                    int64_t N, int64_t P, int64_t M, int32_t levels, int32_t row_blocks, void* dev_ws, size_t ws_bytes,
                    void* stream);

/*
 * norm_inf -- ||X||_inf = max_i sum_j |X_ij| of a dense row-major rows x cols
 * device matrix; each row sum is accumulated left to right (as the oracle does), the max
 * is order-free.  out_device: DEVICE pointer to one double, overwritten.
 */
int norm_inf(const double* X, int64_t rows, int64_t cols, double* out_device, void* stream);

/*
 * mm_lambda -- the device-side lambda rule of mm_winograd_scaled applied to two host
 * norms (for tests of the rule itself); returns lambda.  Runs on the host, no GPU needed.
 */
int32_t mm_lambda(double nA, double nB);

/*
 * mm_winograd_scaled_norms -- mm_winograd_scaled with the two norms supplied by the caller:
 * norms_device is a DEVICE pointer to {||A||_inf, ||B||_inf} (2 doubles), e.g. the global
 * ||A||_inf of a row-sharded A after an all-reduce(max) (multi-GPU path).
 * NULL makes it identical to mm_winograd_scaled.  Same workspace and lambda_out semantics.
 */
int mm_winograd_scaled_norms(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                             const double* norms_device, void* workspace, size_t ws_bytes, int32_t* lambda_out,
                             void* stream);

/*
 * Fused-multiply-add variants (reading R22).  They are NOT the
 * paper's methods -- the paper's C99 rounds every product separately -- but the same
 * algorithms with every "s + x*y" contracted into one fma(x, y, s), all orders unchanged:
 *   mm_kahan_fused           NaivKahan with err = fma(A_ik, B_kj, err)
 *   mm_winograd_fused        WinogradOriginal with y, z, the pair sums and the odd-P
 *                            term accumulated by fma
 *   mm_winograd_scaled_fused WinogradScaled on top of mm_winograd_fused
 * Each equals the oracle's or_*_fused bit for bit.  Arguments, layout, workspace (the same sizes
 * as the literal methods: mm_workspace_size(MM_*_FUSED, ...)), stream and error behaviour are
 * those of mm_kahan / mm_winograd / mm_winograd_scaled.
 */
int mm_kahan_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* stream);
int mm_winograd_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                      void* workspace, size_t ws_bytes, void* stream);
int mm_winograd_scaled_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                             void* workspace, size_t ws_bytes, int32_t* lambda_out, void* stream);

/*
 * Multi-GPU row-block layer (BASELINE.json north_star: "C is partitioned by
 * row blocks of A with B broadcast over NVLink through NCCL").  One process per GPU.  NCCL is
 * loaded at run time (the soname libnccl.so.2 if resident -- e.g. after PyTorch initialised NCCL --
 * else the path in the environment variable MM_NCCL_LIBRARY); without it these return MM_ERR_NCCL
 * and the rest of the library is unaffected.  One communicator per process.
 *
 * mm_dist_get_unique_id -- rank 0 creates the 128-byte NCCL id (HOST buffer) that every rank
 *   passes to mm_dist_init (distribute it out of band, e.g. torch.distributed).
 * mm_dist_init -- join the communicator as `rank` of `world` on CUDA device `device` (made
 *   current).  MM_ERR_ARG if already initialised or arguments are out of range.
 * mm_dist_gemm -- C_shard = A_shard B for this rank's N_local rows (N_local >= 0; a rank without
 *   rows still takes part in the collectives).  B: DEVICE buffer P x M on every rank; the root's
 *   content is broadcast into it in place inside the call.  method: an mm_method id.  The call
 *   executes the schedule mm_dist_schedule(method, P, M, levels, panels) returns: communication
 *   ops in order on the layer's own stream, compute ops (mm_dist_step) in order on `stream`,
 *   joined by events -- the same schedule the torch.distributed driver (paper_1106_1347_b200.dist)
 *   executes.  The schedule depends only on (method, P, M, levels, panels), values every rank
 *   shares, so every rank issues the same collectives.  Classical, Kahan and both Winograds are
 *   bitwise the rows of the one-GPU product; Strassen recurses on the shard (within its
 *   tolerance).  workspace: DEVICE, >= mm_dist_workspace_size(...).  Stream-ordered and
 *   asynchronous like the other entry points; the current device must be the one given to
 *   mm_dist_init.
 * mm_dist_finalize -- destroy the communicator and the layer's stream and events.
 *
 * mm_dist_schedule -- the multi-GPU schedule of one product as a list of ops (HOST array `ops` of
 *   `cap` entries; returns the number of ops, or MM_ERR_ARG for bad arguments / a too small cap --
 *   16 + 12 * panels always suffices).  Pure host function (no GPU).  Ops:
 *     MM_OP_BCAST            comm: broadcast rows [lo, hi) of B from the root
 *     MM_OP_ALLREDUCE_NORMS  comm: max-all-reduce of the two doubles at the workspace start
 *     MM_OP_RECORD / _WAIT   record / wait for event `index` on `stream` (MM_STREAM_*)
 *     MM_OP_NORMS .. _FULL   compute ops, run by mm_dist_step (below) in list order.
 *   With panels > 1 B travels as row panels and the product follows panel by panel (SURVEY 8(f)
 *   NEXT-4): NaivStandard, NaivKahan and WinogradOriginal (+ fused) accumulate k-panels
 *   (mm_naive_ex / mm_kahan_ex / mm_winograd_ex, Kahan/Winograd when P and M are even);
 *   WinogradScaled (P and M even) max-all-reduces {||A_r||, ||B|| of the root} before B moves, so
 *   lambda is known at once, then scales each arriving panel of B (z' continued panel to panel)
 *   and accumulates its pair sums; Strassen (levels >= 1) forms the B-side operands of each
 *   arriving panel -- panel i is the quadrant rows [u_i, u_{i+1}) of the first formation pass,
 *   i.e. the B rows u + r (Pp >> s), r < 2^s, s the levels that pass spans.  Otherwise (panels
 *   <= 1, odd P or M, the paper plan levels = -1): one broadcast, then the one-GPU method.
 *   Panels are listed in increasing k, so every result is bitwise the one-broadcast schedule's.
 * mm_dist_step -- run ONE compute op of a schedule on `stream` (no communication): A_shard, B,
 *   C_shard, workspace as for mm_dist_gemm; is_root: this rank is the broadcast root (MM_OP_NORMS
 *   then contributes ||B||, other ranks 0).  B rows an op reads must already hold the root's data
 *   (the schedule's WAIT ops ensure it).  A rank whose operands cannot use the panel kernels (an
 *   A_shard that is not 16-byte aligned) skips the panel steps and runs the one-GPU kernel at the
 *   last one -- its collectives are unchanged.  N_local == 0: every op but MM_OP_NORMS is a no-op.
 */
#define MM_OP_BCAST 1
#define MM_OP_ALLREDUCE_NORMS 2
#define MM_OP_RECORD 3
#define MM_OP_WAIT 4
#define MM_OP_NORMS 5        /* ||A_r||_inf -> norms[0]; root: ||B||_inf -> norms[1], else 0 */
#define MM_OP_PANEL 6        /* k-panel [lo, hi) with MM_EX_* flags (scaled: on 2^lambda A, 2^-lambda B) */
#define MM_OP_YZ 7           /* WinogradOriginal's y, z of the full operands (before its last panel) */
#define MM_OP_SCALE_A 8      /* lambda from the norms; 2^lambda A and its y' */
#define MM_OP_SCALE_B 9      /* rows [lo, hi) of 2^-lambda B, z' continued (flags & MM_EX_ACCUMULATE) */
#define MM_OP_FORM_A 10      /* Strassen: every A-side formation pass */
#define MM_OP_FORM_B 11      /* Strassen: the first B-side pass on its units [lo, hi) */
#define MM_OP_FORM_B_REST 12 /* Strassen: the remaining B-side passes */
#define MM_OP_LEAF_COMBINE 13 /* Strassen: the batched leaf products and the combination passes */
#define MM_OP_FULL 14        /* the one-GPU method on the shard (B complete) */
/* the alternative partition of mm_s7_schedule (below) */
#define MM_OP_BCAST_A 15     /* comm: broadcast rows [lo, hi) of A from the root */
#define MM_OP_S7_FORM 16     /* the level-1 operands of product `index` (0..6 = H_1..H_7) */
#define MM_OP_S7_PRODUCT 17  /* H_{index+1} = their product, levels - 1 further levels, into slot index */
#define MM_OP_SEND_H 18      /* comm: send H slot `index` to rank lo */
#define MM_OP_RECV_H 19      /* comm: receive H slot `index` from rank lo */
#define MM_OP_S7_COMBINE 20  /* C from the seven H slots (the level-0 combination, P:279-282 / P:307-311) */
#define MM_STREAM_COMPUTE 0
#define MM_STREAM_COMM 1
typedef struct {
  int32_t op;     /* MM_OP_* */
  int32_t stream; /* MM_STREAM_* (RECORD / WAIT) */
  int32_t index;  /* event slot (RECORD / WAIT), panel number (other ops) */
  int32_t flags;  /* MM_EX_* (PANEL, SCALE_B) */
  int64_t lo, hi; /* row range of B (BCAST, SCALE_B), k range (PANEL), unit range (FORM_B) */
} mm_dist_op;
int mm_dist_get_unique_id(void* id_out);
int mm_dist_init(int32_t rank, int32_t world, const void* unique_id, int32_t device);
size_t mm_dist_workspace_size(int method, int64_t N_local, int64_t P, int64_t M, int32_t levels);
int mm_dist_gemm(int method, const double* A_shard, double* B, double* C_shard, int64_t N_local, int64_t P,
                 int64_t M, int32_t root, int32_t levels, int32_t panels, void* workspace, size_t ws_bytes,
                 void* stream);
int mm_dist_finalize(void);
int mm_dist_schedule(int method, int64_t P, int64_t M, int32_t levels, int32_t panels, mm_dist_op* ops, int32_t cap);
int mm_dist_step(int method, const mm_dist_op* op, const double* A_shard, const double* B, double* C_shard,
                 int64_t N_local, int64_t P, int64_t M, int32_t levels, int32_t is_root, void* workspace,
                 size_t ws_bytes, void* stream);

/*
 * Alternative partition: Strassen's seven top-level products (P:270-277 /
 * P:299-306) spread over the ranks -- product p (0..6, H_{p+1}) on rank p % world.  Not the
 * default (DESIGN.md section 7 compares it with the row blocks).  Every rank receives A and B
 * (broadcasts from the root), forms the level-1 operands of its products from the zero-embedded
 * quadrants (the one-GPU formation's per-element operations), multiplies them with levels - 1
 * further levels (the one-GPU recursion on that node), and sends each H to the root, which forms
 * C by the level-0 combination.  The root's C is therefore bitwise the one-GPU mm_strassen /
 * mm_strassen_winograd(levels) product.  method: MM_STRASSEN or MM_STRASSEN_WINOGRAD; levels >= 1
 * (the GPU plan, reading R10).
 *
 * mm_s7_schedule -- the op list of `rank` (HOST array `ops` of `cap` entries, 64 always suffice;
 *   returns the count or MM_ERR_ARG): MM_OP_BCAST_A / MM_OP_BCAST (every rank), RECORD / WAIT,
 *   MM_OP_S7_FORM + MM_OP_S7_PRODUCT per owned product, MM_OP_SEND_H (owner -> root) /
 *   MM_OP_RECV_H (root), MM_OP_S7_COMBINE (root).  A function of (method, N, P, M, levels, world,
 *   rank, root) only; pure host function.  Consecutive SEND_H / RECV_H ops form one NCCL group.
 * mm_s7_workspace_size -- DEVICE workspace bytes of one rank (0 on bad arguments).  Layout, for
 *   h = (Np/2)(Mp/2) with (Np, Pp, Mp) = mm_strassen_plan(N, P, M, levels): seven contiguous H
 *   slots of h doubles at offset 0 (slot p = H_{p+1}, dense (Np/2) x (Mp/2)), then the two level-1
 *   operands and the workspace of the levels - 1 sub-product.  Executors move slot p with SEND_H /
 *   RECV_H.
 * mm_s7_step -- run ONE compute op of an mm_s7_schedule on `stream`: A (N x P) and B (P x M)
 *   DEVICE buffers holding the root's data, C (N x M, DEVICE) used by MM_OP_S7_COMBINE only.
 * mm_dist_strassen7 -- the NCCL executor of that schedule on the communicator of mm_dist_init: A
 *   and B DEVICE buffers on every rank (the root's content broadcast into them in place), C on the
 *   root (may be NULL elsewhere).  Stream-ordered and asynchronous like mm_dist_gemm.
 */
int mm_s7_schedule(int method, int64_t N, int64_t P, int64_t M, int32_t levels, int32_t world, int32_t rank,
                   int32_t root, mm_dist_op* ops, int32_t cap);
size_t mm_s7_workspace_size(int method, int64_t N, int64_t P, int64_t M, int32_t levels);
int mm_s7_step(int method, const mm_dist_op* op, const double* A, const double* B, double* C, int64_t N, int64_t P,
               int64_t M, int32_t levels, void* workspace, size_t ws_bytes, void* stream);
int mm_dist_strassen7(int method, double* A, double* B, double* C, int64_t N, int64_t P, int64_t M, int32_t root,
                      int32_t levels, void* workspace, size_t ws_bytes, void* stream);

/*
 * mm_launch_count -- number of kernels this library has launched in this process (a
 * monotonically increasing diagnostic counter, used by bench.py's "gpu_launches").
 */
uint64_t mm_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MM_B200_H */
