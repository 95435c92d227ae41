// mm_abi.cu -- the extern "C" boundary declared in include/mm.h: argument validation,
// workspace carving and kernel dispatch.  Every arithmetic step runs in the sm_100a kernels
// included below; this file does no arithmetic on matrix data.
#include "../../include/mm.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "dist_nccl.cuh"
#include "gemm_tma.cuh"
#include "host_pipeline.cuh"
#include "kahan.cuh"
#include "repack.cuh"
#include "lines.cuh"
#include "strassen.cuh"
#include "winograd.cuh"

namespace {

constexpr int kMaxDevices = 64;
int g_dev_ok[kMaxDevices];  // 0 unknown, 1 sm_100, -1 other
int g_dev_sms[kMaxDevices];

int check_device(int* sms_out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return MM_ERR_UNSUPPORTED;
  }
  if (dev < 0 || dev >= kMaxDevices) return MM_ERR_UNSUPPORTED;
  if (g_dev_ok[dev] == 0) {
    int major = 0, minor = 0, sms = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      return MM_ERR_UNSUPPORTED;
    }
    g_dev_ok[dev] = (major == 10 && minor == 0) ? 1 : -1;
    g_dev_sms[dev] = sms;
  }
  if (g_dev_ok[dev] != 1) return MM_ERR_UNSUPPORTED;
  if (sms_out) *sms_out = g_dev_sms[dev];
  return MM_OK;
}

bool mul_ok(int64_t a, int64_t b) { return a > 0 && b > 0 && a <= INT64_MAX / 8 / b; }

bool overlaps(const void* p, int64_t pn, const void* q, int64_t qn) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p), a1 = a0 + uintptr_t(pn) * 8;
  const uintptr_t b0 = reinterpret_cast<uintptr_t>(q), b1 = b0 + uintptr_t(qn) * 8;
  return a0 < b1 && b0 < a1;
}

int check_abc(const double* A, const double* B, const double* C, int64_t N, int64_t P, int64_t M) {
  if (!A || !B || !C) return MM_ERR_ARG;
  if (N < 1 || P < 1 || M < 1) return MM_ERR_ARG;
  if (!mul_ok(N, P) || !mul_ok(P, M) || !mul_ok(N, M)) return MM_ERR_ARG;
  if (overlaps(C, N * M, A, N * P) || overlaps(C, N * M, B, P * M)) return MM_ERR_ALIAS;
  return MM_OK;
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return MM_OK;
  cudaGetLastError();
  return MM_ERR_CUDA;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

size_t winograd_ws(int64_t N, int64_t M) {
  return mmk::align256(size_t(N) * 8) + mmk::align256(size_t(M) * 8);
}
// odd P: room for A copied to the even pitch P + 1 (repack.cuh), used when the caller passes it
size_t repack_ws(int64_t N, int64_t P) { return (P & 1) ? mmk::align256(size_t(N) * size_t(P + 1) * 8) : 0; }
constexpr size_t kScaledHeader = 256;  // norms[2] (u64), scale[2] (double), lambda (int)
// header | y | z | 2^lambda A | 2^-lambda B
size_t scaled_ws(int64_t N, int64_t P, int64_t M) {
  return kScaledHeader + winograd_ws(N, M) + mmk::align256(size_t(N) * size_t(mmk::scaled_pitch(P)) * 8) +
         mmk::align256(size_t(P) * size_t(M) * 8);
}

}  // namespace

extern "C" {

const char* mm_version(void) { return "paper_1106_1347_b200 0.1.0 (sm_100a, FP64 DMMA)"; }

const char* mm_status_string(int status) {
  switch (status) {
    case MM_OK: return "ok";
    case MM_ERR_ARG: return "invalid argument (NULL pointer, size < 1 or overflow, bad levels)";
    case MM_ERR_ALIAS: return "C overlaps A or B";
    case MM_ERR_WORKSPACE: return "workspace too small (see mm_workspace_size)";
    case MM_ERR_CUDA: return "CUDA launch or runtime error";
    case MM_ERR_UNSUPPORTED: return "current device is not sm_100 (B200); no fallback exists";
    case MM_ERR_NCCL: return "NCCL unavailable or an NCCL call failed (multi-GPU layer)";
    default: return "unknown status";
  }
}

int32_t mm_lambda(double nA, double nB) { return mmk::lambda_rule(nA, nB); }

int mm_naive(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* stream) {
  mmk::NvtxRange nvtx("mm_naive");
  int rc = check_abc(A, B, C, N, P, M);
  if (rc) return rc;
  int sms = 148;
  if ((rc = check_device(&sms))) return rc;
  mmk::GemmProblem pr{A, B, C, N, P, M, P, M, M, 0, 0, 0, 1};
  return cuda_status(mmk::launch_dgemm(pr, S(stream), sms));
}

int mm_naive_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int64_t N,
                int64_t K, int64_t M, int32_t accumulate, void* stream) {
  if (!A || !B || !C || N < 1 || K < 1 || M < 1 || lda < K || ldb < M || ldc < M) return MM_ERR_ARG;
  if (!mul_ok(N, lda) || !mul_ok(K, ldb) || !mul_ok(N, ldc)) return MM_ERR_ARG;
  const int64_t na = (N - 1) * lda + K, nb = (K - 1) * ldb + M, nc = (N - 1) * ldc + M;  // spans
  if (overlaps(C, nc, A, na) || overlaps(C, nc, B, nb)) return MM_ERR_ALIAS;
  int sms = 148, rc;
  if ((rc = check_device(&sms))) return rc;
  mmk::GemmProblem pr{A, B, C, N, K, M, lda, ldb, ldc, 0, 0, 0, 1};
  pr.accumulate = accumulate ? 1 : 0;
  return cuda_status(mmk::launch_dgemm(pr, S(stream), sms));
}

int mm_kahan(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* stream) {
  mmk::NvtxRange nvtx("mm_kahan");
  int rc = check_abc(A, B, C, N, P, M);
  if (rc) return rc;
  int sms = 148;
  if ((rc = check_device(&sms))) return rc;
  return cuda_status(mmk::launch_kahan(A, B, C, N, P, M, S(stream), sms));
}

int mm_kahan_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* stream) {
  mmk::NvtxRange nvtx("mm_kahan_fused");
  int rc = check_abc(A, B, C, N, P, M);
  if (rc) return rc;
  int sms = 148;
  if ((rc = check_device(&sms))) return rc;
  return cuda_status(mmk::launch_kahan<void, true>(A, B, C, N, P, M, S(stream), sms));
}

// k-panel steps of NaivKahan / WinogradOriginal: TMA-describable operands only
static int ex_check(const double* A, int64_t lda, const double* B, int64_t ldb, const double* C, int64_t N,
                    int64_t K, int64_t M, int32_t flags) {
  if (!A || !B || !C || N < 1 || K < 1 || M < 1 || lda < K || ldb < M) return MM_ERR_ARG;
  if (flags & ~(MM_EX_ACCUMULATE | MM_EX_KEEP_STATE | MM_EX_FUSED)) return MM_ERR_ARG;
  if (!mul_ok(N, lda) || !mul_ok(K, ldb) || !mul_ok(N, M)) return MM_ERR_ARG;
  if (!mmk::simt_tma_ex_ok(A, lda, B, ldb, N, K, M)) return MM_ERR_ARG;
  const int64_t na = (N - 1) * lda + K, nb = (K - 1) * ldb + M;
  if (overlaps(C, N * M, A, na) || overlaps(C, N * M, B, nb)) return MM_ERR_ALIAS;
  return MM_OK;
}

static int ex_flags(int32_t flags) {
  return ((flags & MM_EX_ACCUMULATE) ? mmk::SIMT_EX_ACC : 0) | ((flags & MM_EX_KEEP_STATE) ? mmk::SIMT_EX_KEEP : 0);
}

int mm_kahan_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, double* E, int64_t N,
                int64_t K, int64_t M, int32_t flags, void* stream) {
  mmk::NvtxRange nvtx("mm_kahan_ex");
  int rc = ex_check(A, lda, B, ldb, C, N, K, M, flags);
  if (rc) return rc;
  if ((flags & (MM_EX_ACCUMULATE | MM_EX_KEEP_STATE)) && !E) return MM_ERR_ARG;
  if (E && (overlaps(E, N * M, C, N * M) || overlaps(E, N * M, A, (N - 1) * lda + K) ||
            overlaps(E, N * M, B, (K - 1) * ldb + M)))
    return MM_ERR_ALIAS;
  if ((rc = check_device(nullptr))) return rc;
  const int f = ex_flags(flags);
  return cuda_status((flags & MM_EX_FUSED)
                         ? mmk::launch_kahan_tma_ex<mmk::KahanTma, true>(A, lda, B, ldb, C, E, N, K, M, f, S(stream))
                         : mmk::launch_kahan_tma_ex<mmk::KahanTma, false>(A, lda, B, ldb, C, E, N, K, M, f, S(stream)));
}

int mm_winograd_ex(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, const double* y,
                   const double* z, int64_t N, int64_t K, int64_t M, int32_t flags, void* stream) {
  mmk::NvtxRange nvtx("mm_winograd_ex");
  int rc = ex_check(A, lda, B, ldb, C, N, K, M, flags);
  if (rc) return rc;
  if (K % 2 != 0) return MM_ERR_ARG;  // whole pairs per panel
  if (!(flags & MM_EX_KEEP_STATE) && (!y || !z)) return MM_ERR_ARG;
  if ((y && overlaps(C, N * M, y, N)) || (z && overlaps(C, N * M, z, M))) return MM_ERR_ALIAS;
  if ((rc = check_device(nullptr))) return rc;
  const int f = ex_flags(flags);
  return cuda_status(
      (flags & MM_EX_FUSED)
          ? mmk::launch_winograd_tma_ex<mmk::WinogradTma, true>(A, lda, B, ldb, C, y, z, N, K, M, f, S(stream))
          : mmk::launch_winograd_tma_ex<mmk::WinogradTma, false>(A, lda, B, ldb, C, y, z, N, K, M, f, S(stream)));
}

int mm_winograd_yz(const double* A, const double* B, int64_t N, int64_t P, int64_t M, double* y, double* z,
                   int32_t flags, void* stream) {
  mmk::NvtxRange nvtx("mm_winograd_yz");
  if (!A || !B || !y || !z || N < 1 || P < 1 || M < 1 || !mul_ok(N, P) || !mul_ok(P, M)) return MM_ERR_ARG;
  if (flags & ~MM_EX_FUSED) return MM_ERR_ARG;
  if (overlaps(y, N, A, N * P) || overlaps(y, N, B, P * M) || overlaps(z, M, A, N * P) ||
      overlaps(z, M, B, P * M) || overlaps(y, N, z, M))
    return MM_ERR_ALIAS;
  int rc = check_device(nullptr);
  if (rc) return rc;
  return cuda_status(mmk::launch_yz(A, B, y, z, N, P, M, nullptr, nullptr, nullptr, nullptr, nullptr, S(stream),
                                    (flags & MM_EX_FUSED) != 0));
}

size_t mm_workspace_size(int method, int64_t N, int64_t P, int64_t M, int32_t levels) {
  if (N < 1 || P < 1 || M < 1) return 0;
  switch (method) {
    case MM_NAIVE:
    case MM_KAHAN:
    case MM_KAHAN_FUSED: return repack_ws(N, P);
    case MM_WINOGRAD:
    case MM_WINOGRAD_FUSED: return winograd_ws(N, M) + repack_ws(N, P);
    case MM_WINOGRAD_SCALED:
    case MM_WINOGRAD_SCALED_FUSED: return scaled_ws(N, P, M);
    case MM_STRASSEN:
    case MM_STRASSEN_WINOGRAD: {
      mmk::StrassenPlan pl;
      if (!mmk::make_strassen_plan(N, P, M, levels, &pl)) return 0;
      return pl.total;
    }
    default: return 0;
  }
}

// the repack path: odd P, a large enough grid of the TMA kernel's tiles (>= `waves` full waves at
// 2 CTAs per SM), M even, a 16-byte aligned B and workspace room for the copy
static bool repack_ok(const double* A, const double* B, int64_t N, int64_t P, int64_t M, size_t room, int bm, int bn,
                      int waves, int sms) {
  if (!(P & 1) || P < 3 || M % 2 || room < repack_ws(N, P) || !mmk::tma_ok(B, M)) return false;
  if (N > INT32_MAX || P > INT32_MAX || M > INT32_MAX) return false;
  (void)A;
  return mmk::cdiv(N, int64_t(bm)) * mmk::cdiv(M, int64_t(bn)) >= int64_t(waves) * 2 * sms;
}

static int winograd_common(bool fused, const double* A, const double* B, double* C, int64_t N, int64_t P,
                           int64_t M, void* workspace, size_t ws_bytes, void* stream) {
  mmk::NvtxRange nvtx(fused ? "mm_winograd_fused" : "mm_winograd");
  int rc = check_abc(A, B, C, N, P, M);
  if (rc) return rc;
  if (!workspace) return MM_ERR_ARG;
  if (ws_bytes < winograd_ws(N, M)) return MM_ERR_WORKSPACE;
  int sms = 148;
  if ((rc = check_device(&sms))) return rc;
  double* y = static_cast<double*>(workspace);
  double* z = reinterpret_cast<double*>(static_cast<char*>(workspace) + mmk::align256(size_t(N) * 8));
  double* Ar = reinterpret_cast<double*>(static_cast<char*>(workspace) + winograd_ws(N, M));
  if (repack_ok(A, B, N, P, M, ws_bytes - winograd_ws(N, M), mmk::WinogradTma::BM, mmk::WinogradTma::BN, 2, sms)) {
    // odd P: A at pitch P + 1, then the TMA-fed pair kernel with the odd term in its epilogue
    cudaStream_t st = S(stream);
    cudaError_t e = mmk::launch_repack_rows(A, P, Ar, P + 1, N, P, sms, st);
    if (e == cudaSuccess)
      e = mmk::launch_yz(A, B, y, z, N, P, M, nullptr, nullptr, nullptr, nullptr, nullptr, st, fused);
    if (e == cudaSuccess)
      e = fused ? mmk::launch_winograd_pairs_tma_odd_auto<true>(Ar, P + 1, B, M, C, y, z, N, P, M, st, sms)
                : mmk::launch_winograd_pairs_tma_odd_auto<false>(Ar, P + 1, B, M, C, y, z, N, P, M, st, sms);
    return cuda_status(e);
  }
  return cuda_status(fused ? mmk::launch_winograd<void, true>(A, B, C, y, z, N, P, M, S(stream), sms)
                           : mmk::launch_winograd<void, false>(A, B, C, y, z, N, P, M, S(stream), sms));
}

int mm_winograd(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* workspace,
                size_t ws_bytes, void* stream) {
  return winograd_common(false, A, B, C, N, P, M, workspace, ws_bytes, stream);
}

int mm_winograd_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, void* workspace,
                      size_t ws_bytes, void* stream) {
  return winograd_common(true, A, B, C, N, P, M, workspace, ws_bytes, stream);
}

uint64_t mm_launch_count(void) { return mmk::launch_counter().load(); }

int mm_winograd_scaled(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                       void* workspace, size_t ws_bytes, int32_t* lambda_out, void* stream) {
  return mm_winograd_scaled_norms(A, B, C, N, P, M, nullptr, workspace, ws_bytes, lambda_out, stream);
}

static int winograd_scaled_common(bool fused, const double* A, const double* B, double* C, int64_t N, int64_t P,
                                  int64_t M, const double* norms_device, void* workspace, size_t ws_bytes,
                                  int32_t* lambda_out, void* stream) {
  mmk::NvtxRange nvtx(fused ? "mm_winograd_scaled_fused" : "mm_winograd_scaled");
  int rc = check_abc(A, B, C, N, P, M);
  if (rc) return rc;
  if (!workspace) return MM_ERR_ARG;
  if (ws_bytes < scaled_ws(N, P, M)) return MM_ERR_WORKSPACE;
  int sms = 148;
  if ((rc = check_device(&sms))) return rc;
  char* ws = static_cast<char*>(workspace);
  auto* norms = reinterpret_cast<unsigned long long*>(ws);
  auto* scale = reinterpret_cast<double*>(ws + 16);
  auto* lam = reinterpret_cast<int*>(ws + 32);
  double* y = reinterpret_cast<double*>(ws + kScaledHeader);
  double* z = reinterpret_cast<double*>(ws + kScaledHeader + mmk::align256(size_t(N) * 8));
  double* As = reinterpret_cast<double*>(ws + kScaledHeader + winograd_ws(N, M));
  double* Bs =
      reinterpret_cast<double*>(reinterpret_cast<char*>(As) + mmk::align256(size_t(N) * size_t(mmk::scaled_pitch(P)) * 8));
  cudaStream_t st = S(stream);
  cudaError_t e = cudaSuccess;
  // K4 norms -> lambda + exact copies 2^lambda A, 2^-lambda B + their y, z -> pair sums.
  // With norms_device the caller's {||A||, ||B||} are used (the same 16 bytes, read as bit patterns).
  const auto* given = reinterpret_cast<const unsigned long long*>(norms_device);
  e = fused ? mmk::launch_winograd_scaled<true>(A, B, C, N, P, M, norms, given, lam, scale, y, z, As, Bs, st, sms)
            : mmk::launch_winograd_scaled<false>(A, B, C, N, P, M, norms, given, lam, scale, y, z, As, Bs, st, sms);
  if (e == cudaSuccess && lambda_out) {
    e = cudaMemcpyAsync(lambda_out, lam, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  return cuda_status(e);
}

int mm_winograd_scaled_norms(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                             const double* norms_device, void* workspace, size_t ws_bytes, int32_t* lambda_out,
                             void* stream) {
  return winograd_scaled_common(false, A, B, C, N, P, M, norms_device, workspace, ws_bytes, lambda_out, stream);
}

int mm_winograd_scaled_fused(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                             void* workspace, size_t ws_bytes, int32_t* lambda_out, void* stream) {
  return winograd_scaled_common(true, A, B, C, N, P, M, nullptr, workspace, ws_bytes, lambda_out, stream);
}

int mm_strassen_plan(int64_t N, int64_t P, int64_t M, int32_t levels, int32_t* depth_out, int64_t* Np_out,
                     int64_t* Pp_out, int64_t* Mp_out) {
  mmk::StrassenPlan pl;
  if (!mmk::make_strassen_plan(N, P, M, levels, &pl)) return MM_ERR_ARG;
  if (depth_out) *depth_out = pl.depth;
  if (Np_out) *Np_out = pl.Np;
  if (Pp_out) *Pp_out = pl.Pp;
  if (Mp_out) *Mp_out = pl.Mp;
  return MM_OK;
}

static int strassen_common(int variant, const double* A, const double* B, double* C, int64_t N, int64_t P,
                           int64_t M, int32_t levels, void* workspace, size_t ws_bytes, void* stream) {
  mmk::NvtxRange nvtx(variant == mmk::SV_NAIV ? "mm_strassen" : "mm_strassen_winograd");
  int rc = check_abc(A, B, C, N, P, M);
  if (rc) return rc;
  mmk::StrassenPlan pl;
  if (!mmk::make_strassen_plan(N, P, M, levels, &pl)) return MM_ERR_ARG;
  if (pl.total > 0 && (!workspace || ws_bytes < pl.total)) return MM_ERR_WORKSPACE;
  int sms = 148;
  if ((rc = check_device(&sms))) return rc;
  char* ws = static_cast<char*>(workspace);
  cudaError_t e = variant == mmk::SV_NAIV ? mmk::run_strassen<mmk::SV_NAIV>(A, B, C, N, P, M, pl, ws, sms, S(stream))
                                          : mmk::run_strassen<mmk::SV_WINOGRAD>(A, B, C, N, P, M, pl, ws, sms,
                                                                               S(stream));
  return cuda_status(e);
}

int mm_strassen(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M, int32_t levels,
                void* workspace, size_t ws_bytes, void* stream) {
  return strassen_common(mmk::SV_NAIV, A, B, C, N, P, M, levels, workspace, ws_bytes, stream);
}

int mm_strassen_winograd(const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                         int32_t levels, void* workspace, size_t ws_bytes, void* stream) {
  return strassen_common(mmk::SV_WINOGRAD, A, B, C, N, P, M, levels, workspace, ws_bytes, stream);
}

// NaivStandard / NaivKahan with odd P and the caller's workspace: A copied to the even pitch P + 1
// (repack.cuh), then the TMA-fed kernels on the copy -- bitwise the direct calls' results
static int gemm_repacked(int method, const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
                         void* workspace, size_t ws_bytes, void* stream) {
  int rc = check_abc(A, B, C, N, P, M);
  if (rc) return rc;
  int sms = 148;
  if ((rc = check_device(&sms))) return rc;
  double* Ar = static_cast<double*>(workspace);
  if (overlaps(Ar, N * (P + 1), A, N * P) || overlaps(Ar, N * (P + 1), B, P * M) ||
      overlaps(Ar, N * (P + 1), C, N * M))
    return MM_ERR_ALIAS;
  const bool naive = method == MM_NAIVE;
  const bool ok = naive ? repack_ok(A, B, N, P, M, ws_bytes, mmk::GemmTma::BM, mmk::GemmTma::BN, 2, sms)
                        : repack_ok(A, B, N, P, M, ws_bytes, mmk::KahanTma::BM, mmk::KahanTma::BN, 2, sms);
  if (!ok)
    return naive ? mm_naive(A, B, C, N, P, M, stream)
           : method == MM_KAHAN ? mm_kahan(A, B, C, N, P, M, stream)
                                : mm_kahan_fused(A, B, C, N, P, M, stream);
  cudaStream_t st = S(stream);
  cudaError_t e = mmk::launch_repack_rows(A, P, Ar, P + 1, N, P, sms, st);
  if (e != cudaSuccess) return cuda_status(e);
  if (naive) {
    mmk::GemmProblem pr{Ar, B, C, N, P, M, P + 1, M, M, 0, 0, 0, 1};
    return cuda_status(mmk::launch_dgemm(pr, st, sms));
  }
  return cuda_status(method == MM_KAHAN
                         ? mmk::launch_kahan_tma_ex<mmk::KahanTma, false>(Ar, P + 1, B, M, C, nullptr, N, P, M, 0, st)
                         : mmk::launch_kahan_tma_ex<mmk::KahanTma, true>(Ar, P + 1, B, M, C, nullptr, N, P, M, 0, st));
}

int mm_gemm(int method, const double* A, const double* B, double* C, int64_t N, int64_t P, int64_t M,
            int32_t levels, void* workspace, size_t ws_bytes, int32_t* lambda_out, void* stream) {
  switch (method) {
    case MM_NAIVE:
    case MM_KAHAN:
    case MM_KAHAN_FUSED:
      if (workspace && (P & 1) && ws_bytes >= repack_ws(N, P)) return gemm_repacked(method, A, B, C, N, P, M, workspace,
                                                                                    ws_bytes, stream);
      return method == MM_NAIVE ? mm_naive(A, B, C, N, P, M, stream)
             : method == MM_KAHAN ? mm_kahan(A, B, C, N, P, M, stream)
                                  : mm_kahan_fused(A, B, C, N, P, M, stream);
    case MM_WINOGRAD: return mm_winograd(A, B, C, N, P, M, workspace, ws_bytes, stream);
    case MM_WINOGRAD_SCALED: return mm_winograd_scaled(A, B, C, N, P, M, workspace, ws_bytes, lambda_out, stream);
    case MM_STRASSEN: return mm_strassen(A, B, C, N, P, M, levels, workspace, ws_bytes, stream);
    case MM_STRASSEN_WINOGRAD: return mm_strassen_winograd(A, B, C, N, P, M, levels, workspace, ws_bytes, stream);
    case MM_WINOGRAD_FUSED: return mm_winograd_fused(A, B, C, N, P, M, workspace, ws_bytes, stream);
    case MM_WINOGRAD_SCALED_FUSED:
      return mm_winograd_scaled_fused(A, B, C, N, P, M, workspace, ws_bytes, lambda_out, stream);
    default: return MM_ERR_ARG;
  }
}

// ---------------------------------------------------------------- host buffers (the paper's test program)
// product buffers of mm_methods_host: method i computes into buffer i % 3 once the copy-back of
// method i - 3 has left it, so every copy-back overlaps at least the two methods after it (with two
// buffers a copy-back slower than the next method -- c4's 537 MB behind a 22 ms Strassen call on
// a slow host link -- stalled the third method)
constexpr int kHostCBuffers = 3;

static size_t host_ws_method(const int* methods, int32_t n, int64_t N, int64_t P, int64_t M, int32_t levels) {
  size_t w = 0;
  for (int i = 0; i < n; ++i) {
    const size_t x = mm_workspace_size(methods[i], N, P, M, levels);
    w = x > w ? x : w;
  }
  return w;
}

size_t mm_methods_host_workspace_size(const int* methods, int32_t n, int64_t N, int64_t P, int64_t M,
                                      int32_t levels) {
  if (!methods || n < 1 || N < 1 || P < 1 || M < 1 || !mul_ok(N, P) || !mul_ok(P, M) || !mul_ok(N, M)) return 0;
  const size_t nc = size_t(n < kHostCBuffers ? n : kHostCBuffers);
  return mmk::align256(size_t(N) * size_t(P) * 8) + mmk::align256(size_t(P) * size_t(M) * 8) +
         nc * mmk::align256(size_t(N) * size_t(M) * 8) + host_ws_method(methods, n, N, P, M, levels);
}

int mm_methods_host(const int* methods, int32_t n, const double* A_host, const double* B_host, double* const* C_host,
                    int64_t N, int64_t P, int64_t M, int32_t levels, int32_t row_blocks, void* dev_ws, size_t ws_bytes,
                    void* stream) {
  mmk::NvtxRange nvtx("mm_methods_host");
  if (!methods || n < 1 || !A_host || !B_host || !C_host || N < 1 || P < 1 || M < 1) return MM_ERR_ARG;
  if (!mul_ok(N, P) || !mul_ok(P, M) || !mul_ok(N, M)) return MM_ERR_ARG;
  for (int i = 0; i < n; ++i)
    if (methods[i] < MM_NAIVE || methods[i] > MM_WINOGRAD_SCALED_FUSED || !C_host[i]) return MM_ERR_ARG;
  if (!dev_ws || ws_bytes < mm_methods_host_workspace_size(methods, n, N, P, M, levels)) return MM_ERR_WORKSPACE;
  int rc = check_device(nullptr);
  if (rc) return rc;
  mmk::HostStreams* hs = mmk::host_streams();
  if (!hs) return MM_ERR_CUDA;
  cudaStream_t st = S(stream), si = hs->in, so = hs->out;
  char* w = static_cast<char*>(dev_ws);
  double* dA = reinterpret_cast<double*>(w);
  w += mmk::align256(size_t(N) * size_t(P) * 8);
  double* dB = reinterpret_cast<double*>(w);
  w += mmk::align256(size_t(P) * size_t(M) * 8);
  const int nc = n < kHostCBuffers ? n : kHostCBuffers;
  double* dC[kHostCBuffers];
  for (int k = 0; k < nc; ++k) {
    dC[k] = reinterpret_cast<double*>(w);
    w += mmk::align256(size_t(N) * size_t(M) * 8);
  }
  void* wsm = w;
  const size_t wsm_bytes = host_ws_method(methods, n, N, P, M, levels);

  std::vector<cudaEvent_t> evs;  // every event of this call, destroyed at the end
  auto event = [&](cudaStream_t on, cudaEvent_t* out) -> cudaError_t {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) return r;
    evs.push_back(e);
    *out = e;
    return cudaEventRecord(e, on);
  };
  auto finish = [&](int code) {
    cudaError_t e1 = cudaStreamSynchronize(so), e2 = cudaStreamSynchronize(st), e3 = cudaStreamSynchronize(si);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (code) return code;
    return cuda_status(e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3));
  };
#define MMH_TRY(x)                                \
  do {                                            \
    cudaError_t _e = (x);                         \
    if (_e != cudaSuccess) return finish(cuda_status(_e)); \
  } while (0)
#define MMH_RC(x)                       \
  do {                                  \
    int _r = (x);                       \
    if (_r) return finish(_r);          \
  } while (0)

  cudaEvent_t e0;
  MMH_TRY(event(st, &e0));  // the device buffers may be reused once prior work on `stream` is done
  MMH_TRY(cudaStreamWaitEvent(si, e0, 0));
  MMH_TRY(cudaStreamWaitEvent(so, e0, 0));
  const int rb = row_blocks < 1 ? 1 : (row_blocks > N ? int(N) : row_blocks);
  // ---- inputs: k-panels (first method NaivStandard) or B then row blocks of A
  std::vector<int64_t> kb, ab;
  std::vector<cudaEvent_t> ready;
  if (methods[0] == MM_NAIVE && P >= 4) {
    kb = mmk::host_growing_panels(P, rb);
    for (size_t j = 0; j + 1 < kb.size(); ++j) {
      const int64_t k0 = kb[j], k1 = kb[j + 1];
      MMH_TRY(cudaMemcpy2DAsync(dA + k0, size_t(P) * 8, A_host + k0, size_t(P) * 8, size_t(k1 - k0) * 8, size_t(N),
                                cudaMemcpyHostToDevice, si));
      MMH_TRY(cudaMemcpyAsync(dB + k0 * M, B_host + k0 * M, size_t(k1 - k0) * size_t(M) * 8, cudaMemcpyHostToDevice,
                              si));
      cudaEvent_t e;
      MMH_TRY(event(si, &e));
      ready.push_back(e);
    }
  } else {
    MMH_TRY(cudaMemcpyAsync(dB, B_host, size_t(P) * size_t(M) * 8, cudaMemcpyHostToDevice, si));
    const int nb = mmk::host_row_local(methods[0]) ? rb : 1;
    for (int b = 0; b <= nb; ++b) ab.push_back(N * b / nb);
    for (int b = 0; b < nb; ++b) {
      MMH_TRY(cudaMemcpyAsync(dA + ab[b] * P, A_host + ab[b] * P, size_t(ab[b + 1] - ab[b]) * size_t(P) * 8,
                              cudaMemcpyHostToDevice, si));
      cudaEvent_t e;
      MMH_TRY(event(si, &e));
      ready.push_back(e);
    }
  }
  cudaEvent_t inputs_done = ready.back();
  cudaEvent_t buf_free[kHostCBuffers] = {};
  // ---- the methods
  for (int i = 0; i < n; ++i) {
    const int m = methods[i];
    const int k = i % nc;
    double* C = dC[k];
    if (buf_free[k]) MMH_TRY(cudaStreamWaitEvent(st, buf_free[k], 0));  // its previous product has left
    auto d2h = [&](int64_t lo, int64_t hi) -> cudaError_t {
      cudaEvent_t e;
      cudaError_t r = event(st, &e);
      if (r == cudaSuccess) r = cudaStreamWaitEvent(so, e, 0);
      if (r == cudaSuccess)
        r = cudaMemcpyAsync(C_host[i] + lo * M, C + lo * M, size_t(hi - lo) * size_t(M) * 8, cudaMemcpyDeviceToHost,
                            so);
      return r;
    };
    const bool first = i == 0, last = i == n - 1;
    if (first && !kb.empty()) {  // NaivStandard accumulating k-panels as they land
      for (size_t j = 0; j + 1 < kb.size(); ++j) {
        MMH_TRY(cudaStreamWaitEvent(st, ready[j], 0));
        MMH_RC(mm_naive_ex(dA + kb[j], P, dB + kb[j] * M, M, C, M, N, kb[j + 1] - kb[j], M, j > 0 ? 1 : 0, stream));
      }
      MMH_TRY(d2h(0, N));
    } else if (first && mmk::host_row_local(m) && ab.size() > 2) {  // row blocks as A lands
      for (size_t b = 0; b + 1 < ab.size(); ++b) {
        MMH_TRY(cudaStreamWaitEvent(st, ready[b], 0));
        MMH_RC(mm_gemm(m, dA + ab[b] * P, dB, C + ab[b] * M, ab[b + 1] - ab[b], P, M, levels, wsm, wsm_bytes, nullptr,
                       stream));
        MMH_TRY(d2h(ab[b], ab[b + 1]));
      }
    } else if (last && mmk::host_row_local(m) && n > 1) {  // halving row blocks: a small last copy
      MMH_TRY(cudaStreamWaitEvent(st, inputs_done, 0));
      const std::vector<int64_t> tb = mmk::host_shrinking_rows(N, rb);
      for (size_t b = 0; b + 1 < tb.size(); ++b) {
        MMH_RC(mm_gemm(m, dA + tb[b] * P, dB, C + tb[b] * M, tb[b + 1] - tb[b], P, M, levels, wsm, wsm_bytes, nullptr,
                       stream));
        MMH_TRY(d2h(tb[b], tb[b + 1]));
      }
    } else {
      MMH_TRY(cudaStreamWaitEvent(st, inputs_done, 0));
      MMH_RC(mm_gemm(m, dA, dB, C, N, P, M, levels, wsm, wsm_bytes, nullptr, stream));
      MMH_TRY(d2h(0, N));
    }
    MMH_TRY(event(so, &buf_free[k]));
  }
#undef MMH_TRY
#undef MMH_RC
  return finish(MM_OK);
}

// ---------------------------------------------------------------- multi-GPU row-block layer (K9)
int mm_dist_get_unique_id(void* id_out) {
  if (!id_out) return MM_ERR_ARG;
  mmk::NcclApi* api = mmk::nccl_api();
  if (!api) return MM_ERR_NCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return MM_ERR_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return MM_OK;
}

int mm_dist_init(int32_t rank, int32_t world, const void* unique_id, int32_t device) {
  mmk::DistState& ds = mmk::dist_state();
  if (!unique_id || world < 1 || rank < 0 || rank >= world || device < 0 || ds.comm) return MM_ERR_ARG;
  mmk::NcclApi* api = mmk::nccl_api();
  if (!api) return MM_ERR_NCCL;
  if (cudaSetDevice(device) != cudaSuccess) return cuda_status(cudaErrorInvalidDevice);
  int rc = check_device(nullptr);
  if (rc) return rc;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  if (api->CommInitRank(&ds.comm, world, id, rank) != ncclSuccess) {
    ds.comm = nullptr;
    return MM_ERR_NCCL;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&ds.comm_stream, cudaStreamNonBlocking);
  for (int i = 0; e == cudaSuccess && i < mmk::kDistEvents; ++i)
    e = cudaEventCreateWithFlags(&ds.panel_ev[i], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ds.start_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ds.end_ev, cudaEventDisableTiming);
  ds.rank = rank;
  ds.world = world;
  ds.device = device;
  return cuda_status(e);
}

int mm_dist_finalize(void) {
  mmk::DistState& ds = mmk::dist_state();
  if (!ds.comm) return MM_ERR_ARG;
  mmk::NcclApi* api = mmk::nccl_api();
  const ncclResult_t r = api->CommDestroy(ds.comm);
  if (ds.comm_stream) cudaStreamDestroy(ds.comm_stream);
  for (int i = 0; i < mmk::kDistEvents; ++i)
    if (ds.panel_ev[i]) cudaEventDestroy(ds.panel_ev[i]);
  if (ds.start_ev) cudaEventDestroy(ds.start_ev);
  if (ds.end_ev) cudaEventDestroy(ds.end_ev);
  ds = mmk::DistState();
  return r == ncclSuccess ? MM_OK : MM_ERR_NCCL;
}

constexpr size_t kDistHeader = 256;  // the two norms of the distributed WinogradScaled

size_t mm_dist_workspace_size(int method, int64_t N_local, int64_t P, int64_t M, int32_t levels) {
  const int64_t n = N_local > 0 ? N_local : 1;
  if (method == MM_WINOGRAD_SCALED || method == MM_WINOGRAD_SCALED_FUSED)
    return kDistHeader + mm_workspace_size(method, n, P, M, levels);
  if (method == MM_KAHAN || method == MM_KAHAN_FUSED)  // E, the carried err of the panel schedule
    return mul_ok(n, M) ? mmk::align256(size_t(n) * size_t(M) * 8) : 0;
  return mm_workspace_size(method, n, P, M, levels);
}

int mm_dist_schedule(int method, int64_t P, int64_t M, int32_t levels, int32_t panels, mm_dist_op* ops,
                     int32_t cap) {
  const int n = mmk::build_dist_schedule(method, P, M, levels, panels, ops, cap);
  return n < 0 ? MM_ERR_ARG : n;
}

int mm_dist_step(int method, const mm_dist_op* op, const double* A, const double* B, double* C, int64_t N,
                 int64_t P, int64_t M, int32_t levels, int32_t is_root, void* workspace, size_t ws_bytes,
                 void* stream) {
  if (!op || !B || P < 1 || M < 1 || N < 0 || method < MM_NAIVE || method > MM_WINOGRAD_SCALED_FUSED)
    return MM_ERR_ARG;
  if (N > 0 && (!A || !C)) return MM_ERR_ARG;
  if (!mul_ok(P, M) || (N > 0 && (!mul_ok(N, P) || !mul_ok(N, M)))) return MM_ERR_ARG;
  const size_t need = mm_dist_workspace_size(method, N, P, M, levels);
  if (need > 0 && (!workspace || ws_bytes < need)) return MM_ERR_WORKSPACE;
  int sms = 148;
  int rc = check_device(&sms);
  if (rc) return rc;
  mmk::NvtxRange nvtx("mm_dist_step");
  cudaStream_t st = S(stream);
  const bool scaled = method == MM_WINOGRAD_SCALED || method == MM_WINOGRAD_SCALED_FUSED;
  const bool kahan = method == MM_KAHAN || method == MM_KAHAN_FUSED;
  const bool wino = method == MM_WINOGRAD || method == MM_WINOGRAD_FUSED;
  const bool strassen = method == MM_STRASSEN || method == MM_STRASSEN_WINOGRAD;
  const bool fused = method == MM_KAHAN_FUSED || method == MM_WINOGRAD_FUSED || method == MM_WINOGRAD_SCALED_FUSED;
  char* ws = static_cast<char*>(workspace);
  auto* norms = reinterpret_cast<unsigned long long*>(ws);  // scaled: the (all-reduced) {||A||, ||B||}
  if (op->op == MM_OP_NORMS) {
    if (!scaled) return MM_ERR_ARG;
    cudaError_t e = cudaMemsetAsync(norms, 0, 2 * sizeof(double), st);
    mmk::LineLaunch L{};
    if (N > 0) {
      L.job[L.njobs] = mmk::ln_job(A, P, N, P, true, mmk::LN_ABS);
      L.job[L.njobs++].out_max = norms;
    }
    if (is_root) {
      L.job[L.njobs] = mmk::ln_job(B, M, P, M, true, mmk::LN_ABS);
      L.job[L.njobs++].out_max = norms + 1;
    }
    if (e == cudaSuccess && L.njobs > 0) e = mmk::launch_lines<mmk::LN_ABS>(L, st);
    return cuda_status(e);
  }
  if (N == 0) return MM_OK;  // a rank without rows only contributes to the collectives
  // scaled layout: dist header (norms) | header | y' | z' | 2^lambda A | 2^-lambda B (scaled_ws)
  char* sw = ws + kDistHeader;
  double* ys = reinterpret_cast<double*>(sw + kScaledHeader);
  double* zs = reinterpret_cast<double*>(sw + kScaledHeader + mmk::align256(size_t(N) * 8));
  double* As = reinterpret_cast<double*>(sw + kScaledHeader + winograd_ws(N, M));
  double* Bs =
      reinterpret_cast<double*>(reinterpret_cast<char*>(As) + mmk::align256(size_t(N) * size_t(mmk::scaled_pitch(P)) * 8));
  // Winograd: y | z; Kahan: the carried err E
  double* y = reinterpret_cast<double*>(ws);
  double* z = reinterpret_cast<double*>(ws + mmk::align256(size_t(N) * 8));
  const int64_t lo = op->lo, hi = op->hi;
  switch (op->op) {
    case MM_OP_PANEL: {
      if (lo < 0 || hi > P || lo >= hi || (lo & 1)) return MM_ERR_ARG;
      const bool last = !(op->flags & MM_EX_KEEP_STATE);
      if (method == MM_NAIVE)
        return mm_naive_ex(A + lo, P, B + lo * M, M, C, M, N, hi - lo, M, (op->flags & MM_EX_ACCUMULATE) ? 1 : 0,
                           stream);
      if (!(kahan || wino || scaled)) return MM_ERR_ARG;
      const double* Ao = scaled ? As : A;
      const double* Bo = scaled ? Bs : B;
      if (!mmk::simt_tma_ex_ok(Ao, P, Bo, M, N, P, M)) {
        // this rank's operands cannot take the panel kernels: the one-GPU kernel once B is complete
        if (!last) return MM_OK;
        if (scaled)
          return winograd_scaled_common(fused, A, B, C, N, P, M, reinterpret_cast<const double*>(norms), sw,
                                        ws_bytes - kDistHeader, nullptr, stream);
        return mm_gemm(method, A, B, C, N, P, M, levels, workspace, ws_bytes, nullptr, stream);
      }
      if (kahan)
        return mm_kahan_ex(A + lo, P, B + lo * M, M, C, reinterpret_cast<double*>(ws), N, hi - lo, M, op->flags,
                           stream);
      return mm_winograd_ex(Ao + lo, P, Bo + lo * M, M, C, scaled ? ys : y, scaled ? zs : z, N, hi - lo, M,
                            op->flags, stream);
    }
    case MM_OP_YZ:
      if (!wino) return MM_ERR_ARG;
      if (!mmk::simt_tma_ex_ok(A, P, B, M, N, P, M)) return MM_OK;  // the one-shot kernel makes its own
      return mm_winograd_yz(A, B, N, P, M, y, z, fused ? MM_EX_FUSED : 0, stream);
    case MM_OP_SCALE_A:
      if (!scaled) return MM_ERR_ARG;
      return cuda_status(mmk::launch_scale_rows(A, As, ys, N, P, norms, st, fused));
    case MM_OP_SCALE_B:
      if (!scaled || lo < 0 || hi > P || lo >= hi || (lo & 1)) return MM_ERR_ARG;
      return cuda_status(
          mmk::launch_scale_cols(B, Bs, zs, P, M, lo, hi, (op->flags & MM_EX_ACCUMULATE) != 0, norms, st, fused));
    case MM_OP_FORM_A:
    case MM_OP_FORM_B:
    case MM_OP_FORM_B_REST:
    case MM_OP_LEAF_COMBINE: {
      if (!strassen) return MM_ERR_ARG;
      mmk::StrassenPlan pl;
      if (!mmk::make_strassen_plan(N, P, M, levels, &pl)) return MM_ERR_ARG;
      const int ph = op->op == MM_OP_FORM_A   ? mmk::SP_FORM_A
                     : op->op == MM_OP_FORM_B ? mmk::SP_FORM_B_FIRST
                     : op->op == MM_OP_FORM_B_REST ? mmk::SP_FORM_B_REST
                                                   : mmk::SP_LEAF_COMBINE;
      const int64_t u0 = op->op == MM_OP_FORM_B ? lo : 0, u1 = op->op == MM_OP_FORM_B ? hi : INT64_MAX;
      return cuda_status(method == MM_STRASSEN
                             ? mmk::run_strassen<mmk::SV_NAIV>(A, B, C, N, P, M, pl, ws, sms, st, ph, u0, u1)
                             : mmk::run_strassen<mmk::SV_WINOGRAD>(A, B, C, N, P, M, pl, ws, sms, st, ph, u0, u1));
    }
    case MM_OP_FULL:
      if (scaled)
        return winograd_scaled_common(fused, A, B, C, N, P, M, reinterpret_cast<const double*>(norms), sw,
                                      ws_bytes - kDistHeader, nullptr, stream);
      return mm_gemm(method, A, B, C, N, P, M, levels, workspace, ws_bytes, nullptr, stream);
    default: return MM_ERR_ARG;
  }
}

}  // extern "C"

// The NCCL executor of a schedule: communication ops in list order on the layer's stream (runs of
// broadcasts of one panel, or of point-to-point ops, as one NCCL group), compute ops through
// `step` on the caller's stream, RECORD / WAIT joining the two.
namespace {
bool dist_p2p(int op) { return op == MM_OP_SEND_H || op == MM_OP_RECV_H; }
bool dist_bcast(int op) { return op == MM_OP_BCAST || op == MM_OP_BCAST_A; }
bool dist_same_group(const mm_dist_op& a, const mm_dist_op& b) {
  return (dist_bcast(a.op) && dist_bcast(b.op) && a.index == b.index) || (dist_p2p(a.op) && dist_p2p(b.op));
}

template <class Step>
int run_dist_ops(const mm_dist_op* ops, int n, double* A, int64_t P, double* B, int64_t M, double* ws,
                 int64_t hslot, int32_t root, cudaStream_t st, Step step) {
  mmk::DistState& ds = mmk::dist_state();
  mmk::NcclApi* api = mmk::nccl_api();
  cudaStream_t cs = ds.comm_stream;
  cudaError_t e = cudaEventRecord(ds.start_ev, st);  // buffers may be rewritten once prior work on st is done
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ds.start_ev, 0);
  if (e != cudaSuccess) return cuda_status(e);
  bool grouped = false;
  for (int k = 0; k < n; ++k) {
    const mm_dist_op& o = ops[k];
    cudaStream_t os = o.stream == MM_STREAM_COMM ? cs : st;
    if (dist_bcast(o.op) || dist_p2p(o.op)) {
      const bool more = k + 1 < n && dist_same_group(o, ops[k + 1]);
      if (more && !grouped) {
        if (api->GroupStart() != ncclSuccess) return MM_ERR_NCCL;
        grouped = true;
      }
      ncclResult_t r;
      if (o.op == MM_OP_BCAST) {
        r = api->Broadcast(B + o.lo * M, B + o.lo * M, size_t(o.hi - o.lo) * size_t(M), ncclFloat64, root, ds.comm, cs);
      } else if (o.op == MM_OP_BCAST_A) {
        r = A ? api->Broadcast(A + o.lo * P, A + o.lo * P, size_t(o.hi - o.lo) * size_t(P), ncclFloat64, root, ds.comm,
                               cs)
              : ncclInvalidArgument;
      } else if (o.op == MM_OP_SEND_H) {
        r = api->Send(ws + o.index * hslot, size_t(hslot), ncclFloat64, int(o.lo), ds.comm, cs);
      } else {
        r = api->Recv(ws + o.index * hslot, size_t(hslot), ncclFloat64, int(o.lo), ds.comm, cs);
      }
      if (r != ncclSuccess) {
        if (grouped) api->GroupEnd();  // leave no NCCL group open behind the error
        return MM_ERR_NCCL;
      }
      if (grouped && !more) {
        if (api->GroupEnd() != ncclSuccess) return MM_ERR_NCCL;
        grouped = false;
      }
      continue;
    }
    switch (o.op) {
      case MM_OP_ALLREDUCE_NORMS:
        if (api->AllReduce(ws, ws, 2, ncclFloat64, ncclMax, ds.comm, cs) != ncclSuccess) return MM_ERR_NCCL;
        break;
      case MM_OP_RECORD:
        if ((e = cudaEventRecord(ds.panel_ev[o.index], os)) != cudaSuccess) return cuda_status(e);
        break;
      case MM_OP_WAIT:
        if ((e = cudaStreamWaitEvent(os, ds.panel_ev[o.index], 0)) != cudaSuccess) return cuda_status(e);
        break;
      default: {
        const int rc = step(o);
        if (rc) return rc;
      }
    }
  }
  // the caller's stream continues after every communication op of the product
  if ((e = cudaEventRecord(ds.end_ev, cs)) == cudaSuccess) e = cudaStreamWaitEvent(st, ds.end_ev, 0);
  return cuda_status(e);
}
}  // namespace

extern "C" {

int mm_dist_gemm(int method, const double* A_shard, double* B, double* C_shard, int64_t N_local, int64_t P,
                 int64_t M, int32_t root, int32_t levels, int32_t panels, void* workspace, size_t ws_bytes,
                 void* stream) {
  mmk::NvtxRange nvtx("mm_dist_gemm");
  mmk::DistState& ds = mmk::dist_state();
  if (!ds.comm || !B || P < 1 || M < 1 || N_local < 0 || root < 0 || root >= ds.world) return MM_ERR_ARG;
  if (N_local > 0 && (!A_shard || !C_shard)) return MM_ERR_ARG;
  if (!mul_ok(P, M) || (N_local > 0 && (!mul_ok(N_local, P) || !mul_ok(N_local, M)))) return MM_ERR_ARG;
  const size_t need = mm_dist_workspace_size(method, N_local, P, M, levels);
  if (need > 0 && (!workspace || ws_bytes < need)) return MM_ERR_WORKSPACE;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != ds.device) return MM_ERR_ARG;
  // the schedule depends only on (method, P, M, levels, panels): every rank issues the same collectives
  static thread_local mm_dist_op ops[1024];
  const int n = mmk::build_dist_schedule(method, P, M, levels, panels, ops, 1024);
  if (n < 0) return MM_ERR_ARG;
  return run_dist_ops(ops, n, nullptr, P, B, M, static_cast<double*>(workspace), 0, root, S(stream),
                      [&](const mm_dist_op& o) {
                        return mm_dist_step(method, &o, A_shard, B, C_shard, N_local, P, M, levels,
                                            ds.rank == root ? 1 : 0, workspace, ws_bytes, stream);
                      });
}

}  // extern "C"

// ---------------------------------------------------------------- the alternative partition (S7)
namespace {
struct S7Layout {
  mmk::StrassenPlan pl, sub;
  int64_t h2, p2, m2, hslot;     // level-1 node dims, doubles per H slot
  size_t offL, offR, offSub, total;
};

bool s7_layout(int method, int64_t N, int64_t P, int64_t M, int32_t levels, S7Layout* o) {
  if (method != MM_STRASSEN && method != MM_STRASSEN_WINOGRAD) return false;
  if (levels < 1 || N < 1 || P < 1 || M < 1 || !mul_ok(N, P) || !mul_ok(P, M) || !mul_ok(N, M)) return false;
  if (!mmk::make_strassen_plan(N, P, M, levels, &o->pl)) return false;
  o->h2 = o->pl.Np / 2;
  o->p2 = o->pl.Pp / 2;
  o->m2 = o->pl.Mp / 2;
  // the level-1 node recursed on with levels - 1 levels: its plan pads nothing (R10)
  if (!mmk::make_strassen_plan(o->h2, o->p2, o->m2, levels - 1, &o->sub)) return false;
  if (o->sub.Np != o->h2 || o->sub.Pp != o->p2 || o->sub.Mp != o->m2) return false;
  o->hslot = o->h2 * o->m2;
  o->offL = mmk::align256(size_t(7) * size_t(o->hslot) * 8);
  o->offR = mmk::align256(o->offL + size_t(o->h2) * size_t(o->p2) * 8);
  o->offSub = mmk::align256(o->offR + size_t(o->p2) * size_t(o->m2) * 8);
  o->total = o->offSub + o->sub.total;
  return true;
}
}  // namespace

extern "C" {

size_t mm_s7_workspace_size(int method, int64_t N, int64_t P, int64_t M, int32_t levels) {
  S7Layout l;
  return s7_layout(method, N, P, M, levels, &l) ? l.total : 0;
}

int mm_s7_schedule(int method, int64_t N, int64_t P, int64_t M, int32_t levels, int32_t world, int32_t rank,
                   int32_t root, mm_dist_op* ops, int32_t cap) {
  const int n = mmk::build_s7_schedule(method, N, P, M, levels, world, rank, root, ops, cap);
  return n < 0 ? MM_ERR_ARG : n;
}

int mm_s7_step(int method, const mm_dist_op* op, const double* A, const double* B, double* C, int64_t N, int64_t P,
               int64_t M, int32_t levels, void* workspace, size_t ws_bytes, void* stream) {
  S7Layout l;
  if (!op || !A || !B || !s7_layout(method, N, P, M, levels, &l)) return MM_ERR_ARG;
  if (!workspace || ws_bytes < l.total) return MM_ERR_WORKSPACE;
  if (overlaps(workspace, int64_t(l.total / 8), A, N * P) || overlaps(workspace, int64_t(l.total / 8), B, P * M))
    return MM_ERR_ALIAS;
  int sms = 148;
  int rc = check_device(&sms);
  if (rc) return rc;
  mmk::NvtxRange nvtx("mm_s7_step");
  cudaStream_t st = S(stream);
  char* ws = static_cast<char*>(workspace);
  double* Hs = reinterpret_cast<double*>(ws);
  double* L = reinterpret_cast<double*>(ws + l.offL);
  double* R = reinterpret_cast<double*>(ws + l.offR);
  const bool naiv = method == MM_STRASSEN;
  const int p = op->index;
  switch (op->op) {
    case MM_OP_S7_FORM: {  // child p of the zero-embedded level-0 quadrants, both sides
      if (p < 0 || p > 6) return MM_ERR_ARG;
      for (int side = 0; side < 2; ++side) {
        mmk::FormArgs fa;
        fa.src = side == 0 ? A : B;
        fa.src_pitch = side == 0 ? P : M;
        fa.src_stride = 0;
        fa.rows_valid = side == 0 ? N : P;
        fa.cols_valid = side == 0 ? P : M;
        fa.dst = side == 0 ? L : R;
        fa.h_rows = side == 0 ? l.h2 : l.p2;
        fa.h_cols = side == 0 ? l.p2 : l.m2;
        fa.cnt = 1;
        fa.u0 = 0;
        fa.u1 = fa.h_rows;
        const int v = mmk::pick_vec(fa.src, fa.dst, fa.src_pitch, fa.src_stride, fa.h_cols);
        const cudaError_t e = naiv ? mmk::launch_form_child<mmk::SV_NAIV>(side, fa, p, v, sms, st)
                                   : mmk::launch_form_child<mmk::SV_WINOGRAD>(side, fa, p, v, sms, st);
        if (e != cudaSuccess) return cuda_status(e);
      }
      return MM_OK;
    }
    case MM_OP_S7_PRODUCT: {  // H_{p+1} with the remaining levels - 1 levels (the one-GPU recursion)
      if (p < 0 || p > 6) return MM_ERR_ARG;
      double* H = Hs + p * l.hslot;
      char* sw = ws + l.offSub;
      return cuda_status(naiv ? mmk::run_strassen<mmk::SV_NAIV>(L, R, H, l.h2, l.p2, l.m2, l.sub, sw, sms, st)
                              : mmk::run_strassen<mmk::SV_WINOGRAD>(L, R, H, l.h2, l.p2, l.m2, l.sub, sw, sms, st));
    }
    case MM_OP_S7_COMBINE: {  // the level-0 combination into C, dropping the padding
      if (!C) return MM_ERR_ARG;
      if (overlaps(C, N * M, A, N * P) || overlaps(C, N * M, B, P * M) ||
          overlaps(C, N * M, workspace, int64_t(l.total / 8)))
        return MM_ERR_ALIAS;
      mmk::CombineArgs ca;
      ca.H = Hs;
      ca.dst = C;
      ca.dst_pitch = M;
      ca.dst_stride = 0;
      ca.rows_valid = N;
      ca.cols_valid = M;
      ca.h_rows = l.h2;
      ca.h_cols = l.m2;
      ca.cnt = 1;
      const int v = mmk::pick_vec(ca.dst, ca.H, ca.dst_pitch, ca.dst_stride, ca.h_cols);
      return cuda_status(naiv ? mmk::launch_combine_level<mmk::SV_NAIV>(ca, v, sms, st)
                              : mmk::launch_combine_level<mmk::SV_WINOGRAD>(ca, v, sms, st));
    }
    default: return MM_ERR_ARG;
  }
}

int mm_dist_strassen7(int method, double* A, double* B, double* C, int64_t N, int64_t P, int64_t M, int32_t root,
                      int32_t levels, void* workspace, size_t ws_bytes, void* stream) {
  mmk::NvtxRange nvtx("mm_dist_strassen7");
  mmk::DistState& ds = mmk::dist_state();
  S7Layout l;
  if (!ds.comm || !A || !B || root < 0 || root >= ds.world || !s7_layout(method, N, P, M, levels, &l))
    return MM_ERR_ARG;
  if (ds.rank == root && !C) return MM_ERR_ARG;
  if (!workspace || ws_bytes < l.total) return MM_ERR_WORKSPACE;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != ds.device) return MM_ERR_ARG;
  mm_dist_op ops[64];
  const int n = mmk::build_s7_schedule(method, N, P, M, levels, ds.world, ds.rank, root, ops, 64);
  if (n < 0) return MM_ERR_ARG;
  return run_dist_ops(ops, n, A, P, B, M, static_cast<double*>(workspace), l.hslot, root, S(stream),
                      [&](const mm_dist_op& o) {
                        return mm_s7_step(method, &o, A, B, C, N, P, M, levels, workspace, ws_bytes, stream);
                      });
}

int norm_inf(const double* X, int64_t rows, int64_t cols, double* out_device, void* stream) {
  if (!X || !out_device || rows < 1 || cols < 1 || !mul_ok(rows, cols)) return MM_ERR_ARG;
  int rc = check_device(nullptr);
  if (rc) return rc;
  return cuda_status(
      mmk::launch_norm_inf(X, rows, cols, reinterpret_cast<unsigned long long*>(out_device), S(stream)));
}

}  // extern "C"
