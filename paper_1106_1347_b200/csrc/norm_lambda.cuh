// norm_lambda.cuh -- K4 norm_inf and K5 the lambda rule.
//
// K4: ||X||_inf = max_i sum_j |X_ij|.  One lane owns one row and sums it left to right (the
// oracle's order, so the row sums -- and hence lambda -- are bit-identical to the CPU oracle);
// rows are streamed through the bulk-copy line ring of lines.cuh.  The max over rows is
// order-free: each warp reduces its 32 rows and issues one atomicMax on the IEEE bit pattern
// (non-negative doubles order like their uint64 images).  HBM-bound: 8 rows cols bytes read.
//
// K5: lambda with 1/2 <= 2^(2 lambda) nA / nB <= 2 (lambda_rule in lines.cuh: exact, from
// frexp; reading R7).  It is evaluated on the device by every block of the fused
// scale + y/z pass (winograd.cuh), which reads the two norms K4 left in device memory --
// no host round trip and no separate launch.
#pragma once
#include "lines.cuh"

namespace mmk {

// out: device uint64 slot, zeroed here then max-reduced
inline cudaError_t launch_norm_inf(const double* X, int64_t rows, int64_t cols, unsigned long long* out,
                                   cudaStream_t st) {
  return launch_norms(X, rows, cols, nullptr, 0, 0, out, st);
}

}  // namespace mmk
