// repack.cuh -- an odd-pitch operand copied to an even pitch (a pure copy, no arithmetic).
//
// A tiled TMA box must start on a 16-byte boundary (tools/probes/tma_probe.cu), so the rows of a
// row-major float64 matrix with an odd number of columns -- every other row starting 8 bytes off --
// cannot be streamed by TMA.  When the caller provides the workspace (mm_gemm /
// mm_workspace_size for MM_NAIVE, MM_KAHAN[_FUSED], MM_WINOGRAD[_FUSED] with odd P), A is first
// copied to pitch P + 1 (one HBM pass over A: 2 N P 8 bytes, ~0.01 ms at c3) and the TMA-fed
// kernels run on the copy; the copy holds the same doubles, so every result is bitwise the
// cp.async kernels'.  (WinogradScaled's 2^lambda A copy gets the even pitch directly.)
#pragma once
#include "common.cuh"

namespace mmk {

__global__ void __launch_bounds__(256) repack_rows_kernel(const double* __restrict__ src, int64_t lds,
                                                          double* __restrict__ dst, int64_t ldd, int64_t rows,
                                                          int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    dst[r * ldd + c] = __ldg(src + r * lds + c);
  }
}

inline cudaError_t launch_repack_rows(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                                      int64_t cols, int sms, cudaStream_t st) {
  int64_t blocks = cdiv(rows * cols, int64_t(256));
  const int64_t cap = int64_t(sms) * 8;
  if (blocks > cap) blocks = cap;
  repack_rows_kernel<<<unsigned(blocks < 1 ? 1 : blocks), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  note_launch();
  return cudaGetLastError();
}

}  // namespace mmk
