// host_pipeline.cuh -- mm_methods_host: the paper's test program from HOST memory
// through the C ABI -- several methods applied to the same host operands, A and B copied to the
// device once, every product copied back while the next one computes.  Included by mm_abi.cu
// (which defines mm_gemm / mm_naive_ex / mm_workspace_size used here); no arithmetic on matrix
// data happens here, only copies, events and calls of the entry points.
//
// Pipeline (two library-owned copy streams per device, the caller's stream for the kernels):
//  * first method NaivStandard: A's column panels and B's row panels travel in k-panels of growing
//    width (x1.4: each copy hides under the previous panel's DMMA work) and the product accumulates
//    panel by panel as they land (mm_naive_ex accumulate, reading R23: bitwise the one-shot chain);
//  * first method another row-local one (NaivKahan, WinogradOriginal, fused variants): B first, then
//    A in row blocks, each block's product starting as its rows land;
//  * every product goes back on the output copy stream while the next method computes (two device
//    product buffers alternate); a row-local LAST method runs in row blocks of halving height so only
//    the smallest block's copy follows the last kernel.
#pragma once
#include <cuda_runtime.h>

#include <vector>

namespace mmk {

inline bool host_row_local(int m) {
  return m == MM_NAIVE || m == MM_KAHAN || m == MM_WINOGRAD || m == MM_KAHAN_FUSED || m == MM_WINOGRAD_FUSED;
}

struct HostStreams {
  cudaStream_t in = nullptr, out = nullptr;
};

inline HostStreams* host_streams() {
  constexpr int kMaxDev = 64;
  static HostStreams s[kMaxDev];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (!s[dev].in) {
    if (cudaStreamCreateWithFlags(&s[dev].in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s[dev].out, cudaStreamNonBlocking) != cudaSuccess)
      return nullptr;
  }
  return &s[dev];
}

// consecutive k-panels of P, even boundaries, widths growing by `ratio`
inline std::vector<int64_t> host_growing_panels(int64_t P, int n, double ratio = 1.4) {
  if (n < 1) n = 1;
  if (P >= 2 && n > P / 2) n = int(P / 2);
  if (P < 2) n = 1;
  std::vector<double> w(n);
  double tot = 0, x = 1;
  for (int i = 0; i < n; ++i, x *= ratio) tot += (w[i] = x);
  std::vector<int64_t> b{0};
  double acc = 0;
  for (int i = 0; i + 1 < n; ++i) {
    acc += w[i];
    const int64_t c = 2 * int64_t(P * acc / tot / 2 + 0.5);
    if (c > b.back() && c < P) b.push_back(c);
  }
  b.push_back(P);
  return b;
}

// at most n row blocks of N halving in size (multiples of 64 rows, none below min_rows)
inline std::vector<int64_t> host_shrinking_rows(int64_t N, int n, int64_t min_rows = 1024) {
  std::vector<int64_t> b{0};
  if (n > 1 && N >= 2 * min_rows) {
    int64_t rest = N;
    for (int i = 0; i + 1 < n; ++i) {
      int64_t sz = (rest / 2) / 64 * 64;
      if (sz < 64) sz = 64;
      if (rest - sz < min_rows) break;
      b.push_back(b.back() + sz);
      rest -= sz;
    }
  }
  b.push_back(N);
  return b;
}

}  // namespace mmk
