// Stream-write probe: is strassen_form3_kernel's 5.25 TB/s (0.537 GB read + 2.82 GB written) set
// by its access pattern -- every position writes one value into each of 343 arrays -- rather than
// by its arithmetic?  Times, on 2.82 GB of output:
//   seq      : contiguous 16-byte stores (grid-stride), the write ceiling
//   streams S: form3's layout without arithmetic, S arrays of 2.82 GB / S, one row unit of 128
//              consecutive positions per 128-thread CTA, each position writing its S values
//              (V = 1: 8-byte stores as form3; V = 2: 16-byte stores, two positions per thread)
//   form3pat : form3's full pattern with trivial arithmetic -- 64 reads per position from the
//              8 x 8 sub-block grid of a 8192 x 8192 parent, 343 writes
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_write_probe stream_write_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void seq_kernel(double2* p, int64_t n2) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = make_double2(double(i), 1.0);
}

// rows x cols per array, S arrays; CTA = 128 threads over one row of `cols` positions
template <int V>
__global__ void __launch_bounds__(128) streams_kernel(double* dst, int S, int64_t rows, int64_t cols) {
  const int64_t gelems = rows * cols;
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
    for (int64_t j = int64_t(threadIdx.x) * V; j < cols; j += 128 * V) {
      double* p = dst + i * cols + j;
      const double v = double(i + j);
#pragma unroll 1
      for (int t0 = 0; t0 < S; t0 += 7) {
#pragma unroll
        for (int t = 0; t < 7; ++t) {
          if (V == 2)
            *reinterpret_cast<double2*>(p) = make_double2(v + t, v - t);
          else
            *p = v + t;
          p += gelems;
        }
      }
    }
  }
}

// form3's memory pattern: parent 8h x 8h (pitch 8h), 64 loads per position, 343 stores
__global__ void __launch_bounds__(128) form3pat_kernel(const double* src, double* dst, int64_t h) {
  extern __shared__ double xs_all[];
  double* xs = xs_all + threadIdx.x;
  const int64_t gelems = h * h, pitch = 8 * h;
  for (int64_t i = blockIdx.x; i < h; i += gridDim.x) {
    for (int64_t j = threadIdx.x; j < h; j += 128) {
#pragma unroll 1
      for (int pr0 = 0; pr0 < 8; pr0 += 2) {
        double v[16];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int pc = 0; pc < 8; ++pc) v[r * 8 + pc] = __ldg(src + (i + (pr0 + r) * h) * pitch + j + pc * h);
#pragma unroll
        for (int k = 0; k < 16; ++k) xs[(pr0 * 8 + k) * 128] = v[k];
      }
      const volatile double* xv = xs;
      double* p = dst + i * h + j;
#pragma unroll 1
      for (int c = 0; c < 49; ++c) {
        const double a = xv[(c & 63) * 128], b = xv[((c * 5) & 63) * 128];
#pragma unroll
        for (int t = 0; t < 7; ++t) {
          *p = a + b * t;
          p += gelems;
        }
      }
    }
  }
}

__device__ __forceinline__ unsigned su32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

// form3pat with the 64 inputs of a block of NT positions staged by 1-D bulk copies (one per
// sub-block row segment, NT * 8 bytes) into an NST-deep ring, issued NST blocks ahead
template <int NT, int NST>
__global__ void __launch_bounds__(NT) form3bulk_kernel(const double* src, double* dst, int64_t h) {
  extern __shared__ __align__(16) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * 64 * NT);
  const int64_t gelems = h * h, pitch = 8 * h, bpr = h / NT, nblk = h * bpr;
  auto issue = [&](int s, int64_t b) {
    const int64_t i = b / bpr, j0 = (b - i * bpr) * NT;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])), "r"(64 * NT * 8)
                 : "memory");
    for (int k = 0; k < 64; ++k) {
      const double* g = src + (i + (k >> 3) * h) * pitch + j0 + (k & 7) * h;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              su32(sm + (s * 64 + k) * NT)),
          "l"(g), "r"(NT * 8), "r"(su32(&full[s]))
          : "memory");
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < NST; ++s)
      if (blockIdx.x + int64_t(s) * gridDim.x < nblk) issue(s, blockIdx.x + int64_t(s) * gridDim.x);
  int it = 0;
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x, ++it) {
    const int s = it % NST;
    const unsigned par = (it / NST) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
            su32(&full[s])),
        "r"(par)
        : "memory");
    const int64_t i = b / bpr, j = (b - i * bpr) * NT + threadIdx.x;
    const volatile double* xv = sm + s * 64 * NT + threadIdx.x;
    double* p = dst + i * h + j;
#pragma unroll 1
    for (int c = 0; c < 49; ++c) {
      const double a = xv[(c & 63) * NT], bb = xv[((c * 5) & 63) * NT];
#pragma unroll
      for (int t = 0; t < 7; ++t) {
        *p = a + bb * t;
        p += gelems;
      }
    }
    __syncthreads();
    const int64_t nb = b + int64_t(NST) * gridDim.x;
    if (threadIdx.x == 0 && nb < nblk) issue(s, nb);
  }
}

template <class F>
float time_ms(F f, int reps = 10) {
  f();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t h = 1024, total = 343 * h * h;  // doubles written: 2.82 GB
  double *dst, *src;
  cudaMalloc(&dst, total * 8);
  cudaMalloc(&src, 64 * h * h * 8);
  cudaMemset(src, 0, 64 * h * h * 8);
  const double gb = total * 8 / 1e9;
  for (int mult : {4, 8, 16}) {
    float ms = time_ms([&] { seq_kernel<<<sms * mult, 256>>>(reinterpret_cast<double2*>(dst), total / 2); });
    printf("{\"kernel\": \"seq\", \"grid\": %d, \"ms\": %.4f, \"GBps\": %.0f}\n", sms * mult, ms, gb / ms * 1e3);
  }
  for (int S : {7, 49, 343}) {
    const int64_t rows = total / S / h;  // arrays of rows x 1024
    for (int ctas : {3, 6, 12}) {
      float ms1 = time_ms([&] { streams_kernel<1><<<sms * ctas, 128>>>(dst, S, rows, h); });
      float ms2 = time_ms([&] { streams_kernel<2><<<sms * ctas, 128>>>(dst, S, rows, h); });
      printf("{\"kernel\": \"streams\", \"S\": %d, \"ctas_per_sm\": %d, \"V1_ms\": %.4f, \"V1_GBps\": %.0f, "
             "\"V2_ms\": %.4f, \"V2_GBps\": %.0f}\n",
             S, ctas, ms1, gb / ms1 * 1e3, ms2, gb / ms2 * 1e3);
    }
  }
  const size_t smem = 64 * 128 * 8;
  cudaFuncSetAttribute(form3pat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int ctas : {3}) {
    float ms = time_ms([&] { form3pat_kernel<<<sms * ctas, 128, smem>>>(src, dst, h); });
    const double tot = gb + 64 * h * h * 8 / 1e9;
    printf("{\"kernel\": \"form3pat\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps_total\": %.0f}\n", ctas, ms,
           tot / ms * 1e3);
  }
  auto bulk = [&](auto kern, int nt, int nst, int ctas) {
    const size_t sm = size_t(nst) * 64 * nt * 8 + 64;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    float ms = time_ms([&] { kern<<<sms * ctas, nt, sm>>>(src, dst, h); });
    const double tot = gb + 64 * h * h * 8 / 1e9;
    printf("{\"kernel\": \"form3bulk\", \"NT\": %d, \"NST\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, "
           "\"GBps_total\": %.0f, \"err\": \"%s\"}\n", nt, nst, ctas, ms, tot / ms * 1e3,
           cudaGetErrorString(cudaGetLastError()));
  };
  bulk(form3bulk_kernel<64, 2>, 64, 2, 3);
  bulk(form3bulk_kernel<64, 3>, 64, 3, 2);
  bulk(form3bulk_kernel<64, 2>, 64, 2, 2);
  bulk(form3bulk_kernel<128, 1>, 128, 1, 3);
  bulk(form3bulk_kernel<128, 2>, 128, 2, 1);
  bulk(form3bulk_kernel<32, 3>, 32, 3, 4);
  bulk(form3bulk_kernel<32, 2>, 32, 2, 6);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
