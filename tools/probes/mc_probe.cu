// mc_probe.cu -- does this B200 offer NVLink SHARP multicast (NVLS) to one process, and what does a
// multimem store stream cost?  Probe for SURVEY 8(f)4 "NVLS/multicast broadcast".
//
// 1. device attributes: MULTICAST_SUPPORTED, POSIX-fd and fabric handle export;
// 2. a one-device multicast object: create, add the device, bind a cuMemCreate allocation, map the
//    multicast handle and the allocation into two VA ranges;
// 3. a kernel that streams a source buffer into the multicast VA with multimem.st.global.v4.f32
//    (the root's side of a multicast broadcast); the unicast VA must read back the same doubles;
// 4. a release-ordered flag written with multimem.red after the data, observed through the unicast
//    VA by cuStreamWaitValue32 (the receivers' side of a panel-arrival signal).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_probe mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    CUresult r_ = (x);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                  \
      const char* s_ = nullptr;                                                \
      cuGetErrorString(r_, &s_);                                               \
      printf("{\"step\":\"%s\",\"error\":\"%s\"}\n", #x, s_ ? s_ : "?");       \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void mc_store(const double* __restrict__ src, double* mc, int64_t n2) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += int64_t(gridDim.x) * blockDim.x) {
    // 16 bytes per store; multimem.st has no .v2.f64 form, and a store only moves bits
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 2 * i), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
  }
}

__global__ void uc_copy(const double* __restrict__ src, double* dst, int64_t n2) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += int64_t(gridDim.x) * blockDim.x)
    reinterpret_cast<double2*>(dst)[i] = reinterpret_cast<const double2*>(src)[i];
}

__global__ void mc_flag(unsigned* mc_flag_ptr, unsigned v) {
  asm volatile("fence.proxy.alias;" ::: "memory");
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_flag_ptr), "r"(v) : "memory");
}

__global__ void fill(double* x, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] = double(i % 1000003) * 0.5 - 7.25;
}

__global__ void cmp(const double* a, const double* b, int64_t n, unsigned long long* bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    if (a[i] != b[i]) atomicAdd(bad, 1ull);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8192ll * 8192;  // doubles (c4's B)
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mc = 0, fd = 0, fab = 0, sms = 0;
  CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  printf("{\"multicast_supported\":%d,\"posix_fd\":%d,\"fabric\":%d,\"sms\":%d}\n", mc, fd, fab, sms);
  fflush(stdout);
  cudaSetDevice(0);
  cudaFree(0);  // primary context
  if (!mc) return 0;

  const size_t bytes_data = size_t(n) * 8, bytes = bytes_data + 4096;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  size_t gmc = 0, gmin = 0;
  CK(cuMulticastGetGranularity(&gmc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CK(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gmem = 0;
  CK(cuMemGetAllocationGranularity(&gmem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  size_t g = gmc > gmem ? gmc : gmem;
  const size_t size = (bytes + g - 1) / g * g;
  mp.size = size;
  printf("{\"mc_granularity\":%zu,\"mc_min_granularity\":%zu,\"mem_granularity\":%zu,\"size\":%zu}\n", gmc, gmin, gmem,
         size);
  fflush(stdout);

  // which (devices, handle types, size) does cuMulticastCreate accept on this node?
  int ok_types = -1;
  for (int nd = 1; nd <= 2; ++nd)
    for (int ht : {int(CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), int(CU_MEM_HANDLE_TYPE_FABRIC), 0,
                   int(CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR | CU_MEM_HANDLE_TYPE_FABRIC)})
      for (size_t sz : {size_t(2) << 20, size}) {
        CUmulticastObjectProp q = {};
        q.numDevices = nd;
        q.handleTypes = ht;
        q.size = sz;
        CUmemGenericAllocationHandle h;
        CUresult r = cuMulticastCreate(&h, &q);
        const char* es = nullptr;
        cuGetErrorString(r, &es);
        printf("{\"mc_create\":{\"devices\":%d,\"handle_types\":%d,\"size\":%zu},\"result\":\"%s\"}\n", nd, ht, sz,
               es ? es : "?");
        if (r == CUDA_SUCCESS) {
          if (nd == 1 && sz == size && ok_types < 0) ok_types = ht;
          cuMemRelease(h);
        }
      }
  fflush(stdout);
  if (ok_types < 0) return 0;
  mp.handleTypes = CUmemAllocationHandleType(ok_types);
  ap.requestedHandleTypes = CUmemAllocationHandleType(ok_types);

  CUmemGenericAllocationHandle mch, memh;
  CK(cuMulticastCreate(&mch, &mp));
  CK(cuMulticastAddDevice(mch, dev));
  CK(cuMemCreate(&memh, size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, memh, 0, size, 0));
  CUdeviceptr uc = 0, mcp = 0;
  CK(cuMemAddressReserve(&uc, size, g, 0, 0));
  CK(cuMemMap(uc, size, 0, memh, 0));
  CK(cuMemAddressReserve(&mcp, size, g, 0, 0));
  CK(cuMemMap(mcp, size, 0, mch, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, size, &ad, 1));
  CK(cuMemSetAccess(mcp, size, &ad, 1));

  double* src;
  unsigned long long* bad;
  cudaMalloc(&src, bytes_data);
  cudaMalloc(&bad, 8);
  fill<<<sms * 4, 256>>>(src, n);
  cudaMemset(reinterpret_cast<void*>(uc), 0, size);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int64_t n2 = n / 2;
  double* ucd = reinterpret_cast<double*>(uc);
  double* mcd = reinterpret_cast<double*>(mcp);
  unsigned* uflag = reinterpret_cast<unsigned*>(uc + bytes_data);
  unsigned* mflag = reinterpret_cast<unsigned*>(mcp + bytes_data);

  mc_store<<<sms * 8, 256, 0, st>>>(src, mcd, n2);
  mc_flag<<<1, 1, 0, st>>>(mflag, 1);
  cudaStream_t st2;
  cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
  CK(cuStreamWaitValue32(reinterpret_cast<CUstream>(st2), uc + bytes_data, 1, CU_STREAM_WAIT_VALUE_GEQ));
  cudaMemsetAsync(bad, 0, 8, st2);
  cmp<<<sms * 4, 256, 0, st2>>>(src, ucd, n, bad);
  unsigned long long nb = ~0ull;
  cudaMemcpyAsync(&nb, bad, 8, cudaMemcpyDeviceToHost, st2);
  cudaStreamSynchronize(st2);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned fl = 0;
  cudaMemcpy(&fl, uflag, 4, cudaMemcpyDeviceToHost);
  printf("{\"multimem_store_mismatch\":%llu,\"flag\":%u,\"err\":\"%s\"}\n", nb, fl, cudaGetErrorString(e));
  fflush(stdout);

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    for (int w = 0; w < 3; ++w)
      mode ? uc_copy<<<sms * 8, 256, 0, st>>>(src, ucd, n2) : mc_store<<<sms * 8, 256, 0, st>>>(src, mcd, n2);
    cudaEventRecord(e0, st);
    const int reps = 10;
    for (int r = 0; r < reps; ++r)
      mode ? uc_copy<<<sms * 8, 256, 0, st>>>(src, ucd, n2) : mc_store<<<sms * 8, 256, 0, st>>>(src, mcd, n2);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("{\"kernel\":\"%s\",\"bytes\":%zu,\"ms\":%.4f,\"GBps_read_plus_write\":%.1f,\"err\":\"%s\"}\n",
           mode ? "unicast_copy" : "multimem_st_v4_f32", bytes_data, ms, 2.0 * bytes_data / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  CK(cuMemUnmap(mcp, size));
  CK(cuMemUnmap(uc, size));
  CK(cuMulticastUnbind(mch, dev, 0, size));
  CK(cuMemRelease(memh));
  CK(cuMemRelease(mch));
  CK(cuMemAddressFree(mcp, size));
  CK(cuMemAddressFree(uc, size));
  printf("{\"done\":true}\n");
  return 0;
}
