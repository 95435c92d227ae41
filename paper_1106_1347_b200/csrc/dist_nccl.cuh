// dist_nccl.cuh -- K9, the multi-GPU row-block layer behind the C ABI.
//
// C = A B split by row blocks: rank r owns rows of A and C, B is broadcast from `root` inside
// every product -- the one real exchange of the path.  NCCL (over NVLink 5 / NVSwitch) is loaded
// at run time with dlopen (the soname libnccl.so.2, already resident when PyTorch initialised
// NCCL, else the path in MM_NCCL_LIBRARY), so the rest of the library has no NCCL dependency.
//
//  * NaivStandard with panels > 1: B is broadcast as consecutive row panels
//    on a dedicated communication stream, one event per panel; the caller's stream waits for
//    panel i only before mm_naive_ex(accumulate) multiplies it, so panel i+1 crosses NVLink while
//    panel i is on the tensor cores.  Every entry's DMMA chain continues from C in k order
//    (reading R23): bitwise the one-shot product.
//  * WinogradScaled: the rank's ||A_r||_inf (K4) is max-all-reduced (8 bytes) into the global
//    ||A||_inf; ||B||_inf is local (B is replicated), so lambda equals the 1-GPU lambda.
//  * the other methods: broadcast on the caller's stream, then the single-GPU entry point.  Per
//    entry arithmetic depends only on (row of A, column of B, P), so the shards are bitwise the
//    rows of the 1-GPU product (Strassen recurses on the shard: within its tolerance only).
#pragma once
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; every function is resolved with dlsym

#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace mmk {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

inline NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* p = std::getenv("MM_NCCL_LIBRARY");
      if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    if (api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.AllReduce && api.GroupStart &&
        api.GroupEnd)
      api.handle = h;
  });
  return api.handle ? &api : nullptr;
}

struct DistState {
  ncclComm_t comm = nullptr;
  int rank = -1, world = 0, device = -1;
  cudaStream_t comm_stream = nullptr;
  static constexpr int kMaxPanels = 64;
  cudaEvent_t panel_ev[kMaxPanels] = {};
  cudaEvent_t start_ev = nullptr;
};

inline DistState& dist_state() {
  static DistState s;
  return s;
}

// consecutive k-panels [k0, k1) covering 0..P with even boundaries (16-byte aligned views; the
// same rule as paper_1106_1347_b200.dist.panel_bounds)
inline int dist_panel_bounds(int64_t P, int panels, int64_t* bounds) {
  if (panels < 1) panels = 1;
  if (panels > DistState::kMaxPanels) panels = DistState::kMaxPanels;
  if (panels > P) panels = int(P);
  int n = 0;
  bounds[n++] = 0;
  for (int i = 1; i < panels; ++i) {
    const int64_t c = 2 * ((P * i) / (2 * int64_t(panels)));
    if (c > bounds[n - 1] && c < P) bounds[n++] = c;
  }
  bounds[n++] = P;
  return n - 1;
}

}  // namespace mmk
