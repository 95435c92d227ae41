// dist_nccl.cuh -- K9, the multi-GPU row-block layer behind the C ABI.
//
// C = A B split by row blocks: rank r owns rows of A and C, B is broadcast from `root` inside
// every product -- the one real exchange of the path.  NCCL (over NVLink 5 / NVSwitch) is loaded
// at run time with dlopen (the soname libnccl.so.2, already resident when PyTorch initialised
// NCCL, else the path in MM_NCCL_LIBRARY), so the rest of the library has no NCCL dependency.
//
// ONE schedule (build_dist_schedule, exported as mm_dist_schedule) describes a product as a list
// of communication ops (broadcasts of row ranges of B, the max-all-reduce of the norms) and
// compute ops (mm_dist_step), joined by record / wait events.  mm_dist_gemm executes it with NCCL
// on the layer's stream; the torch.distributed driver (dist.py) executes the same list over
// NCCL or gloo -- which is how the schedule is tested with two ranks on CPU.  It is a function of
// (method, P, M, levels, panels) only, values every rank shares, so all ranks issue the same
// collectives whatever their shard (per-rank eligibility must not change them).
//
//  * panel methods: B crosses NVLink as row panels while the previous panel
//    is multiplied; every entry's running state (DMMA chain / Kahan (sum, err) / Winograd pair
//    sum) continues from panel to panel in k order, so the shard is bitwise the one-shot product.
//  * WinogradScaled: {||A_r||, ||B|| on the root} are max-all-reduced BEFORE B moves (the root
//    holds B), so lambda -- equal to the 1-GPU lambda -- is known at once; each arriving panel of
//    B is scaled (z' continued) and its pair sums accumulated on the scaled copies.
//  * Strassen: the A-side formation runs while B moves; each arriving panel feeds the first
//    B-side formation pass on its quadrant rows; leaf products and combination follow.
//  * otherwise one broadcast, then the one-GPU method.
#pragma once
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; every function is resolved with dlsym

#include <cstdlib>
#include <mutex>

#include "../../include/mm.h"
#include "common.cuh"
#include "strassen.cuh"

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
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
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
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
    if (api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.AllReduce && api.GroupStart &&
        api.GroupEnd && api.Send && api.Recv)
      api.handle = h;
  });
  return api.handle ? &api : nullptr;
}

struct DistState {
  ncclComm_t comm = nullptr;
  int rank = -1, world = 0, device = -1;
  cudaStream_t comm_stream = nullptr;
  static constexpr int kMaxPanels = 64;
  cudaEvent_t panel_ev[kMaxPanels + 2] = {};  // panels, then the local / reduced norms
  cudaEvent_t start_ev = nullptr, end_ev = nullptr;
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

// ---- the schedule -------------------------------------------------------------------------------
// Event slots: panel i completes on event i (< kMaxPanels); two more for the norms.
constexpr int kEvNormsLocal = DistState::kMaxPanels, kEvNormsReduced = DistState::kMaxPanels + 1;
constexpr int kDistEvents = DistState::kMaxPanels + 2;

struct OpList {
  mm_dist_op* ops;
  int cap, n;
  bool ok;
  void add(int32_t op, int32_t stream, int32_t index, int32_t flags, int64_t lo, int64_t hi) {
    if (n >= cap) {
      ok = false;
      return;
    }
    ops[n++] = mm_dist_op{op, stream, index, flags, lo, hi};
  }
  void record(int stream, int ev) { add(MM_OP_RECORD, stream, ev, 0, 0, 0); }
  void wait(int stream, int ev) { add(MM_OP_WAIT, stream, ev, 0, 0, 0); }
};

inline bool dist_panel_method(int method, int64_t P, int64_t M) {
  if (method == MM_NAIVE) return true;
  const bool even = P % 2 == 0 && M % 2 == 0;  // whole Winograd pairs, TMA-fed panel kernels
  return even && (method == MM_KAHAN || method == MM_KAHAN_FUSED || method == MM_WINOGRAD ||
                  method == MM_WINOGRAD_FUSED || method == MM_WINOGRAD_SCALED || method == MM_WINOGRAD_SCALED_FUSED);
}

// Strassen panel geometry: the first formation pass spans `span` levels; its units are the
// quadrant rows [0, h), h = Pp >> span, unit u reading B rows u + r h (r < 2^span).
inline void dist_strassen_geometry(int64_t P, int32_t levels, int* span, int64_t* h) {
  const int64_t q = int64_t(2) << levels;
  const int64_t Pp = cdiv(P, q) * q;
  *span = first_form_span(levels);
  *h = Pp >> *span;
}

// returns the number of ops, -1 on bad arguments or a too small list
inline int build_dist_schedule(int method, int64_t P, int64_t M, int32_t levels, int32_t panels, mm_dist_op* ops,
                               int cap) {
  if (!ops || cap < 1 || P < 1 || M < 1 || method < MM_NAIVE || method > MM_WINOGRAD_SCALED_FUSED) return -1;
  if (levels < -1 || levels > 8) return -1;
  OpList L{ops, cap, 0, true};
  const bool scaled = method == MM_WINOGRAD_SCALED || method == MM_WINOGRAD_SCALED_FUSED;
  const bool strassen = method == MM_STRASSEN || method == MM_STRASSEN_WINOGRAD;
  const bool wino = method == MM_WINOGRAD || method == MM_WINOGRAD_FUSED;
  const int fused = (method == MM_KAHAN_FUSED || method == MM_WINOGRAD_FUSED || method == MM_WINOGRAD_SCALED_FUSED)
                        ? MM_EX_FUSED
                        : 0;
  if (panels > DistState::kMaxPanels) panels = DistState::kMaxPanels;
  const bool use_panels = panels > 1 && (strassen ? levels >= 1 : dist_panel_method(method, P, M));
  if (scaled) {  // the norms first: lambda is known before B moves (the root holds B)
    L.add(MM_OP_NORMS, MM_STREAM_COMPUTE, 0, 0, 0, 0);
    L.record(MM_STREAM_COMPUTE, kEvNormsLocal);
    L.wait(MM_STREAM_COMM, kEvNormsLocal);
    L.add(MM_OP_ALLREDUCE_NORMS, MM_STREAM_COMM, 0, 0, 0, 0);
    L.record(MM_STREAM_COMM, kEvNormsReduced);
  }
  if (!use_panels) {
    L.add(MM_OP_BCAST, MM_STREAM_COMM, 0, 0, 0, P);
    L.record(MM_STREAM_COMM, 0);
    if (scaled) L.wait(MM_STREAM_COMPUTE, kEvNormsReduced);
    L.wait(MM_STREAM_COMPUTE, 0);
    L.add(MM_OP_FULL, MM_STREAM_COMPUTE, 0, 0, 0, P);
    return L.ok ? L.n : -1;
  }
  if (strassen) {
    int span;
    int64_t h;
    dist_strassen_geometry(P, levels, &span, &h);
    const int np = int(panels < h ? panels : h);
    int64_t ub[DistState::kMaxPanels + 1];
    for (int i = 0; i <= np; ++i) ub[i] = h * i / np;
    for (int i = 0; i < np; ++i) {
      for (int r = 0; r < (1 << span); ++r) {  // the B rows of units [ub[i], ub[i+1])
        const int64_t lo = r * h + ub[i], hi = r * h + ub[i + 1] < P ? r * h + ub[i + 1] : P;
        if (lo < hi) L.add(MM_OP_BCAST, MM_STREAM_COMM, i, 0, lo, hi);
      }
      L.record(MM_STREAM_COMM, i);
    }
    L.add(MM_OP_FORM_A, MM_STREAM_COMPUTE, 0, 0, 0, 0);  // overlaps the broadcast
    for (int i = 0; i < np; ++i) {
      L.wait(MM_STREAM_COMPUTE, i);
      L.add(MM_OP_FORM_B, MM_STREAM_COMPUTE, i, 0, ub[i], ub[i + 1]);
    }
    L.add(MM_OP_FORM_B_REST, MM_STREAM_COMPUTE, 0, 0, 0, 0);
    L.add(MM_OP_LEAF_COMBINE, MM_STREAM_COMPUTE, 0, 0, 0, 0);
    return L.ok ? L.n : -1;
  }
  int64_t kb[DistState::kMaxPanels + 1];
  const int np = dist_panel_bounds(P, panels, kb);
  for (int i = 0; i < np; ++i) {
    L.add(MM_OP_BCAST, MM_STREAM_COMM, i, 0, kb[i], kb[i + 1]);
    L.record(MM_STREAM_COMM, i);
  }
  if (scaled) {
    L.wait(MM_STREAM_COMPUTE, kEvNormsReduced);
    L.add(MM_OP_SCALE_A, MM_STREAM_COMPUTE, 0, 0, 0, P);
  }
  for (int i = 0; i < np; ++i) {
    const bool last = i == np - 1;
    const int32_t fl = fused | (i > 0 ? MM_EX_ACCUMULATE : 0) | (last ? 0 : MM_EX_KEEP_STATE);
    L.wait(MM_STREAM_COMPUTE, i);
    if (scaled) L.add(MM_OP_SCALE_B, MM_STREAM_COMPUTE, i, i > 0 ? MM_EX_ACCUMULATE : 0, kb[i], kb[i + 1]);
    if (wino && last) L.add(MM_OP_YZ, MM_STREAM_COMPUTE, i, fused, 0, P);
    L.add(MM_OP_PANEL, MM_STREAM_COMPUTE, i, fl, kb[i], kb[i + 1]);
  }
  return L.ok ? L.n : -1;
}

// ---- the alternative partition: Strassen's seven top-level products on the
// ranks, product p (H_{p+1}) on rank p % world; A and B broadcast, each H sent to the root, which
// combines.  Events: 0 = A and B arrived, 1 + p = product p done, 8 = every H at the root.
constexpr int kS7EvInputs = 0, kS7EvGathered = 8;

inline int s7_owner(int p, int world) { return p % world; }

inline int build_s7_schedule(int method, int64_t N, int64_t P, int64_t M, int32_t levels, int32_t world, int32_t rank,
                             int32_t root, mm_dist_op* ops, int cap) {
  if (!ops || cap < 1 || N < 1 || P < 1 || M < 1 || levels < 1 || levels > 8) return -1;
  if (method != MM_STRASSEN && method != MM_STRASSEN_WINOGRAD) return -1;
  if (world < 1 || rank < 0 || rank >= world || root < 0 || root >= world) return -1;
  OpList L{ops, cap, 0, true};
  L.add(MM_OP_BCAST_A, MM_STREAM_COMM, 0, 0, 0, N);
  L.add(MM_OP_BCAST, MM_STREAM_COMM, 0, 0, 0, P);
  L.record(MM_STREAM_COMM, kS7EvInputs);
  L.wait(MM_STREAM_COMPUTE, kS7EvInputs);
  for (int p = 0; p < 7; ++p) {
    if (s7_owner(p, world) != rank) continue;
    L.add(MM_OP_S7_FORM, MM_STREAM_COMPUTE, p, 0, 0, 0);
    L.add(MM_OP_S7_PRODUCT, MM_STREAM_COMPUTE, p, 0, 0, 0);
    if (rank != root) {
      L.record(MM_STREAM_COMPUTE, 1 + p);
      L.wait(MM_STREAM_COMM, 1 + p);
      L.add(MM_OP_SEND_H, MM_STREAM_COMM, p, 0, root, 0);
    }
  }
  if (rank == root) {
    for (int p = 0; p < 7; ++p)
      if (s7_owner(p, world) != root) L.add(MM_OP_RECV_H, MM_STREAM_COMM, p, 0, s7_owner(p, world), 0);
    L.record(MM_STREAM_COMM, kS7EvGathered);
    L.wait(MM_STREAM_COMPUTE, kS7EvGathered);
    L.add(MM_OP_S7_COMBINE, MM_STREAM_COMPUTE, 0, 0, 0, 0);
  }
  return L.ok ? L.n : -1;
}

}  // namespace mmk
