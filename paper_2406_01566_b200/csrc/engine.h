// engine.h — internal types shared by the engine's translation units.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/helio_gpu.h"

namespace helio_engine {

// ---------------------------------------------------------------------------
// Device-side cluster constants (K0 output).
struct ClusterDev {
  int N, L, Mv;
  // SCORE solver for graphs with more than 128 vertices: 0 = push-relabel
  // with global relabels every pr_gr pulses (default), 1 = Edmonds-Karp with
  // the batched queue BFS (HELIO_LARGE_SOLVER / HELIO_PR_GR, tuning knobs)
  int large_solver, pr_gr;
  const int16_t* kmax;      // [N]
  const int32_t* lexrank;   // [N]
  const int16_t* lexnode;   // [N] node at lex rank r
  const int32_t* cap_off;   // [N] start of node's compute-capacity row (j = 1..k)
  const double* cap_tab;    // compute_edge_capacity(c, node, j)
  const uint32_t* link_pack;  // [Mv] (src+1) | (dst+1) << 16, 0 = coordinator
  const double* link_cap;     // [Mv] link_token_capacity with the reference payload
  const double* cin_cap;      // [N] capacity of node -> coordinator edge (value sum)
  // SCORE builder (arc order free): per-node link lists.
  const int32_t* cout_link;   // [N] link index of coordinator -> node, -1 none
  const int32_t* cin_link;    // [N] link index of node -> coordinator, -1 none
  const int32_t* out_beg;     // [N+1] into out_list
  const int32_t* in_beg;      // [N+1] into in_list
  const int2* out_list;       // (dst node, link index) of node -> node links
  const int2* in_list;        // (src node, link index)
  const unsigned long long* out_mask;  // [N] (N <= 64 only) node -> node link targets
  const int32_t* pair_link;            // [N*N] (N <= 64 only) link index or -1
  const unsigned long long* less_cout; // [N] (N <= 64 only) nodes whose coord->node link comes first
  const unsigned long long* less_cin;  // [N] (N <= 64 only) nodes whose node->coord link comes first
};

// Shared-memory slot layout of one graph (byte offsets from the slot base).
struct Layout {
  int V, A, N, M;  // vertex, arc, node, raw-edge capacities
  int o_vs, o_cap, o_ex, o_to, o_rv, o_abeg, o_h, o_cur, o_q, o_cnt, o_inq, o_ps, o_pe, o_vin, o_unode,
      o_efwd;
  int bytes;
};

}  // namespace helio_engine

struct helio_gpu_ctx {
  mutable std::recursive_mutex mu;  // every C ABI entry holds it: a context serialises its callers
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;
  std::string err;
  int64_t launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timed = false;

  bool has_cluster = false;
  int N = 0, L = 0, Mv = 0, Vmax = 0;
  std::vector<int32_t> h_kmax;
  std::vector<int32_t> h_cap_off;
  std::vector<double> h_cap_tab;
  std::vector<int32_t> h_lexrank;
  std::vector<double> h_vram;
  double bytes_per_layer = 0, kv_token_layer_bytes = 0;
  helio_engine::ClusterDev cd{};
  void* d_cluster = nullptr;  // one allocation for all constant arrays
  int32_t* d_kmax32 = nullptr;
  helio_engine::Layout small{}, big{};  // PARITY slots (also the split pipeline's)
  int small_warps = 4, small_blocks[2] = {0, 0}, big_blocks[2] = {0, 0};
  // per-mode slots for score_kernel<MODE> (SCORE uses a compact layout when N > 64)
  helio_engine::Layout slot_small[2]{}, slot_big[2]{};
  // middle tier between the small and the big slot (dense placements, e.g. the
  // heuristics' replicated stages, which overflow the small slot)
  helio_engine::Layout slot_mid[2]{};
  int mid_warps[2] = {1, 1}, mid_blocks[2] = {0, 0};
  bool slot_mid_ok[2] = {false, false};
  int slot_warps[2] = {4, 4};
  bool slot_big_ok[2] = {false, false};
  int mode = 0;  // HELIO_MODE_PARITY
  // SCORE path: general builder + push-relabel when split graphs exceed 128
  // vertices (N >= 64), else the cover-mask builder + bitset Edmonds-Karp
  bool score_gen = false;
  bool big_ok = false;

  // scratch sets: kPipeSets for the host-buffer pipeline (one per stream;
  // three so a chunk's overflow pass, which waits for the next chunk's kernel
  // to release the SMs, never holds up the following H2D), plus kApiSet for
  // the device-pointer entries and search.cu
  static constexpr int kPipeSets = 3, kApiSet = 3, kSets = 4;
  unsigned long long* d_work = nullptr;  // [32]: raw [0], split.cu [8]/[9], set k [16+4k, 16+4k+3]
  unsigned int* d_ovf_count = nullptr;   // [3 * kSets]: small -> mid, mid -> big, big -> global
  int64_t* d_ovf[kSets] = {nullptr, nullptr, nullptr, nullptr};   // small-slot overflows
  int64_t* d_ovf2[kSets] = {nullptr, nullptr, nullptr, nullptr};  // mid-slot overflows
  int64_t* d_ovf3[kSets] = {nullptr, nullptr, nullptr, nullptr};  // big-slot overflows (global tier)
  // global-memory tier: per-mode slot for the structural maximum when the big
  // slot cannot hold it; one slot per warp of glob_warps one-warp CTAs
  helio_engine::Layout slot_glob[2]{};
  bool glob_ok[2] = {false, false};
  int glob_warps = 0;
  char* d_glob = nullptr;
  int64_t ovf_cap[kSets] = {0, 0, 0, 0};
  double* d_pv = nullptr;      // argmax partials: kSets + 1 scratch rows of 4096
  long long* d_pi = nullptr;
  double* d_best = nullptr;   // per-chunk best of score_best_host
  int64_t* d_bidx = nullptr;

  // host-call staging
  int16_t* d_pl[kPipeSets] = {nullptr, nullptr, nullptr};
  double* d_val[kPipeSets] = {nullptr, nullptr, nullptr};
  int32_t* d_st[kPipeSets] = {nullptr, nullptr, nullptr};
  int16_t* h_pl_pin[kPipeSets] = {nullptr, nullptr, nullptr};
  double* h_val_pin[kPipeSets] = {nullptr, nullptr, nullptr};
  int32_t* h_st_pin[kPipeSets] = {nullptr, nullptr, nullptr};
  int64_t stage_cap = 0;
  cudaStream_t pipe[kPipeSets] = {nullptr, nullptr, nullptr};

  // resident staging for pinned callers: the whole batch on the device, its
  // H2D issued up front on `copy`, one event per chunk
  int16_t* d_pl_all = nullptr;
  double* d_val_all = nullptr;
  int32_t* d_st_all = nullptr;
  int64_t all_cap = 0;
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;

  // walk generator adjacency (gen.h hg_candidate_walk)
  const int32_t* d_walk_beg = nullptr;
  const int32_t* d_walk_list = nullptr;
  std::vector<int32_t> h_walk_beg, h_walk_list;

  // Ordering of the shared device-pointer scratch (set kApiSet, the argmax
  // row kSets, the split pipeline's counters) across caller streams: the host
  // mutex only serialises enqueue, so every use makes its stream wait for the
  // previous use's completion event and then records its own (api_begin/end).
  cudaEvent_t api_ev = nullptr;
  bool api_ev_used = false;

  // grow-only device scratch of the synchronous host entries (flows_host,
  // maxflow_raw_host): carved per call, so the per-call path makes no
  // cudaMalloc/cudaFree (cudaFree synchronises the whole device)
  void* d_host_arena = nullptr;
  size_t host_arena_cap = 0;

  // routing arena (route.cu), grows only
  void* d_route = nullptr;
  size_t route_cap = 0;

  // pinned host staging of the routing and flows entries, grows only
  void* h_stage_pin = nullptr;
  size_t stage_pin_cap = 0;
};


namespace helio_engine {

inline int fail(helio_gpu_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(ctx, HELIO_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Carves typed, 256-byte aligned pieces out of one allocation.  With base ==
// nullptr it only measures (pass 1), then the same sequence is replayed on the
// real base (pass 2).
struct Carve {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* r = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += sizeof(T) * (n ? n : 1);
    return r;
  }
};

// The host-entry arena (helio_gpu_ctx::d_host_arena) with at least `bytes`.
inline int host_arena(helio_gpu_ctx* ctx, size_t bytes, char** out) {
  if (ctx->host_arena_cap < bytes) {
    cudaFree(ctx->d_host_arena);
    ctx->d_host_arena = nullptr;
    ctx->host_arena_cap = 0;
    const size_t cap = std::max<size_t>(bytes + bytes / 4, size_t(1) << 20);
    CK(cudaMalloc(&ctx->d_host_arena, cap));
    ctx->host_arena_cap = cap;
  }
  *out = static_cast<char*>(ctx->d_host_arena);
  return HELIO_OK;
}

// Pageable <-> pinned staging copy split over a few host threads (helio_gpu.cu).
void stage_copy(void* dst, const void* src, size_t bytes);
// cudaPointerGetAttributes says page-locked host memory.
bool is_pinned(const void* p);

// The host entries' pinned staging buffer with at least `bytes`.
inline int host_pin(helio_gpu_ctx* ctx, size_t bytes, char** out) {
  if (ctx->stage_pin_cap < bytes) {
    cudaFreeHost(ctx->h_stage_pin);
    ctx->h_stage_pin = nullptr;
    ctx->stage_pin_cap = 0;
    const size_t cap = std::max<size_t>(bytes + bytes / 4, size_t(1) << 20);
    CK(cudaMallocHost(&ctx->h_stage_pin, cap));
    ctx->stage_pin_cap = cap;
  }
  *out = static_cast<char*>(ctx->h_stage_pin);
  return HELIO_OK;
}

// See helio_gpu_ctx::api_ev.
inline cudaError_t api_begin(helio_gpu_ctx* c, cudaStream_t st) {
  return c->api_ev_used ? cudaStreamWaitEvent(st, c->api_ev, 0) : cudaSuccess;
}
inline cudaError_t api_end(helio_gpu_ctx* c, cudaStream_t st) {
  c->api_ev_used = true;
  return cudaEventRecord(c->api_ev, st);
}

}  // namespace helio_engine
