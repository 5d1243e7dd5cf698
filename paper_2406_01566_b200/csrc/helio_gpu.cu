// helio_gpu.cu — B200 (sm_100a) engine behind include/helio_gpu.h: kernels,
// K0 cluster compiler, launchers and the C ABI entry points.
//
// Device code is split by role (all included into this translation unit):
//   device_common.cuh  shared-memory slot layout, per-warp views, warp helpers
//   build.cuh          K1: placement row -> flow network in shared memory
//   solve_parity.cuh   K2 PARITY: bit-exact FIFO preflow-push replay + read-out
//   solve_score.cuh    K2 SCORE: value-only bitset Edmonds-Karp (V <= 128) and
//                      push-relabel with global relabels (larger graphs)
//
// Kernels here (SIMT; the path is FP64 min/add/compare graph work — no tensor
// cores):
//   score_kernel<MODE, GEN>
//                       placement rows -> graph -> max-flow value, one warp per
//                       graph, persistent CTAs pulling work from an atomic
//                       counter; graphs whose arcs exceed the small slot are
//                       queued for the same kernel with a middle slot (twice
//                       the arcs), and what overflows that for one warp per CTA
//                       with a slot for every declared link.
//   raw_kernel          max_flow on caller-supplied raw graphs (AC1 style).
//   argmax_*            (max value, min index) reduction (enumerate.hpp:59).
//   gen_kernel / gen_walk_kernel   counter-based candidate generators (gen.h).
// route.cu holds K3 (IWRR routing), search.cu the exhaustive, local and
// sampled placement searches, split.cu the split K1 -> HBM -> K2 pipeline.
//
// Everything is compiled with -fmad=false; the only FP operations on the path
// are min / + / - / compare on doubles, in the reference's order.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <thread>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/helio_gpu.h"
#include "engine.h"
#include "gen.h"

using namespace helio_engine;

#define FLOW_EPS 1e-12  // kFlowEps, flow_graph.cpp:15
#define FULL 0xffffffffu
#define ST_OVERFLOW 100  // internal: arcs exceed the small slot

#include "device_common.cuh"
#include "build.cuh"
#include "solve_parity.cuh"
#include "solve_score.cuh"

namespace {

struct FlowOut {
  helio_edge* edges;  // [B][max_e] or nullptr
  int32_t* nv;
  int32_t* ne;
  int max_e;
};

// Persistent: every warp loops fetching candidate indices — all B of them
// (in_list == nullptr) or the *in_count entries of in_list.  Graphs whose arcs
// exceed this launch's slot are appended to out_list for the next tier, or
// reported HELIO_CAND_TOO_LARGE when there is none.  Tiers (launch_score_mode):
// small slot -> middle slot -> big slot (one warp per CTA, every declared link)
// -> a slot in global memory (gbase != nullptr: clusters whose structural
// maximum does not fit one SM's shared memory; L1/L2 cached).
// GEN (SCORE only): an instantiation with only the general builder and the
// push-relabel solver, for clusters whose split graphs exceed 128 vertices
// (N >= 64), so that path's register allocation is its own; the default one
// keeps both paths (het42 runs it at 64 registers, 8 CTAs per SM).
// HELIO_PARITY_DIAG_MINB (diagnostic builds only): cap the PARITY kernel's
// registers through __launch_bounds__(128, n) — the configuration that faults
// (see DESIGN.md §4), for bounds-checked reproduction with HELIO_BOUNDS.
#ifdef HELIO_PARITY_DIAG_MINB
#define HELIO_SCORE_BOUNDS __launch_bounds__(128, MODE == HELIO_MODE_PARITY ? HELIO_PARITY_DIAG_MINB : 1)
#else
#define HELIO_SCORE_BOUNDS
#endif
template <int MODE, bool GEN, bool GLOBAL = false>
__global__ void HELIO_SCORE_BOUNDS score_kernel(ClusterDev cd, Layout lay, const int16_t* __restrict__ pl, int64_t B,
                                           int partial, double* __restrict__ values, int32_t* __restrict__ status,
                                           unsigned long long* work, const int64_t* in_list,
                                           const unsigned int* in_count, int64_t* out_list, unsigned int* out_count,
                                           char* gbase, FlowOut fo) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  // GLOBAL is a template parameter so the shared-memory instantiations keep
  // statically shared addressing (32-bit LDS/STS, not generic 64-bit)
  char* slot = GLOBAL ? gbase + ((size_t)blockIdx.x * (blockDim.x >> 5) + wib) * lay.bytes : smem + wib * lay.bytes;
  const Gs g = slot_view(slot, lay);
  const int64_t total = in_list ? (int64_t)*in_count : B;
  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(work, 1ull);
    w = __shfl_sync(FULL, w, 0);
    if ((int64_t)w >= total) break;
    const int64_t b = in_list ? in_list[w] : (int64_t)w;
    int V = 0, E = 0;
    double cut = 1.0e300;  // SCORE, N <= 64: the builder's layer cut (an upper bound to stop at)
    int st = MODE == HELIO_MODE_SCORE
                 ? (!GEN && cd.out_mask ? build_graph_score_small(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E, cut)
                 : GEN                  ? build_graph_score_contract(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E)
                                        : build_graph_score_r1(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E))
                 : (cd.less_cout
                        ? build_graph_small(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E)
                        : build_graph(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E));
    if (st == ST_OVERFLOW) {
      if (out_list) {
        if (lane == 0) out_list[atomicAdd(out_count, 1u)] = b;
        continue;
      }
      st = HELIO_CAND_TOO_LARGE;
    }
    double value = 0.0;
    if (st == 0 && MODE == HELIO_MODE_SCORE) {
      value = !GEN && V <= 128  ? solve_ek_bits(g, V, 0, 1, lane, cut)
              : cd.large_solver ? solve_ek_batched(g, V, 0, 1, lane)
                                : solve_pr<GEN>(g, V, 0, 1, lane, cd.pr_gr);
    } else if (st == 0) {
#ifdef HELIO_BOUNDS
      {  // diagnostic: the built CSR is well formed
        const int na = g.abeg[V];
        HB_CHECK(na, lay.A + 1, "arc count");
        for (int x = lane; x < V; x += 32) HB_CHECK(g.abeg[x + 1] - g.abeg[x], na + 1, "abeg order");
        for (int a = lane; a < na; a += 32) {
          HB_CHECK(g.to[a], V, "arc head");
          HB_CHECK(g.rv[a], na, "arc reverse");
          HB_CHECK(g.rv[g.rv[a]] == a ? 0 : 1, 1, "reverse pairing");
        }
        __syncwarp();
      }
#endif
      solve_fifo2(g, V, 0, 1, lane);
      value = built_value(cd, g, lane);
      if (fo.edges) {
        if (E <= fo.max_e) emit_edges(cd, g, (V - 2) / 2, partial, lane, fo.edges + b * fo.max_e);
        else st = HELIO_CAND_EDGE_BUFFER;
      }
    }
    if (lane == 0) {
      values[b] = value;
      status[b] = st;
      if (MODE == HELIO_MODE_PARITY && fo.nv) {  // SCORE calls never carry FlowOut
        fo.nv[b] = V;
        fo.ne[b] = E;
      }
    }
    __syncwarp();
  }
}

// The kernels: score_body instantiated per mode, plus the large-graph SCORE
// variant (GEN), each with its own register allocation.  No register caps:
// capping (__maxnreg__ / __launch_bounds__) measured 33M instead of 70M
// evals/s on het42 SCORE, and the default instantiations keep round 1's code
// (64 registers, 8 four-warp CTAs per SM on het42).

// ---------------------------------------------------------------------------
// max_flow on raw graphs.  Arc construction follows :140-145 literally (lane
// 0, edge order; a self-loop's forward arc gets rev = itself because adj[v].
// size() is read before the push_back).
template <bool GLOBAL>
__global__ void raw_kernel(Layout lay, int64_t G, const int32_t* __restrict__ gn,
                           const int32_t* __restrict__ gs, const int32_t* __restrict__ gt,
                           const int64_t* __restrict__ eoff, const int32_t* __restrict__ eu,
                           const int32_t* __restrict__ ev, const double* __restrict__ ecap,
                           double* __restrict__ values, double* __restrict__ flows,
                           unsigned long long* work, char* gbase) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  // gbase: graphs larger than one SM's shared memory work in global memory
  char* slot = GLOBAL ? gbase + ((size_t)blockIdx.x * (blockDim.x >> 5) + wib) * lay.bytes : smem + wib * lay.bytes;
  const Gs g = slot_view(slot, lay);
  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(work, 1ull);
    w = __shfl_sync(FULL, w, 0);
    if ((int64_t)w >= G) break;
    const int64_t gi = (int64_t)w;
    const int n = gn[gi], s = gs[gi], t = gt[gi];
    const int64_t e0 = eoff[gi];
    const int m = (int)(eoff[gi + 1] - e0);
    for (int x = lane; x < n; x += 32) g.cur[x] = 0;
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < m; ++i) {
        g.cur[eu[e0 + i]] += 1;
        g.cur[ev[e0 + i]] += 1;
      }
      int run = 0;
      for (int x = 0; x < n; ++x) {
        g.abeg[x] = (int16_t)run;
        run += g.cur[x];
        g.cur[x] = 0;
      }
      g.abeg[n] = (int16_t)run;
      for (int i = 0; i < m; ++i) {
        const int a = eu[e0 + i], bb = ev[e0 + i];
        const int pa = g.cur[a];
        const int rpos = g.abeg[bb] + g.cur[bb];
        const int fa = g.abeg[a] + pa;
        g.cur[a] += 1;
        g.to[fa] = (int16_t)bb;
        g.cap[fa] = ecap[e0 + i];
        g.rv[fa] = (int16_t)rpos;
        const int ra = g.abeg[bb] + g.cur[bb];
        g.cur[bb] += 1;
        g.to[ra] = (int16_t)a;
        g.cap[ra] = 0.0;
        g.rv[ra] = (int16_t)fa;
        g.efwd[i] = (int16_t)fa;
      }
    }
    __syncwarp();
    solve_fifo2(g, n, s, t, lane);
    if (flows) {
      for (int i = lane; i < m; i += 32) {
        double f = ecap[e0 + i] - g.cap[g.efwd[i]];
        if (f < FLOW_EPS) f = 0.0;
        flows[e0 + i] = f;
      }
    }
    if (lane == 0) {
      double value = 0.0;
      for (int i = 0; i < m; ++i) {
        double f = ecap[e0 + i] - g.cap[g.efwd[i]];
        if (f < FLOW_EPS) f = 0.0;
        if (ev[e0 + i] == t) value += f;
        if (eu[e0 + i] == t) value -= f;
      }
      values[gi] = value;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// K4: argmax, (value desc, index asc) among status == 0 && value > 0.
__device__ __forceinline__ bool better(double v1, long long i1, double v2, long long i2) {
  return v1 > v2 || (v1 == v2 && i1 < i2);
}

__global__ void argmax_partial(const double* __restrict__ values, const int32_t* __restrict__ status,
                               int64_t B, double* pv, long long* pi) {
  double bv = 0.0;
  long long bi = -1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (status[i] != 0) continue;
    const double v = values[i];
    if (v > 0.0 && (bi < 0 || better(v, i, bv, bi))) {
      bv = v;
      bi = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(FULL, bv, o);
    const long long oi = __shfl_down_sync(FULL, bi, o);
    if (oi >= 0 && (bi < 0 || better(ov, oi, bv, bi))) {
      bv = ov;
      bi = oi;
    }
  }
  __shared__ double sv[32];
  __shared__ long long si[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sv[wid] = bv;
    si[wid] = bi;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : 0.0;
    bi = lane < nw ? si[lane] : -1;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(FULL, bv, o);
      const long long oi = __shfl_down_sync(FULL, bi, o);
      if (oi >= 0 && (bi < 0 || better(ov, oi, bv, bi))) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      pv[blockIdx.x] = bv;
      pi[blockIdx.x] = bi;
    }
  }
}

__global__ void argmax_final(const double* pv, const long long* pi, int P, int64_t base,
                             double* best, int64_t* index) {
  if (threadIdx.x != 0) return;
  double bv = 0.0;
  long long bi = -1;
  for (int p = 0; p < P; ++p)
    if (pi[p] >= 0 && (bi < 0 || better(pv[p], pi[p], bv, bi))) {
      bv = pv[p];
      bi = pi[p];
    }
  *best = bv;
  *index = bi < 0 ? -1 : bi + base;
}

// ---------------------------------------------------------------------------
#define GEN_MAX_N 1024
__global__ void gen_kernel(const int32_t* __restrict__ kmax, int N, int L, uint64_t seed,
                           int64_t first, int64_t B, uint32_t ppm, int16_t* __restrict__ out) {
  int16_t perm[GEN_MAX_N];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B;
       i += (int64_t)gridDim.x * blockDim.x)
    hg_candidate(kmax, N, L, seed, (uint64_t)(first + i), ppm, perm, out + i * 2 * N);
}

__global__ void gen_walk_kernel(const int32_t* __restrict__ kmax, int N, int L, uint64_t seed, int64_t first,
                                int64_t B, const int32_t* __restrict__ wbeg, const int32_t* __restrict__ wlist,
                                int16_t* __restrict__ out) {
  uint32_t used[GEN_MAX_N / 32];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B;
       i += (int64_t)gridDim.x * blockDim.x)
    hg_candidate_walk(kmax, N, L, seed, (uint64_t)(first + i), wbeg, wlist, used, out + i * 2 * N);
}

}  // namespace

// ===========================================================================
// Host side: context, K0 cluster compiler, launchers.


namespace {

double host_min(double a, double b) { return b < a ? b : a; }
double host_max(double a, double b) { return a < b ? b : a; }

int configure_layouts(helio_gpu_ctx* ctx) {
  const int N = ctx->N, V = 2 * N + 2;
  ctx->Vmax = V;
  // Small slot: sized for the common case; rarer dense graphs overflow to the
  // big slot.  Arc budget 8N (4N edges): covering chains average E ~3.3N
  // (het42: mean 140, p99 159, max seen 165 of 168), and at N = 42 the slot
  // (12A + 27V + 8N bytes = 6.7 KB) lets 8 four-warp CTAs share an SM — the
  // register limit at 64 registers — instead of 7.
  // Sparse interconnects: link-walking placements carry ~2.6N edges (max
  // seen 2.75N on syn256), so 6N arcs hold them and the smaller slot buys
  // resident warps.  PARITY (and the split pipeline's slab) switches below 16
  // declared links per node; SCORE's compact general layout below 32 (both
  // directions and the coordinator's count: syn256's 12 peers give ~25).
  // The N <= 64 builders keep per-layer cover/start masks in cap[] while they
  // run, so every slot holds at least 2L + 2 arcs (tiny sparse clusters with
  // many layers have fewer structural arcs than that).
  const int a_masks = 2 * ctx->L + 2;
  auto small_arcs = [&](int sparse_below) {
    int a = ctx->Mv < sparse_below * N ? 6 * N : 8 * N;
    const int a_struct = 2 * (N + ctx->Mv);
    if (a > a_struct) a = a_struct;
    return std::max(a, a_masks);
  };
  const int a_struct = 2 * (N + ctx->Mv);
  const size_t max_smem = 227 * 1024;
  // One mode's slots: the small one with the warps per CTA that keep the most
  // warps resident per SM (228 KB, 1 KB reserved per CTA; larger CTAs on
  // ties), and the big one for the structural maximum (every declared link
  // valid) or the largest arc count that still fits one CTA.
  auto best_warps = [&](const Layout& l) {
    int warps = 1, best_res = -1;
    for (int w : {4, 2, 1}) {
      const size_t cta = (size_t)l.bytes * w;
      if (cta > max_smem) continue;
      const int res = w * (int)std::min<size_t>(32, (228 * 1024) / (cta + 1024));
      if (res > best_res) {
        best_res = res;
        warps = w;
      }
    }
    return warps;
  };
  auto plan = [&](bool compact, int a_small, Layout& small, Layout& big, int& warps_out, bool& big_ok) {
    auto mk = [&](int a) { return compact ? make_layout_score_general(V, a, N) : make_layout(V, a, N, 0); };
    small = mk(a_small);
    warps_out = best_warps(small);
    int a_big = std::max(a_struct, a_masks);
    if (a_big > 32766) a_big = 32766;
    big = mk(a_big);
    big_ok = (size_t)big.bytes <= max_smem;
    if (!big_ok) {
      int lo = 2, hi = a_big;
      while (lo < hi) {
        int mid = (lo + hi + 1) / 2;
        if ((size_t)mk(mid).bytes <= max_smem) lo = mid;
        else hi = mid - 1;
      }
      big = mk(lo);
      big_ok = (size_t)big.bytes <= max_smem;
    }
  };
  plan(false, small_arcs(16), ctx->small, ctx->big, ctx->small_warps, ctx->big_ok);
  if ((size_t)ctx->small.bytes * ctx->small_warps > max_smem)
    return fail(ctx, HELIO_ERR_TOO_LARGE, "cluster too large: one graph slot exceeds shared memory");
  ctx->slot_small[HELIO_MODE_PARITY] = ctx->small;
  ctx->slot_big[HELIO_MODE_PARITY] = ctx->big;
  ctx->slot_warps[HELIO_MODE_PARITY] = ctx->small_warps;
  ctx->slot_big_ok[HELIO_MODE_PARITY] = ctx->big_ok;
  // SCORE: N <= 64 runs the cover-mask builder and bitset solver on the full
  // layout (residual rows in the VState bytes); the large-graph kernel
  // (score_gen) builds series-contracted networks (make_layout_contract: V, A
  // count contracted vertices / arcs; the small slot holds 5N/4 + 8 vertices
  // and 4N arcs — syn256 link walks contract to p99 277 / 986)
  if (ctx->score_gen) {
    const int Vs = std::min(V, 5 * N / 4 + 8);
    const int As = std::min(std::max(a_struct, a_masks), std::max(4 * N, 2 * ctx->L + 2));
    Layout& sm = ctx->slot_small[HELIO_MODE_SCORE];
    Layout& bg = ctx->slot_big[HELIO_MODE_SCORE];
    sm = make_layout_contract(Vs, As, N);
    ctx->slot_warps[HELIO_MODE_SCORE] = best_warps(sm);
    int a_big = std::min(std::max(a_struct, a_masks), 32766);
    bg = make_layout_contract(V, a_big, N);
    if ((size_t)bg.bytes > max_smem) {
      int lo = 2, hi = a_big;
      while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if ((size_t)make_layout_contract(V, mid, N).bytes <= max_smem) lo = mid;
        else hi = mid - 1;
      }
      bg = make_layout_contract(V, lo, N);
    }
    ctx->slot_big_ok[HELIO_MODE_SCORE] = (size_t)bg.bytes <= max_smem;
  } else {
    plan(N > 64, small_arcs(N > 64 ? 32 : 16), ctx->slot_small[HELIO_MODE_SCORE], ctx->slot_big[HELIO_MODE_SCORE],
         ctx->slot_warps[HELIO_MODE_SCORE], ctx->slot_big_ok[HELIO_MODE_SCORE]);
  }
  // middle tier: twice the small slot's arcs (placements with replicated
  // stages — the heuristics' petals/swarm layouts carry ~5N edges on het42),
  // with its own warps per CTA; skipped when it would not beat the big slot
  auto mk_mode = [&](int m, int a) {
    if (m == HELIO_MODE_SCORE && ctx->score_gen) return make_layout_contract(V, a, N);
    return m == HELIO_MODE_SCORE && N > 64 ? make_layout_score_general(V, a, N) : make_layout(V, a, N, 0);
  };
  for (int m = 0; m < 2; ++m) {
    const int a_small = ctx->slot_small[m].A;
    const int a_mid = std::min(2 * a_small, ctx->slot_big[m].A);
    ctx->slot_mid_ok[m] = false;
    if (ctx->slot_big_ok[m] && a_mid < ctx->slot_big[m].A && (a_mid > a_small || ctx->slot_small[m].V < V)) {
      ctx->slot_mid[m] = mk_mode(m, a_mid);
      ctx->mid_warps[m] = best_warps(ctx->slot_mid[m]);
      ctx->slot_mid_ok[m] = (size_t)ctx->slot_mid[m].bytes * ctx->mid_warps[m] <= max_smem;
    }
  }
  // global tier: when even the big slot is smaller than the structural
  // maximum (every declared link valid; int16 arc indices), a slot of that
  // size in global memory finishes what overflows it
  ctx->glob_warps = 2 * ctx->sm_count;
  for (int m = 0; m < 2; ++m) {
    const int a_full = std::min(std::max(a_struct, a_masks), 32766);
    const int a_have = ctx->slot_big_ok[m] ? ctx->slot_big[m].A : ctx->slot_small[m].A;
    ctx->glob_ok[m] = a_full > a_have;
    if (ctx->glob_ok[m]) ctx->slot_glob[m] = mk_mode(m, a_full);
  }
  // occupancy of both instantiations (PARITY / SCORE)
  void* fns[2] = {reinterpret_cast<void*>(score_kernel<HELIO_MODE_PARITY, false>),
                  ctx->score_gen ? reinterpret_cast<void*>(score_kernel<HELIO_MODE_SCORE, true>)
                                 : reinterpret_cast<void*>(score_kernel<HELIO_MODE_SCORE, false>)};
  for (int m = 0; m < 2; ++m) {
    CK(cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem));
    // the whole unified L1/shared array as shared memory: the driver's default
    // carveout (200 KB here) would cap het42 at 7 four-warp CTAs per SM
    CK(cudaFuncSetAttribute(fns[m], cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    const int w = ctx->slot_warps[m];
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[m], 32 * w, ctx->slot_small[m].bytes * w));
    if (per_sm < 1) per_sm = 1;
    ctx->small_blocks[m] = per_sm * ctx->sm_count;
    int per_sm_big = 1;
    if (ctx->slot_big_ok[m]) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_big, fns[m], 32, ctx->slot_big[m].bytes));
      if (per_sm_big < 1) per_sm_big = 1;
    }
    ctx->big_blocks[m] = per_sm_big * ctx->sm_count;
    int per_sm_mid = 1;
    if (ctx->slot_mid_ok[m]) {
      const int wm = ctx->mid_warps[m];
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_mid, fns[m], 32 * wm, ctx->slot_mid[m].bytes * wm));
      if (per_sm_mid < 1) per_sm_mid = 1;
    }
    ctx->mid_blocks[m] = per_sm_mid * ctx->sm_count;
  }
  return HELIO_OK;
}

int ensure_ovf(helio_gpu_ctx* ctx, int set, int64_t B) {
  if (ctx->ovf_cap[set] >= B) return HELIO_OK;
  cudaFree(ctx->d_ovf[set]);
  cudaFree(ctx->d_ovf2[set]);
  cudaFree(ctx->d_ovf3[set]);
  ctx->d_ovf[set] = ctx->d_ovf2[set] = ctx->d_ovf3[set] = nullptr;
  ctx->ovf_cap[set] = 0;
  int64_t cap = std::max<int64_t>(B, 1 << 16);
  CK(cudaMalloc(&ctx->d_ovf[set], sizeof(int64_t) * cap));
  CK(cudaMalloc(&ctx->d_ovf2[set], sizeof(int64_t) * cap));
  CK(cudaMalloc(&ctx->d_ovf3[set], sizeof(int64_t) * cap));
  ctx->ovf_cap[set] = cap;
  return HELIO_OK;
}

template <int MODE, bool GEN = false>
void launch_score_mode(helio_gpu_ctx* ctx, int set, const int16_t* d_pl, int64_t B, int partial, double* d_val,
                       int32_t* d_st, cudaStream_t st, FlowOut fo, bool timed) {
  unsigned long long* work = ctx->d_work + 16 + 4 * set;
  unsigned int* oc = ctx->d_ovf_count + 3 * set;
  int64_t* l1 = ctx->d_ovf[set];
  int64_t* l2 = ctx->d_ovf2[set];
  int64_t* l3 = ctx->d_ovf3[set];
  const bool glob = ctx->glob_ok[MODE] && ctx->d_glob != nullptr;
  if (timed) cudaEventRecord(ctx->ev0, st);
  const Layout& sl = ctx->slot_small[MODE];
  if (B == 1 && !timed) {
    // one candidate (the per-call entries): straight into the biggest shared
    // slot — one warp either way, and the small and middle tiers' launches
    // are saved; only a graph beyond one SM goes on to the global tier
    const Layout& bl1 = ctx->slot_big_ok[MODE] ? ctx->slot_big[MODE] : sl;
    auto K1 = score_kernel<MODE, GEN>;
    K1<<<1, 32, bl1.bytes, st>>>(ctx->cd, bl1, d_pl, B, partial, d_val, d_st, work + 2, nullptr, nullptr,
                                 glob ? l3 : nullptr, oc + 2, nullptr, fo);
    if (glob) {
      score_kernel<MODE, GEN, true><<<1, 32, 0, st>>>(ctx->cd, ctx->slot_glob[MODE], d_pl, B, partial, d_val, d_st,
                                                      work + 3, l3, oc + 2, nullptr, nullptr, ctx->d_glob, fo);
      ctx->launches += 1;
    }
    return;
  }
  const int warps = ctx->slot_warps[MODE];
  const int grid = (int)std::min<int64_t>(ctx->small_blocks[MODE], (B + warps - 1) / warps);
  auto K = score_kernel<MODE, GEN>;
  K<<<grid, 32 * warps, sl.bytes * warps, st>>>(ctx->cd, sl, d_pl, B, partial, d_val, d_st, work, nullptr, nullptr,
                                                 l1, oc, nullptr, fo);
  // graphs that overflowed the small slot: the same kernel with the middle
  // slot, then whatever overflows that with the big slot (one warp per CTA),
  // then — for clusters too large for one SM — a slot in global memory
  const Layout& bl = ctx->slot_big_ok[MODE] ? ctx->slot_big[MODE] : sl;
  const int64_t* big_in = l1;
  const unsigned int* big_cnt = oc;
  if (ctx->slot_mid_ok[MODE]) {
    const Layout& ml = ctx->slot_mid[MODE];
    const int wm = ctx->mid_warps[MODE];
    K<<<ctx->mid_blocks[MODE], 32 * wm, ml.bytes * wm, st>>>(ctx->cd, ml, d_pl, B, partial, d_val, d_st, work + 1, l1,
                                                            oc, l2, oc + 1, nullptr, fo);
    big_in = l2;
    big_cnt = oc + 1;
    ctx->launches += 1;
  }
  K<<<ctx->big_blocks[MODE], 32, bl.bytes, st>>>(ctx->cd, bl, d_pl, B, partial, d_val, d_st, work + 2, big_in,
                                                 big_cnt, glob ? l3 : nullptr, oc + 2, nullptr, fo);
  if (glob) {
    score_kernel<MODE, GEN, true><<<ctx->glob_warps, 32, 0, st>>>(ctx->cd, ctx->slot_glob[MODE], d_pl, B, partial, d_val, d_st, work + 3, l3,
                                      oc + 2, nullptr, nullptr, ctx->d_glob, fo);
    ctx->launches += 1;
  }
  // kernel time = all tier launches
  if (timed) cudaEventRecord(ctx->ev1, st);
}

int launch_score(helio_gpu_ctx* ctx, int set, const int16_t* d_pl, int64_t B, int partial,
                 double* d_val, int32_t* d_st, cudaStream_t st, FlowOut fo, bool timed, int mode) {
  if (B <= 0) return HELIO_OK;
  int rc = ensure_ovf(ctx, set, B);
  if (rc) return rc;
  // global-memory tier scratch (one slot per warp), allocated on first use
  if (ctx->glob_ok[mode] && ctx->d_glob == nullptr) {
    size_t bytes = 0;
    for (int m = 0; m < 2; ++m)
      if (ctx->glob_ok[m]) bytes = std::max(bytes, (size_t)ctx->glob_warps * ctx->slot_glob[m].bytes);
    CK(cudaMalloc(&ctx->d_glob, bytes));
  }
  CK(cudaMemsetAsync(ctx->d_work + 16 + 4 * set, 0, 4 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(ctx->d_ovf_count + 3 * set, 0, 3 * sizeof(unsigned int), st));
  if (mode == HELIO_MODE_SCORE && fo.edges == nullptr && fo.nv == nullptr && ctx->score_gen)
    launch_score_mode<HELIO_MODE_SCORE, true>(ctx, set, d_pl, B, partial, d_val, d_st, st, fo, timed);
  else if (mode == HELIO_MODE_SCORE && fo.edges == nullptr && fo.nv == nullptr)
    launch_score_mode<HELIO_MODE_SCORE, false>(ctx, set, d_pl, B, partial, d_val, d_st, st, fo, timed);
  else
    launch_score_mode<HELIO_MODE_PARITY>(ctx, set, d_pl, B, partial, d_val, d_st, st, fo, timed);
  CK(cudaGetLastError());
  ctx->launches += (B == 1 && !timed) ? 1 : 2;
  if (timed) ctx->timed = true;
  return HELIO_OK;
}

}  // namespace

// PARITY scoring of device rows on `st` (used by search.cu).
int helio_engine_score_parity(helio_gpu_ctx* ctx, const int16_t* d_pl, int64_t B, int partial, double* d_val,
                              int32_t* d_st, cudaStream_t st) {
  FlowOut fo{nullptr, nullptr, nullptr, 0};
  CK(api_begin(ctx, st));
  const int rc =
      launch_score(ctx, helio_gpu_ctx::kApiSet, d_pl, B, partial, d_val, d_st, st, fo, false, HELIO_MODE_PARITY);
  CK(api_end(ctx, st));
  return rc;
}

namespace {

int ensure_stage(helio_gpu_ctx* ctx, int64_t chunk) {
  if (ctx->stage_cap >= chunk) return HELIO_OK;
  // every set is released (and nulled, cap 0) before any reallocation, so a
  // failed allocation leaves no dangling pointer behind
  for (int i = 0; i < helio_gpu_ctx::kPipeSets; ++i) {
    cudaFree(ctx->d_pl[i]);
    cudaFree(ctx->d_val[i]);
    cudaFree(ctx->d_st[i]);
    cudaFreeHost(ctx->h_pl_pin[i]);
    cudaFreeHost(ctx->h_val_pin[i]);
    cudaFreeHost(ctx->h_st_pin[i]);
    ctx->d_pl[i] = nullptr;
    ctx->d_val[i] = nullptr;
    ctx->d_st[i] = nullptr;
    ctx->h_pl_pin[i] = nullptr;
    ctx->h_val_pin[i] = nullptr;
    ctx->h_st_pin[i] = nullptr;
  }
  ctx->stage_cap = 0;
  for (int i = 0; i < helio_gpu_ctx::kPipeSets; ++i) {
    CK(cudaMalloc(&ctx->d_pl[i], sizeof(int16_t) * 2 * ctx->N * chunk));
    CK(cudaMalloc(&ctx->d_val[i], sizeof(double) * chunk));
    CK(cudaMalloc(&ctx->d_st[i], sizeof(int32_t) * chunk));
    CK(cudaMallocHost(&ctx->h_pl_pin[i], sizeof(int16_t) * 2 * ctx->N * chunk));
    CK(cudaMallocHost(&ctx->h_val_pin[i], sizeof(double) * chunk));
    CK(cudaMallocHost(&ctx->h_st_pin[i], sizeof(int32_t) * chunk));
  }
  ctx->stage_cap = chunk;
  return HELIO_OK;
}

}  // namespace

namespace helio_engine {
// Pageable <-> pinned staging copies: large ones are split over a few host
// threads (one thread copies ~10 GB/s; het42's 256k-row chunk is 43 MB).
void stage_copy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPart = size_t(8) << 20;
  const int nt = (int)std::min<size_t>(8, bytes / kPart);
  if (nt < 2) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> pool;
  const size_t step = (bytes + nt - 1) / nt;
  for (int t = 1; t < nt; ++t) {
    const size_t lo = t * step, hi = std::min(bytes, lo + step);
    if (lo < hi)
      pool.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo); });
  }
  std::memcpy(dst, src, std::min(bytes, step));
  for (auto& th : pool) th.join();
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
}  // namespace helio_engine

// ===========================================================================
extern "C" {

int helio_gpu_create(int device, helio_gpu_ctx** out) {
  if (!out) return HELIO_ERR_INVALID;
  *out = nullptr;
  helio_gpu_ctx* ctx = new helio_gpu_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return HELIO_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10) {
    delete ctx;
    return HELIO_ERR_CUDA;  // built for sm_100a only
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->pipe[0], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->pipe[1], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->pipe[2], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->api_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&ctx->d_work, 32 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&ctx->d_ovf_count, 3 * helio_gpu_ctx::kSets * sizeof(unsigned int)) != cudaSuccess ||
      cudaMalloc(&ctx->d_pv, (helio_gpu_ctx::kSets + 1) * 4096 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ctx->d_pi, (helio_gpu_ctx::kSets + 1) * 4096 * sizeof(long long)) != cudaSuccess ||
      cudaMalloc(&ctx->d_best, 2 * 4096 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ctx->d_bidx, 2 * 4096 * sizeof(int64_t)) != cudaSuccess) {
    helio_gpu_destroy(ctx);
    return HELIO_ERR_CUDA;
  }
  *out = ctx;
  return HELIO_OK;
}

void helio_gpu_destroy(helio_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < helio_gpu_ctx::kPipeSets; ++i) {
    if (ctx->pipe[i]) {
      cudaStreamSynchronize(ctx->pipe[i]);
      cudaStreamDestroy(ctx->pipe[i]);
    }
    cudaFree(ctx->d_pl[i]);
    cudaFree(ctx->d_val[i]);
    cudaFree(ctx->d_st[i]);
    cudaFreeHost(ctx->h_pl_pin[i]);
    cudaFreeHost(ctx->h_val_pin[i]);
    cudaFreeHost(ctx->h_st_pin[i]);
  }
  for (int i = 0; i < helio_gpu_ctx::kSets; ++i) {
    cudaFree(ctx->d_ovf[i]);
    cudaFree(ctx->d_ovf2[i]);
    cudaFree(ctx->d_ovf3[i]);
  }
  cudaFree(ctx->d_glob);
  if (ctx->copy) {
    cudaStreamSynchronize(ctx->copy);
    cudaStreamDestroy(ctx->copy);
  }
  cudaFree(ctx->d_pl_all);
  cudaFree(ctx->d_val_all);
  cudaFree(ctx->d_st_all);
  for (cudaEvent_t e : ctx->ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev_out) cudaEventDestroy(e);
  cudaFree(ctx->d_cluster);
  cudaFree(ctx->d_kmax32);
  cudaFree(ctx->d_work);
  cudaFree(ctx->d_ovf_count);
  cudaFree(ctx->d_pv);
  cudaFree(ctx->d_pi);
  cudaFree(ctx->d_best);
  cudaFree(ctx->d_bidx);
  cudaFree(ctx->d_route);
  cudaFree(ctx->d_host_arena);
  cudaFreeHost(ctx->h_stage_pin);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->api_ev) cudaEventDestroy(ctx->api_ev);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* helio_gpu_last_error(const helio_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int helio_gpu_sync(helio_gpu_ctx* ctx) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < helio_gpu_ctx::kPipeSets; ++i) CK(cudaStreamSynchronize(ctx->pipe[i]));
  return HELIO_OK;
}

// K0 — compile a ClusterSpec into the device constants.  Same expressions as
// ClusterSpec::max_layers/throughput/nic_in/nic_out (cluster.cpp:62-100),
// compute_edge_capacity (flow_graph.cpp:38-43) and link_token_capacity
// (cluster.cpp:98-100).  Links that can never yield an edge (coordinator ->
// coordinator, self-links, undeclared endpoints) are dropped; duplicate
// (src, dst) links merge by capacity sum in declaration order, exactly as
// add_merged_edge does (flow_graph.cpp:25-34).
int helio_gpu_set_cluster(helio_gpu_ctx* ctx, const helio_cluster_desc* d, int32_t* k_out) {
  if (!ctx || !d) return fail(ctx, HELIO_ERR_INVALID, "null argument");
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  CK(cudaSetDevice(ctx->device));
  const int N = d->num_nodes, M = d->num_links, L = d->num_layers;
  if (N < 1 || N > 16000) return fail(ctx, HELIO_ERR_INVALID, "num_nodes must be in [1, 16000]");
  if (L < 1 || L > 32767) return fail(ctx, HELIO_ERR_INVALID, "num_layers must be in [1, 32767]");
  if (M < 0) return fail(ctx, HELIO_ERR_INVALID, "num_links must be >= 0");
  if (!d->vram_bytes || !d->kv_reserve || !d->peak_layer_tokens || !d->nic_in_bps || !d->nic_out_bps ||
      !d->lex_rank || (M > 0 && (!d->link_src || !d->link_dst || !d->link_bandwidth_bps)))
    return fail(ctx, HELIO_ERR_INVALID, "missing cluster array");
  std::vector<int> seen(N, 0);
  std::vector<int16_t> lexnode(N);
  for (int k = 0; k < N; ++k) {
    int r = d->lex_rank[k];
    if (r < 0 || r >= N || seen[r]) return fail(ctx, HELIO_ERR_INVALID, "lex_rank must be a permutation");
    seen[r] = 1;
    lexnode[r] = (int16_t)k;
  }
  for (int l = 0; l < M; ++l)
    if (d->link_src[l] < -2 || d->link_src[l] >= N || d->link_dst[l] < -2 || d->link_dst[l] >= N)
      return fail(ctx, HELIO_ERR_INVALID, "link endpoint index out of range");

  const double bpl = d->param_bytes / L;  // ModelSpec::bytes_per_layer
  std::vector<int32_t> kmax(N), cap_off(N);
  std::vector<double> cap_tab;
  std::vector<int16_t> kmax16(N);
  for (int k = 0; k < N; ++k) {
    double usable = d->vram_bytes[k] * (1.0 - d->kv_reserve[k]);
    double q = std::floor(usable / bpl);
    int kk = q > 1e9 ? 1000000000 : (q < -1e9 ? -1000000000 : (int)q);
    int tl = d->table_off ? d->table_off[k + 1] - d->table_off[k] : 0;
    if (tl > 0) kk = std::min(kk, tl);
    kk = std::min(kk, L);
    kmax[k] = kk;
    kmax16[k] = (int16_t)std::max(kk, -1);
    // nic_in / nic_out (cluster.cpp:82-96)
    double nin = d->nic_in_bps[k], nout = d->nic_out_bps[k];
    double inc = 0;
    for (int l = 0; l < M; ++l)
      if (d->link_src[l] == k || d->link_dst[l] == k) inc = host_max(inc, d->link_bandwidth_bps[l]);
    if (!(nin > 0)) nin = inc;
    if (!(nout > 0)) nout = inc;
    const double act = d->activation_bytes;
    const double nic_rate = host_min(nin, nout) / (8.0 * act);
    cap_off[k] = (int32_t)cap_tab.size();
    for (int j = 1; j <= kk; ++j) {
      double rate = tl > 0 ? d->table_val[d->table_off[k] + j - 1] : d->peak_layer_tokens[k] / j;
      cap_tab.push_back(host_min(rate, nic_rate));
    }
  }
  if (cap_tab.empty()) cap_tab.push_back(0.0);
  // compacted links
  std::map<std::pair<int, int>, int> dedup;
  std::vector<uint32_t> pack;
  std::vector<double> lcap;
  std::vector<double> cin(N, 0.0);
  for (int l = 0; l < M; ++l) {
    int a = d->link_src[l], b = d->link_dst[l];
    if (a == -2 || b == -2) continue;  // undeclared endpoint: never used (flow_graph.cpp:90,103,116)
    if (a == -1 && b == -1) continue;  // coordinator loop
    if (a >= 0 && a == b) continue;    // self-link: a.end < a.end never holds
    double payload = (a == -1 || b == -1) ? d->token_bytes : d->activation_bytes;
    double c = d->link_bandwidth_bps[l] / (8.0 * payload);
    auto key = std::make_pair(a, b);
    auto it = dedup.find(key);
    if (it != dedup.end()) {
      lcap[it->second] += c;
      continue;
    }
    dedup[key] = (int)pack.size();
    pack.push_back((uint32_t)(a + 1) | ((uint32_t)(b + 1) << 16));
    lcap.push_back(c);
  }
  for (size_t i = 0; i < pack.size(); ++i) {
    int a = (int)(pack[i] & 0xffffu) - 1, b = (int)(pack[i] >> 16) - 1;
    if (b == -1 && a >= 0) cin[a] = lcap[i];
  }
  const int Mv = (int)pack.size();
  // SCORE builder tables: per-node out-/in-link lists (other endpoint, link
  // index) over node<->node links, and each node's coordinator links.
  std::vector<int32_t> cout(N, -1), cinl(N, -1), obeg(N + 1, 0), ibeg(N + 1, 0);
  for (int i = 0; i < Mv; ++i) {
    int a = (int)(pack[i] & 0xffffu) - 1, b = (int)(pack[i] >> 16) - 1;
    if (a < 0) cout[b] = i;
    else if (b < 0) cinl[a] = i;
    else {
      obeg[a + 1]++;
      ibeg[b + 1]++;
    }
  }
  for (int k = 0; k < N; ++k) {
    obeg[k + 1] += obeg[k];
    ibeg[k + 1] += ibeg[k];
  }
  std::vector<int32_t> olist(2 * std::max(obeg[N], 1)), ilist(2 * std::max(ibeg[N], 1));
  {
    std::vector<int32_t> fo(N, 0), fi(N, 0);
    for (int i = 0; i < Mv; ++i) {
      int a = (int)(pack[i] & 0xffffu) - 1, b = (int)(pack[i] >> 16) - 1;
      if (a < 0 || b < 0) continue;
      int po = obeg[a] + fo[a]++, pi = ibeg[b] + fi[b]++;
      olist[2 * po] = b;
      olist[2 * po + 1] = i;
      ilist[2 * pi] = a;
      ilist[2 * pi + 1] = i;
    }
  }
  // walk generator adjacency: row 0 = coordinator's targets, row 1+k = node k's
  // (declared links, compacted order)
  std::vector<int32_t> wbeg(N + 2, 0), wlist;
  for (int row = -1; row < N; ++row) {
    wbeg[row + 1] = (int32_t)wlist.size();
    for (int i = 0; i < Mv; ++i) {
      int a = (int)(pack[i] & 0xffffu) - 1, b = (int)(pack[i] >> 16) - 1;
      if (a == row && b >= 0) wlist.push_back(b);
    }
  }
  wbeg[N + 1] = (int32_t)wlist.size();
  if (wlist.empty()) wlist.push_back(0);
  // N <= 64: node sets fit one 64-bit word; out-neighbour masks and a pair ->
  // link-index matrix drive the cover-mask SCORE builder.
  const bool small_n = N <= 64;
  std::vector<unsigned long long> outmask(small_n ? N : 1, 0ull);
  std::vector<int32_t> pairlink(small_n ? (size_t)N * N : 1, -1);
  // less_cout[b] = nodes whose coordinator->node link precedes b's (link order);
  // less_cin[a] likewise for node->coordinator links (PARITY small builder)
  std::vector<unsigned long long> less_cout(small_n ? N : 1, 0ull), less_cin(small_n ? N : 1, 0ull);
  if (small_n) {
    for (int i = 0; i < Mv; ++i) {
      int a = (int)(pack[i] & 0xffffu) - 1, b = (int)(pack[i] >> 16) - 1;
      if (a < 0 || b < 0) continue;
      outmask[a] |= 1ull << b;
      pairlink[(size_t)a * N + b] = i;
    }
    for (int x = 0; x < N; ++x)
      for (int y = 0; y < N; ++y) {
        if (cout[x] >= 0 && cout[y] >= 0 && cout[y] < cout[x]) less_cout[x] |= 1ull << y;
        if (cinl[x] >= 0 && cinl[y] >= 0 && cinl[y] < cinl[x]) less_cin[x] |= 1ull << y;
      }
  }
  // one device allocation for all constants
  auto al = [](size_t x) { return (x + 15) / 16 * 16; };
  size_t o_kmax = 0;
  size_t o_lexrank = o_kmax + al(2 * N);
  size_t o_lexnode = o_lexrank + al(4 * N);
  size_t o_capoff = o_lexnode + al(2 * N);
  size_t o_captab = o_capoff + al(4 * N);
  size_t o_pack = o_captab + al(8 * cap_tab.size());
  size_t o_lcap = o_pack + al(4 * std::max(Mv, 1));
  size_t o_cin = o_lcap + al(8 * std::max(Mv, 1));
  size_t o_cout = o_cin + al(8 * N);
  size_t o_cinl = o_cout + al(4 * N);
  size_t o_obeg = o_cinl + al(4 * N);
  size_t o_ibeg = o_obeg + al(4 * (N + 1));
  size_t o_olist = o_ibeg + al(4 * (N + 1));
  size_t o_ilist = o_olist + al(4 * olist.size());
  size_t o_omask = o_ilist + al(4 * ilist.size());
  size_t o_pair = o_omask + al(8 * outmask.size());
  size_t o_lcout = o_pair + al(4 * pairlink.size());
  size_t o_lcin = o_lcout + al(8 * less_cout.size());
  size_t o_wbeg = o_lcin + al(8 * less_cin.size());
  size_t o_wlist = o_wbeg + al(4 * wbeg.size());
  size_t total = o_wlist + al(4 * wlist.size());
  std::vector<char> hbuf(total, 0);
  std::memcpy(hbuf.data() + o_kmax, kmax16.data(), 2 * N);
  std::memcpy(hbuf.data() + o_lexrank, d->lex_rank, 4 * N);
  std::memcpy(hbuf.data() + o_lexnode, lexnode.data(), 2 * N);
  std::memcpy(hbuf.data() + o_capoff, cap_off.data(), 4 * N);
  std::memcpy(hbuf.data() + o_captab, cap_tab.data(), 8 * cap_tab.size());
  if (Mv) {
    std::memcpy(hbuf.data() + o_pack, pack.data(), 4 * Mv);
    std::memcpy(hbuf.data() + o_lcap, lcap.data(), 8 * Mv);
  }
  std::memcpy(hbuf.data() + o_cin, cin.data(), 8 * N);
  std::memcpy(hbuf.data() + o_cout, cout.data(), 4 * N);
  std::memcpy(hbuf.data() + o_cinl, cinl.data(), 4 * N);
  std::memcpy(hbuf.data() + o_obeg, obeg.data(), 4 * (N + 1));
  std::memcpy(hbuf.data() + o_ibeg, ibeg.data(), 4 * (N + 1));
  std::memcpy(hbuf.data() + o_olist, olist.data(), 4 * olist.size());
  std::memcpy(hbuf.data() + o_ilist, ilist.data(), 4 * ilist.size());
  std::memcpy(hbuf.data() + o_omask, outmask.data(), 8 * outmask.size());
  std::memcpy(hbuf.data() + o_pair, pairlink.data(), 4 * pairlink.size());
  std::memcpy(hbuf.data() + o_lcout, less_cout.data(), 8 * less_cout.size());
  std::memcpy(hbuf.data() + o_lcin, less_cin.data(), 8 * less_cin.size());
  std::memcpy(hbuf.data() + o_wbeg, wbeg.data(), 4 * wbeg.size());
  std::memcpy(hbuf.data() + o_wlist, wlist.data(), 4 * wlist.size());
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->d_cluster) cudaFree(ctx->d_cluster);
  if (ctx->d_kmax32) cudaFree(ctx->d_kmax32);
  ctx->d_cluster = nullptr;
  ctx->d_kmax32 = nullptr;
  CK(cudaMalloc(&ctx->d_cluster, total));
  CK(cudaMemcpy(ctx->d_cluster, hbuf.data(), total, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&ctx->d_kmax32, 4 * N));
  CK(cudaMemcpy(ctx->d_kmax32, kmax.data(), 4 * N, cudaMemcpyHostToDevice));
  char* base = static_cast<char*>(ctx->d_cluster);
  ctx->cd.N = N;
  ctx->cd.L = L;
  ctx->cd.Mv = Mv;
  {
    const char* ls = getenv("HELIO_LARGE_SOLVER");
    const char* gr = getenv("HELIO_PR_GR");
    ctx->cd.large_solver = (ls && atoi(ls) == 1) ? 1 : 0;
    ctx->cd.pr_gr = gr && atoi(gr) > 0 ? atoi(gr) : 20;
  }
  ctx->cd.kmax = reinterpret_cast<const int16_t*>(base + o_kmax);
  ctx->cd.lexrank = reinterpret_cast<const int32_t*>(base + o_lexrank);
  ctx->cd.lexnode = reinterpret_cast<const int16_t*>(base + o_lexnode);
  ctx->cd.cap_off = reinterpret_cast<const int32_t*>(base + o_capoff);
  ctx->cd.cap_tab = reinterpret_cast<const double*>(base + o_captab);
  ctx->cd.link_pack = reinterpret_cast<const uint32_t*>(base + o_pack);
  ctx->cd.link_cap = reinterpret_cast<const double*>(base + o_lcap);
  ctx->cd.cin_cap = reinterpret_cast<const double*>(base + o_cin);
  ctx->cd.cout_link = reinterpret_cast<const int32_t*>(base + o_cout);
  ctx->cd.cin_link = reinterpret_cast<const int32_t*>(base + o_cinl);
  ctx->cd.out_beg = reinterpret_cast<const int32_t*>(base + o_obeg);
  ctx->cd.in_beg = reinterpret_cast<const int32_t*>(base + o_ibeg);
  ctx->cd.out_list = reinterpret_cast<const int2*>(base + o_olist);
  ctx->cd.in_list = reinterpret_cast<const int2*>(base + o_ilist);
  ctx->cd.out_mask = small_n ? reinterpret_cast<const unsigned long long*>(base + o_omask) : nullptr;
  ctx->cd.pair_link = small_n ? reinterpret_cast<const int32_t*>(base + o_pair) : nullptr;
  ctx->cd.less_cout = small_n ? reinterpret_cast<const unsigned long long*>(base + o_lcout) : nullptr;
  ctx->cd.less_cin = small_n ? reinterpret_cast<const unsigned long long*>(base + o_lcin) : nullptr;
  ctx->d_walk_beg = reinterpret_cast<const int32_t*>(base + o_wbeg);
  ctx->d_walk_list = reinterpret_cast<const int32_t*>(base + o_wlist);
  ctx->h_walk_beg = wbeg;
  ctx->h_walk_list = wlist;
  ctx->N = N;
  ctx->L = L;
  ctx->Mv = Mv;
  ctx->h_kmax = kmax;
  ctx->h_cap_off = cap_off;
  ctx->h_cap_tab = cap_tab;
  ctx->h_lexrank.assign(d->lex_rank, d->lex_rank + N);
  ctx->h_vram.assign(d->vram_bytes, d->vram_bytes + N);
  ctx->bytes_per_layer = bpl;
  ctx->kv_token_layer_bytes =
      d->kv_bytes_per_token_layer > 0 ? d->kv_bytes_per_token_layer : 2.0 * d->activation_bytes;
  ctx->has_cluster = true;
  ctx->score_gen = 2 * N + 2 > 128;
  int rc = configure_layouts(ctx);
  if (rc) {
    ctx->has_cluster = false;
    return rc;
  }
  if (k_out) std::memcpy(k_out, kmax.data(), 4 * N);
  return HELIO_OK;
}

int helio_gpu_set_mode(helio_gpu_ctx* ctx, int mode) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (mode != HELIO_MODE_PARITY && mode != HELIO_MODE_SCORE) return fail(ctx, HELIO_ERR_INVALID, "unknown mode");
  ctx->mode = mode;
  return HELIO_OK;
}

int helio_gpu_get_mode(const helio_gpu_ctx* ctx) { return ctx ? ctx->mode : -1; }

int helio_gpu_compute_edge_capacity(const helio_gpu_ctx* ctx, int32_t node, int32_t j, double* out) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
  if (!ctx->has_cluster || !out) return HELIO_ERR_NO_CLUSTER;
  if (node < 0 || node >= ctx->N || j < 1 || j > ctx->h_kmax[node]) return HELIO_ERR_INVALID;
  *out = ctx->h_cap_tab[ctx->h_cap_off[node] + j - 1];
  return HELIO_OK;
}

int helio_gpu_score(helio_gpu_ctx* ctx, const int16_t* d_pl, int64_t B, int allow_partial,
                    double* d_values, int32_t* d_status, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (B < 0 || (B > 0 && (!d_pl || !d_values || !d_status))) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  FlowOut fo{nullptr, nullptr, nullptr, 0};
  CK(api_begin(ctx, st));
  const int rc = launch_score(ctx, helio_gpu_ctx::kApiSet, d_pl, B, allow_partial ? 1 : 0, d_values, d_status, st,
                              fo, true, ctx->mode);
  CK(api_end(ctx, st));
  return rc;
}

}  // extern "C"

namespace {
int argmax_on(helio_gpu_ctx* ctx, int scratch, const double* d_values, const int32_t* d_status, int64_t B,
              int64_t index_base, double* d_best, int64_t* d_index, cudaStream_t st);

// Pinned caller buffers and a batch that fits kResidentStageBytes: every
// chunk's H2D is issued up front on the copy stream into a device-resident
// copy of the batch (no staging reuse, so copies stream back to back at full
// link rate); chunk c's kernels on pipe[0] wait only for chunk c's copy, and
// its D2H runs on pipe[1] behind an event, off the kernel stream.
constexpr size_t kResidentStageBytes = size_t(2) << 30;

int score_host_resident(helio_gpu_ctx* ctx, const int16_t* h_pl, int64_t B, int allow_partial, double* h_values,
                        int32_t* h_status, double* h_best, int64_t* h_index, const std::vector<int64_t>& clo,
                        const std::vector<int64_t>& cn) {
  const size_t row = sizeof(int16_t) * 2 * ctx->N;
  const int64_t nchunks = (int64_t)clo.size();
  if (ctx->all_cap < B) {
    cudaFree(ctx->d_pl_all);
    cudaFree(ctx->d_val_all);
    cudaFree(ctx->d_st_all);
    ctx->d_pl_all = nullptr;
    ctx->d_val_all = nullptr;
    ctx->d_st_all = nullptr;
    ctx->all_cap = 0;
    CK(cudaMalloc(&ctx->d_pl_all, row * B));
    CK(cudaMalloc(&ctx->d_val_all, sizeof(double) * B));
    CK(cudaMalloc(&ctx->d_st_all, sizeof(int32_t) * B));
    ctx->all_cap = B;
  }
  while ((int64_t)ctx->ev_in.size() < nchunks) {
    cudaEvent_t a, b;
    CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    ctx->ev_in.push_back(a);
    ctx->ev_out.push_back(b);
  }
  for (int64_t c = 0; c < nchunks; ++c) {
    CK(cudaMemcpyAsync(ctx->d_pl_all + clo[c] * 2 * ctx->N, h_pl + clo[c] * 2 * ctx->N, row * cn[c],
                       cudaMemcpyHostToDevice, ctx->copy));
    CK(cudaEventRecord(ctx->ev_in[c], ctx->copy));
  }
  FlowOut fo{nullptr, nullptr, nullptr, 0};
  // kernels alternate between pipe[0] and pipe[2] (scratch sets 0 and 2) so
  // one chunk's tail overlaps the next chunk's start; D2H on pipe[1]
  cudaStream_t os = ctx->pipe[1];
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t lo = clo[c], n = cn[c];
    const int set = (c & 1) ? 2 : 0;
    cudaStream_t ks = ctx->pipe[set];
    CK(cudaStreamWaitEvent(ks, ctx->ev_in[c], 0));
    int rc = launch_score(ctx, set, ctx->d_pl_all + lo * 2 * ctx->N, n, allow_partial ? 1 : 0, ctx->d_val_all + lo,
                          ctx->d_st_all + lo, ks, fo, false, ctx->mode);
    if (rc) return rc;
    if (h_best) {
      rc = argmax_on(ctx, set, ctx->d_val_all + lo, ctx->d_st_all + lo, n, lo, ctx->d_best + c, ctx->d_bidx + c, ks);
      if (rc) return rc;
    }
    if (h_values) {
      CK(cudaEventRecord(ctx->ev_out[c], ks));
      CK(cudaStreamWaitEvent(os, ctx->ev_out[c], 0));
      CK(cudaMemcpyAsync(h_values + lo, ctx->d_val_all + lo, sizeof(double) * n, cudaMemcpyDeviceToHost, os));
      CK(cudaMemcpyAsync(h_status + lo, ctx->d_st_all + lo, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, os));
    }
  }
  CK(cudaStreamSynchronize(ctx->pipe[0]));
  CK(cudaStreamSynchronize(ctx->pipe[2]));
  CK(cudaStreamSynchronize(os));
  CK(cudaStreamSynchronize(ctx->copy));
  if (h_best) {
    std::vector<double> bv(nchunks);
    std::vector<int64_t> bi(nchunks);
    CK(cudaMemcpy(bv.data(), ctx->d_best, sizeof(double) * nchunks, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(bi.data(), ctx->d_bidx, sizeof(int64_t) * nchunks, cudaMemcpyDeviceToHost));
    double best = 0.0;
    int64_t idx = -1;
    for (int64_t c = 0; c < nchunks; ++c)  // chunks in index order: strict '>' keeps the first max
      if (bi[c] >= 0 && (idx < 0 || bv[c] > best)) {
        best = bv[c];
        idx = bi[c];
      }
    *h_best = best;
    if (h_index) *h_index = idx;
  }
  return HELIO_OK;
}

// Host-buffer scoring, pipelined over two streams in chunks: H2D of chunk c+1
// and D2H of chunk c-1 overlap the kernels of chunk c.  With pinned caller
// buffers everything is enqueued up front (no host waits until the end);
// pageable buffers go through pinned staging.  Optionally reduces the first
// maximum on the device per chunk (best/index).
int score_host_impl(helio_gpu_ctx* ctx, const int16_t* h_pl, int64_t B, int allow_partial, double* h_values,
                    int32_t* h_status, double* h_best, int64_t* h_index) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (B < 0 || (B > 0 && (!h_pl || (!h_values) != (!h_status) || (!h_values && !h_best))))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (B == 0) {
    if (h_best) *h_best = 0.0;
    if (h_index) *h_index = -1;
    return HELIO_OK;
  }
  CK(cudaSetDevice(ctx->device));
  // Chunks ramp up from 16k to 256k candidates: the first kernel starts after
  // a short H2D instead of a full chunk's, then copies hide behind kernels.
  const int64_t chunk = std::min<int64_t>(B, 1 << 18);
  std::vector<int64_t> clo, cn;
  for (int64_t lo = 0, sz = std::min<int64_t>(chunk, 1 << 14); lo < B; lo += sz, sz = std::min(chunk, 2 * sz)) {
    clo.push_back(lo);
    cn.push_back(std::min(sz, B - lo));
  }
  const int64_t nchunks = (int64_t)clo.size();
  if (h_best && nchunks > 2 * 4096) return fail(ctx, HELIO_ERR_TOO_LARGE, "batch too large for the best reduction");
  int rc = ensure_stage(ctx, chunk);
  if (rc) return rc;
  const bool pin_in = is_pinned(h_pl);
  const bool want_vals = h_values != nullptr;
  const bool pin_out = want_vals && is_pinned(h_values) && is_pinned(h_status);
  const size_t row = sizeof(int16_t) * 2 * ctx->N;
  FlowOut fo{nullptr, nullptr, nullptr, 0};
  if (pin_in && (!want_vals || pin_out) && (size_t)B * (row + 12) <= kResidentStageBytes)
    return score_host_resident(ctx, h_pl, B, allow_partial, h_values, h_status, h_best, h_index, clo, cn);
  for (int64_t c = 0; c < nchunks; ++c) {
    const int s = (int)(c % helio_gpu_ctx::kPipeSets);
    cudaStream_t st = ctx->pipe[s];
    const int64_t lo = clo[c], n = cn[c];
    if (c >= helio_gpu_ctx::kPipeSets && (!pin_in || (want_vals && !pin_out))) {
      // staging buffers of chunk c-3 are reused: retire it first
      CK(cudaStreamSynchronize(st));
      if (want_vals && !pin_out) {
        const int64_t plo = clo[c - helio_gpu_ctx::kPipeSets], pn = cn[c - helio_gpu_ctx::kPipeSets];
        stage_copy(h_values + plo, ctx->h_val_pin[s], sizeof(double) * pn);
        stage_copy(h_status + plo, ctx->h_st_pin[s], sizeof(int32_t) * pn);
      }
    }
    const void* src = h_pl + lo * 2 * ctx->N;
    if (!pin_in) {
      stage_copy(ctx->h_pl_pin[s], src, row * n);
      src = ctx->h_pl_pin[s];
    }
    CK(cudaMemcpyAsync(ctx->d_pl[s], src, row * n, cudaMemcpyHostToDevice, st));
    rc = launch_score(ctx, s, ctx->d_pl[s], n, allow_partial ? 1 : 0, ctx->d_val[s], ctx->d_st[s], st, fo,
                      false, ctx->mode);
    if (rc) return rc;
    if (h_best) {
      rc = argmax_on(ctx, s, ctx->d_val[s], ctx->d_st[s], n, lo, ctx->d_best + c, ctx->d_bidx + c, st);
      if (rc) return rc;
    }
    if (want_vals) {
      double* vdst = pin_out ? h_values + lo : ctx->h_val_pin[s];
      int32_t* sdst = pin_out ? h_status + lo : ctx->h_st_pin[s];
      CK(cudaMemcpyAsync(vdst, ctx->d_val[s], sizeof(double) * n, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(sdst, ctx->d_st[s], sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    }
  }
  const int64_t first_tail = (pin_in && (!want_vals || pin_out)) ? 0 : std::max<int64_t>(0, nchunks - helio_gpu_ctx::kPipeSets);
  for (int64_t c = first_tail; c < nchunks; ++c) {
    const int s = (int)(c % helio_gpu_ctx::kPipeSets);
    CK(cudaStreamSynchronize(ctx->pipe[s]));
    if (want_vals && !pin_out) {
      const int64_t lo = clo[c], n = cn[c];
      stage_copy(h_values + lo, ctx->h_val_pin[s], sizeof(double) * n);
      stage_copy(h_status + lo, ctx->h_st_pin[s], sizeof(int32_t) * n);
    }
  }
  if (h_best) {
    std::vector<double> bv(nchunks);
    std::vector<int64_t> bi(nchunks);
    CK(cudaMemcpy(bv.data(), ctx->d_best, sizeof(double) * nchunks, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(bi.data(), ctx->d_bidx, sizeof(int64_t) * nchunks, cudaMemcpyDeviceToHost));
    double best = 0.0;
    int64_t idx = -1;
    for (int64_t c = 0; c < nchunks; ++c)  // chunks in index order: strict '>' keeps the first max
      if (bi[c] >= 0 && (idx < 0 || bv[c] > best)) {
        best = bv[c];
        idx = bi[c];
      }
    *h_best = best;
    if (h_index) *h_index = idx;
  }
  return HELIO_OK;
}
}  // namespace

extern "C" {

int helio_gpu_score_host(helio_gpu_ctx* ctx, const int16_t* h_pl, int64_t B, int allow_partial,
                         double* h_values, int32_t* h_status) {
  if (!h_values || !h_status) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  return score_host_impl(ctx, h_pl, B, allow_partial, h_values, h_status, nullptr, nullptr);
}

int helio_gpu_score_best_host(helio_gpu_ctx* ctx, const int16_t* h_pl, int64_t B, int allow_partial,
                              double* h_values, int32_t* h_status, double* h_best, int64_t* h_index) {
  if (!h_best || !h_index) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  return score_host_impl(ctx, h_pl, B, allow_partial, h_values, h_status, h_best, h_index);
}

int helio_gpu_flows_host(helio_gpu_ctx* ctx, const int16_t* h_pl, int64_t K, int allow_partial,
                         int32_t max_edges, int32_t* h_nv, int32_t* h_ne, helio_edge* h_edges,
                         double* h_values, int32_t* h_status) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (K <= 0) return HELIO_OK;
  if (!h_pl || !h_nv || !h_ne || !h_values || !h_status || max_edges < 0 || (max_edges > 0 && !h_edges))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t row = sizeof(int16_t) * 2 * ctx->N;
  const size_t ne_alloc = (size_t)K * std::max(max_edges, 1);
  auto carve = [&](Carve& c, int16_t*& pl, double*& val, int32_t*& sts, int32_t*& nv, int32_t*& ne,
                   helio_edge*& ed) {
    pl = c.take<int16_t>(2 * ctx->N * (size_t)K);
    val = c.take<double>(K);
    sts = c.take<int32_t>(K);
    nv = c.take<int32_t>(K);
    ne = c.take<int32_t>(K);
    ed = c.take<helio_edge>(ne_alloc);
  };
  int16_t* d_pl;
  double* d_val;
  int32_t *d_st, *d_nv, *d_ne;
  helio_edge* d_ed;
  Carve measure;
  carve(measure, d_pl, d_val, d_st, d_nv, d_ne, d_ed);
  Carve c;
  int rc = host_arena(ctx, measure.off, &c.base);
  if (rc) return rc;
  carve(c, d_pl, d_val, d_st, d_nv, d_ne, d_ed);
  CK(api_begin(ctx, st));
  // small calls (the per-call entries) go through the pinned staging buffer
  // both ways: the outputs are one carved range, copied back in one DMA
  const char* d_first = reinterpret_cast<const char*>(d_val);
  const size_t span = (size_t)(reinterpret_cast<const char*>(d_ed + ne_alloc) - d_first);
  char* pin = nullptr;
  const bool staged = span <= (size_t(32) << 20) && host_pin(ctx, std::max(span, row * K), &pin) == HELIO_OK;
  if (staged) {
    std::memcpy(pin, h_pl, row * K);
    CK(cudaMemcpyAsync(d_pl, pin, row * K, cudaMemcpyHostToDevice, st));
  } else {
    CK(cudaMemcpyAsync(d_pl, h_pl, row * K, cudaMemcpyHostToDevice, st));
  }
  FlowOut fo{d_ed, d_nv, d_ne, max_edges};
  rc = launch_score(ctx, helio_gpu_ctx::kApiSet, d_pl, K, allow_partial ? 1 : 0, d_val, d_st, st, fo, false,
                    HELIO_MODE_PARITY);
  CK(api_end(ctx, st));
  if (rc) return rc;
  // the outputs are one carved range: a single DMA into pinned staging, then
  // host copies (one round trip instead of five pageable copies; only each
  // candidate's ne edges are copied out)
  if (!staged) {  // large batches: direct copies
    CK(cudaMemcpyAsync(h_values, d_val, 8 * K, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_status, d_st, 4 * K, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_nv, d_nv, 4 * K, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_ne, d_ne, 4 * K, cudaMemcpyDeviceToHost, st));
    if (max_edges > 0)
      CK(cudaMemcpyAsync(h_edges, d_ed, sizeof(helio_edge) * (size_t)K * max_edges, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HELIO_OK;
  }
  CK(cudaMemcpyAsync(pin, d_first, span, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  auto at = [&](const void* d) { return pin + (reinterpret_cast<const char*>(d) - d_first); };
  std::memcpy(h_values, at(d_val), 8 * K);
  std::memcpy(h_status, at(d_st), 4 * K);
  std::memcpy(h_nv, at(d_nv), 4 * K);
  std::memcpy(h_ne, at(d_ne), 4 * K);
  if (max_edges > 0) {
    const helio_edge* src = reinterpret_cast<const helio_edge*>(at(d_ed));
    for (int64_t k = 0; k < K; ++k) {
      const int64_t n = std::min<int64_t>(std::max<int32_t>(h_ne[k], 0), max_edges);
      std::memcpy(h_edges + k * max_edges, src + k * max_edges, sizeof(helio_edge) * n);
    }
  }
  return HELIO_OK;
}

int helio_gpu_maxflow_raw_host(helio_gpu_ctx* ctx, int64_t G, const int32_t* h_n, const int32_t* h_s,
                               const int32_t* h_t, const int64_t* h_off, const int32_t* h_u,
                               const int32_t* h_v, const double* h_cap, double* h_values,
                               double* h_flows) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (G <= 0) return HELIO_OK;
  if (!h_n || !h_s || !h_t || !h_off || !h_values) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  int nmax = 1, mmax = 0;
  const int64_t Etot = h_off[G] - h_off[0];
  if (h_off[0] != 0) return fail(ctx, HELIO_ERR_INVALID, "edge_off[0] must be 0");
  if (Etot > 0 && (!h_u || !h_v || !h_cap)) return fail(ctx, HELIO_ERR_INVALID, "bad edge buffers");
  for (int64_t g = 0; g < G; ++g) {
    const int n = h_n[g];
    const int64_t m = h_off[g + 1] - h_off[g];
    if (n < 1 || m < 0) return fail(ctx, HELIO_ERR_INVALID, "graph needs n >= 1 and m >= 0");
    if (h_s[g] < 0 || h_s[g] >= n || h_t[g] < 0 || h_t[g] >= n)
      return fail(ctx, HELIO_ERR_INVALID, "source/sink out of range");
    for (int64_t i = h_off[g]; i < h_off[g + 1]; ++i)
      if (h_u[i] < 0 || h_u[i] >= n || h_v[i] < 0 || h_v[i] >= n)
        return fail(ctx, HELIO_ERR_INVALID, "edge endpoint out of range");
    nmax = std::max(nmax, n);
    mmax = (int)std::max<int64_t>(mmax, m);
  }
  if (nmax > 16000 || 2 * (int64_t)mmax > 32766)
    return fail(ctx, HELIO_ERR_TOO_LARGE, "raw graph exceeds the device limits (V <= 16000, 2E <= 32766)");
  Layout lay = make_layout(nmax, std::max(2 * mmax, 2), 0, std::max(mmax, 1));
  const size_t max_smem = 227 * 1024;
  // graphs larger than one SM's shared memory: one-warp CTAs whose slots live
  // in global memory (L1/L2 cached), carved from the host-entry arena below
  const bool in_global = (size_t)lay.bytes > max_smem;
  int warps = in_global ? 1 : (int)std::max<size_t>(1, std::min<size_t>(4, max_smem / lay.bytes));
  int per_sm = 2;
  if (!in_global) {
    CK(cudaFuncSetAttribute(raw_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem));
    CK(cudaFuncSetAttribute(raw_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raw_kernel<false>, 32 * warps, lay.bytes * warps));
    if (per_sm < 1) per_sm = 1;
  }
  const int grid = (int)std::min<int64_t>((int64_t)per_sm * ctx->sm_count, (G + warps - 1) / warps);
  cudaStream_t st = ctx->stream;
  const int64_t Ea = std::max<int64_t>(Etot, 1);
  auto carve = [&](Carve& c, int32_t*& n, int32_t*& s, int32_t*& t, int64_t*& off, int32_t*& u, int32_t*& v,
                   double*& cap, double*& val, double*& fl) {
    n = c.take<int32_t>(G);
    s = c.take<int32_t>(G);
    t = c.take<int32_t>(G);
    off = c.take<int64_t>(G + 1);
    u = c.take<int32_t>(Ea);
    v = c.take<int32_t>(Ea);
    cap = c.take<double>(Ea);
    val = c.take<double>(G);
    fl = c.take<double>(h_flows ? Ea : 1);
  };
  int32_t *d_n, *d_s, *d_t, *d_u, *d_v;
  int64_t* d_off;
  double *d_cap, *d_val, *d_fl;
  char* d_slots = nullptr;
  Carve measure;
  carve(measure, d_n, d_s, d_t, d_off, d_u, d_v, d_cap, d_val, d_fl);
  if (in_global) measure.take<char>((size_t)grid * lay.bytes);
  Carve c;
  int rc = host_arena(ctx, measure.off, &c.base);
  if (rc) return rc;
  carve(c, d_n, d_s, d_t, d_off, d_u, d_v, d_cap, d_val, d_fl);
  if (in_global) d_slots = c.take<char>((size_t)grid * lay.bytes);
  if (!h_flows) d_fl = nullptr;
  CK(api_begin(ctx, st));
  CK(cudaMemcpyAsync(d_n, h_n, 4 * G, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_s, h_s, 4 * G, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_t, h_t, 4 * G, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_off, h_off, 8 * (G + 1), cudaMemcpyHostToDevice, st));
  if (Etot > 0) {
    CK(cudaMemcpyAsync(d_u, h_u, 4 * Etot, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_v, h_v, 4 * Etot, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_cap, h_cap, 8 * Etot, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(ctx->d_work, 0, sizeof(unsigned long long), st));
  if (in_global)
    raw_kernel<true><<<grid, 32, 0, st>>>(lay, G, d_n, d_s, d_t, d_off, d_u, d_v, d_cap, d_val, d_fl, ctx->d_work,
                                          d_slots);
  else
    raw_kernel<false><<<grid, 32 * warps, lay.bytes * warps, st>>>(lay, G, d_n, d_s, d_t, d_off, d_u, d_v, d_cap,
                                                                    d_val, d_fl, ctx->d_work, nullptr);
  CK(cudaGetLastError());
  CK(api_end(ctx, st));
  ctx->launches++;
  CK(cudaMemcpyAsync(h_values, d_val, 8 * G, cudaMemcpyDeviceToHost, st));
  if (h_flows && Etot > 0) CK(cudaMemcpyAsync(h_flows, d_fl, 8 * Etot, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HELIO_OK;
}

}  // extern "C"

namespace {
int argmax_on(helio_gpu_ctx* ctx, int scratch, const double* d_values, const int32_t* d_status, int64_t B,
              int64_t index_base, double* d_best, int64_t* d_index, cudaStream_t st) {
  const int P = (int)std::min<int64_t>(std::max<int64_t>((B + 255) / 256, 1), 2 * ctx->sm_count);
  double* pv = ctx->d_pv + 4096 * scratch;
  long long* pi = ctx->d_pi + 4096 * scratch;
  argmax_partial<<<P, 256, 0, st>>>(d_values, d_status, B, pv, pi);
  argmax_final<<<1, 32, 0, st>>>(pv, pi, P, index_base, d_best, d_index);
  CK(cudaGetLastError());
  ctx->launches += 2;
  return HELIO_OK;
}
}  // namespace

// The device argmax on the argmax scratch row (multi.cu's ranked argmax).
int helio_engine_argmax(helio_gpu_ctx* ctx, const double* d_values, const int32_t* d_status, int64_t B,
                        int64_t index_base, double* d_best, int64_t* d_index, cudaStream_t st) {
  return argmax_on(ctx, helio_gpu_ctx::kSets, d_values, d_status, B, index_base, d_best, d_index, st);
}

extern "C" {

int helio_gpu_argmax(helio_gpu_ctx* ctx, const double* d_values, const int32_t* d_status, int64_t B,
                     int64_t index_base, double* d_best, int64_t* d_index, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!d_best || !d_index || (B > 0 && (!d_values || !d_status))) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  CK(api_begin(ctx, st));
  const int rc = argmax_on(ctx, helio_gpu_ctx::kSets, d_values, d_status, B, index_base, d_best, d_index, st);
  CK(api_end(ctx, st));
  return rc;
}

int helio_gpu_generate(helio_gpu_ctx* ctx, uint64_t seed, int64_t first, int64_t B, uint32_t ppm,
                       int16_t* d_out, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (ctx->N > GEN_MAX_N) return fail(ctx, HELIO_ERR_TOO_LARGE, "generator supports up to 1024 nodes");
  if (B <= 0) return HELIO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  int grid = (int)std::min<int64_t>((B + 127) / 128, 8 * ctx->sm_count);
  gen_kernel<<<grid, 128, 0, st>>>(ctx->d_kmax32, ctx->N, ctx->L, seed, first, B, ppm, d_out);
  CK(cudaGetLastError());
  ctx->launches++;
  return HELIO_OK;
}

int helio_gpu_generate_walk(helio_gpu_ctx* ctx, uint64_t seed, int64_t first, int64_t B, int16_t* d_out,
                            void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (ctx->N > GEN_MAX_N) return fail(ctx, HELIO_ERR_TOO_LARGE, "generator supports up to 1024 nodes");
  if (B <= 0) return HELIO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  int grid = (int)std::min<int64_t>((B + 127) / 128, 8 * ctx->sm_count);
  gen_walk_kernel<<<grid, 128, 0, st>>>(ctx->d_kmax32, ctx->N, ctx->L, seed, first, B, ctx->d_walk_beg,
                                        ctx->d_walk_list, d_out);
  CK(cudaGetLastError());
  ctx->launches++;
  return HELIO_OK;
}

int helio_gpu_generate_walk_host(const helio_gpu_ctx* ctx, uint64_t seed, int64_t first, int64_t B,
                                 int16_t* h_out) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
  if (!ctx->has_cluster || (B > 0 && !h_out)) return HELIO_ERR_INVALID;
  std::vector<uint32_t> used((ctx->N + 31) / 32 + 1);
  for (int64_t i = 0; i < B; ++i)
    hg_candidate_walk(ctx->h_kmax.data(), ctx->N, ctx->L, seed, (uint64_t)(first + i), ctx->h_walk_beg.data(),
                      ctx->h_walk_list.data(), used.data(), h_out + i * 2 * ctx->N);
  return HELIO_OK;
}

void helio_generate_host(const int32_t* k, int32_t N, int32_t L, uint64_t seed, int64_t first,
                         int64_t B, uint32_t ppm, int16_t* h_out) {
  std::vector<int16_t> perm(N > 0 ? N : 1);
  for (int64_t i = 0; i < B; ++i)
    hg_candidate(k, N, L, seed, (uint64_t)(first + i), ppm, perm.data(), h_out + i * 2 * N);
}

int64_t helio_gpu_launch_count(const helio_gpu_ctx* ctx) { return ctx ? ctx->launches : 0; }

double helio_gpu_last_kernel_ms(const helio_gpu_ctx* ctx) {
  if (!ctx || !ctx->timed) return -1.0;
  float ms = -1.0f;
  if (cudaEventSynchronize(ctx->ev1) != cudaSuccess) return -1.0;
  if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) != cudaSuccess) return -1.0;
  return ms;
}

}  // extern "C"
