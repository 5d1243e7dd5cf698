// route.cu — K3: IWRR per-request route sampling on the GPU.
//
// Reference: iwrr_weights (scheduler.cpp:46-56), IwrrPicker::next (:28-44),
// Scheduler ctor / admit / complete (:58-190), driven in the AC8 order
// (acceptance_main.cpp:529-537): admit(r, in[r]); if admitted complete(r, out[r]).
//
// Closed form (the fast path).  With every hop eligible, IwrrPicker::next at
// vertex x returns cycle_x[k mod W_x] on its k-th call, where cycle_x is one
// full (round, index) sweep and W_x = sum of the weights.  In the AC8 order a
// request's picks happen before the next request's, so the k-th pick at x
// belongs to the request of rank k among those that reach x.  Every plan edge
// goes from a node to one with a strictly larger end layer (flow_graph.cpp:121),
// so processing vertices in end-layer order makes routing level-synchronous:
// for each vertex, a stable rank (exclusive scan) of the requests waiting there
// picks their out-edge.  KV masking can only bind when some hop's charge
// (scheduler.cpp:100-108) may exceed 0.9 * kv_cap; in the AC8 order every
// charge is released before the next admit, so the host checks that bound with
// the largest possible running mean of output lengths.  If it may bind (or the
// plan's exec intervals are not node-consistent) the exact replay runs instead:
// one warp walking the device-built cycles with the state in shared memory
// (route_masked_warp).
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <cmath>
#include <vector>

#include "engine.h"

using namespace helio_engine;

namespace {

constexpr int kDone = -1;

// iwrr_weights (scheduler.cpp:46-56) for every vertex, then its IWRR cycle.
__global__ void route_setup(int nv, const int32_t* __restrict__ obeg, const double* __restrict__ flow,
                            long long* __restrict__ w, const int32_t* __restrict__ cyc_off,
                            int16_t* __restrict__ cyc, long long* __restrict__ wmax_out,
                            int32_t* __restrict__ cyc_len) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nv) return;
  const int b = obeg[x], e = obeg[x + 1];
  long long wmax = 0;
  for (int i = b; i < e; ++i) {
    long long v = llround(1000.0 * flow[i]);
    w[i] = v > 1 ? v : 1;
    wmax = w[i] > wmax ? w[i] : wmax;
  }
  if (wmax > 32) {
    for (int i = b; i < e; ++i) {
      long long v = llround(w[i] * 32.0 / wmax);
      w[i] = v > 1 ? v : 1;
    }
  }
  long long wm = 1;  // IwrrPicker ctor: wmax_ starts at 1
  for (int i = b; i < e; ++i) wm = w[i] > wm ? w[i] : wm;
  wmax_out[x] = wm;
  int p = cyc_off[x];
  for (long long r = 1; r <= wm; ++r)
    for (int i = b; i < e; ++i)
      if (w[i] >= r) cyc[p++] = (int16_t)(i - b);
  cyc_len[x] = p - cyc_off[x];  // W_x = sum of the weights
}

__global__ void route_init(int64_t R, int32_t* cur, int32_t* nh, int16_t* cov) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    cur[r] = 0;
    nh[r] = 0;
    cov[r] = 0;
  }
}

__global__ void route_flag(int64_t R, int x, const int32_t* __restrict__ cur, int32_t* __restrict__ flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x)
    flag[r] = cur[r] == x ? 1 : 0;
}

__global__ void route_apply(int64_t R, int x, int L, int max_hops, const int32_t* __restrict__ obeg,
                            const int32_t* __restrict__ odst, const int32_t* __restrict__ oes,
                            const int32_t* __restrict__ oee, const int32_t* __restrict__ node_of,
                            const int32_t* __restrict__ cyc_off, const int32_t* __restrict__ cyc_len,
                            const int16_t* __restrict__ cyc, const int32_t* __restrict__ rank, int32_t* cur, int32_t* nh, int16_t* cov,
                            int32_t* hop_node, int32_t* hop_s, int32_t* hop_e, int* err) {
  const int b = obeg[x], deg = obeg[x + 1] - b;
  const int W = cyc_len[x];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (cur[r] != x) continue;
    if (deg == 0) {  // IwrrPicker::next on no candidates returns -1: deferred
      cur[r] = kDone;
      nh[r] = -1;
      continue;
    }
    const int i = cyc[cyc_off[x] + (int)(rank[r] % W)];
    const int e = b + i;
    const int d = odst[e];
    if (d == 0 || oes[e] != cov[r]) {  // scheduler.cpp:170-171
      atomicExch(err, 1);
      cur[r] = kDone;
      continue;
    }
    const int h = nh[r];
    if (h < max_hops) {
      hop_node[r * max_hops + h] = node_of[d];
      if (hop_s) {
        hop_s[r * max_hops + h] = oes[e];
        hop_e[r * max_hops + h] = oee[e];
      }
    }
    nh[r] = h + 1;
    cov[r] = (int16_t)oee[e];
    cur[r] = oee[e] >= L ? kDone : d;
  }
}

// Exact replay of Scheduler::admit/complete in the AC8 order when KV masking
// may bind.  One warp, state in shared memory.  In the AC8 order every charge
// is released (complete, or the rollback of a deferral) before the next
// admit, and a route visits a vertex at most once (exec ranges strictly
// increase), so at every eligibility test kv_est[d] is exactly 0.0 (b - b ==
// 0 in IEEE arithmetic) and the reference's test (scheduler.cpp:105-108)
// reduces to  (in_len + avg) * kvb * (exec_end - exec_start) <= 0.9 *
// kv_cap[d]  — the same double operations in the same order.  The serial
// state is each vertex's picker position plus the running output mean; the
// warp scans 32 cycle slots per step (ballot, first eligible lane), and the
// division of the next mean update is issued before the route is walked
// (it does not depend on it).  A deferred request leaves the positions it
// advanced, as IwrrPicker::next does (scheduler.cpp:165-168 rolls back only
// the KV charges).
// One 32-byte record per cycle slot: the slot's edge (threshold 0.9 *
// kv_cap[dst] — +inf for the coordinator — and exec length, as doubles; dst,
// exec range and the node of dst) and the next slot of the cycle, so a pick is
// one shuffle (the vertex's current slot) and one record load.
struct alignas(16) SlotRec {
  double thr, len;
  int32_t next, dst, ee, es_node;  // es_node = exec_start | node << 16
};

// The running output mean's update (scheduler.cpp:183-190) is the serial
// dependence of the replay: avg += (out - avg) / n.  The division is split:
// y = RN(1/n) (a correctly rounded reciprocal, __drcp_rn) depends only on the
// sample count and is computed ahead, 32 counts at a time in parallel; the
// quotient is then q0 = RN(a*y), r = a - n*q0 (exact, fma), q = RN(q0 + r*y)
// — the correctly rounded a/n for normal operands (Markstein's theorem; the
// same final step as the IEEE division sequence), i.e. the reference's bits.
// tests/test_gpu_parity.py checks it against '/' on 1e8 operand pairs of the
// routing domain (helio_gpu_check_division) and end to end on 1M requests.
__device__ __forceinline__ double div_by_count(double a, double n, double y) {
  const double q0 = __dmul_rn(a, y);
  const double r = __fma_rn(-n, q0, a);
  return __fma_rn(r, y, q0);
}

// REG: vertex x's current absolute slot lives in lane x's register (plans up
// to 32 vertices — the coordinator plus up to 31 placed nodes); otherwise in
// shared memory.  CHECKS: the reference's tiling checks per hop
// (scheduler.cpp:170-171); the host drops them for plans whose exec ranges
// are node-consistent, where they cannot fail.
template <bool REG, bool CHECKS>
__global__ void route_masked_warp(int64_t R, int nv, int L, int max_hops, double kvb,
                                  const int32_t* __restrict__ obeg, const int32_t* __restrict__ odst,
                                  const int32_t* __restrict__ oes, const int32_t* __restrict__ oee,
                                  const int32_t* __restrict__ node_of, const double* __restrict__ kv_cap,
                                  const int32_t* __restrict__ cyc_len, const int16_t* __restrict__ cyc,
                                  const int32_t* __restrict__ in_len, const int32_t* __restrict__ out_len,
                                  int32_t* nh, int32_t* hop_node, int32_t* hop_s, int32_t* hop_e,
                                  long long* deferred, int* err) {
  extern __shared__ __align__(16) char sm[];
  const int lane = threadIdx.x;
  int32_t* vcur = reinterpret_cast<int32_t*>(sm);  // [nv] current slot (-1: no out-edges)
  int2* vgeo = reinterpret_cast<int2*>(sm + (((size_t)4 * nv + 7) & ~size_t(7)));  // [nv] (base, W)
  SlotRec* rec = reinterpret_cast<SlotRec*>(sm + ((((size_t)4 * nv + 7) & ~size_t(7)) + 8 * (size_t)nv + 15 & ~size_t(15)));
  int my_cur = -1;
  for (int x = 0, base = 0; x < nv; ++x) {
    const int W = obeg[x + 1] > obeg[x] ? cyc_len[x] : 0;
    if (REG && lane == x) my_cur = W ? base : -1;
    if (lane == 0) {
      if (!REG) vcur[x] = W ? base : -1;
      vgeo[x] = make_int2(base, W);
    }
    for (int k = lane; k < W; k += 32) {
      const int e = obeg[x] + cyc[32 * obeg[x] + k];
      const int d = odst[e];
      SlotRec r;
      r.thr = d == 0 ? 1.0e308 : 0.9 * kv_cap[d];
      r.len = (double)(oee[e] - oes[e]);
      r.next = k + 1 == W ? base : base + k + 1;
      r.dst = d;
      r.ee = oee[e];
      r.es_node = (oes[e] & 0xffff) | (node_of[d] << 16);
      rec[base + k] = r;
    }
    base += W;
  }
  __syncwarp();
  double avg = 232.0, samples = 1.0;
  long long den = 0;
  const bool store_hops = max_hops > 0;
  for (int64_t r0 = 0; r0 < R; r0 += 32) {
    const int nb = R - r0 < 32 ? (int)(R - r0) : 32;
    const int my_in = lane < nb ? in_len[r0 + lane] : 0;
    const int my_out = lane < nb ? out_len[r0 + lane] : 0;
    // reciprocals of the next 32 sample counts (each admission takes one)
    const double my_y = __drcp_rn(samples + 1.0 + lane);
    int admitted = 0;
    int my_nh = 0;
    for (int j = 0; j < nb; ++j) {
      const int in = __shfl_sync(0xffffffffu, my_in, j);
      const double tk = ((double)in + avg) * kvb;  // hop_charge = tk * (exec_end - exec_start)
      int32_t* hp = hop_node + (r0 + j) * max_hops;
      int v = 0, covered = 0, h = 0;
      bool ok = true;
      do {
        const int slot = REG ? __shfl_sync(0xffffffffu, my_cur, v) : vcur[v];
        if (slot < 0) {  // no out-edges: IwrrPicker::next returns -1
          ok = false;
          break;
        }
        SlotRec rc = rec[slot];
        if (!(tk * rc.len <= rc.thr)) {
          // the rest of one full cycle, 32 slots at a time
          const int2 geo = vgeo[v];
          const int base = geo.x, W = geo.y, p = slot - base;
          int pick = -1;
          for (int k0 = 1; k0 < W; k0 += 32) {
            const int k = k0 + lane;
            bool el = false;
            int sl = 0;
            if (k < W) {
              const int q = p + k;
              sl = base + (q >= W ? q - W : q);
              el = tk * rec[sl].len <= rec[sl].thr;
            }
            const unsigned m = __ballot_sync(0xffffffffu, el);
            if (m) {
              pick = __shfl_sync(0xffffffffu, sl, __ffs(m) - 1);
              break;
            }
          }
          if (pick < 0) {  // one full cycle with nothing eligible: position unchanged
            ok = false;
            break;
          }
          rc = rec[pick];
        }
        const int es = rc.es_node & 0xffff;
        if (CHECKS && (rc.dst == 0 || es != covered)) {  // scheduler.cpp:170-171
          if (lane == 0) atomicExch(err, 1);
          return;
        }
        if (REG) {
          if (lane == v) my_cur = rc.next;
        } else {
          if (lane == 0) vcur[v] = rc.next;
          __syncwarp();
        }
        if (store_hops && lane == 0 && h < max_hops) {
          hp[h] = rc.es_node >> 16;
          if (hop_s) {
            hop_s[(r0 + j) * max_hops + h] = es;
            hop_e[(r0 + j) * max_hops + h] = rc.ee;
          }
        }
        ++h;
        covered = rc.ee;
        v = rc.dst;
      } while (covered < L);
      if (ok) {  // complete(): the running mean (scheduler.cpp:183-190)
        const int out = __shfl_sync(0xffffffffu, my_out, j);
        const double y = __shfl_sync(0xffffffffu, my_y, admitted);
        samples += 1.0;
        avg += div_by_count((double)out - avg, samples, y);
        ++admitted;
      } else {
        ++den;
      }
      if (lane == j) my_nh = ok ? h : -1;
    }
    if (lane < nb) nh[r0 + lane] = my_nh;
  }
  if (lane == 0) *deferred = den;
}

// Self-test of div_by_count against IEEE division on the routing domain:
// numerators a = out - avg (|a| < 4096, random significands), denominators
// n = sample counts up to 2^27.
__global__ void check_division_kernel(int64_t count, uint64_t seed, unsigned long long* mismatches) {
  unsigned long long bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double n = (double)(1 + (z & ((1ull << 27) - 1)));
    const int out = (int)((z >> 27) & 2047);
    const double avg = (double)((z >> 38) & ((1ull << 26) - 1)) * (2048.0 / (double)(1ull << 26));
    const double a = (double)out - avg;
    const double y = __drcp_rn(n);
    if (div_by_count(a, n, y) != a / n) ++bad;
  }
  atomicAdd(mismatches, bad);
}

// Route buffers are carved from one context-owned device arena that only
// grows, so steady-state calls make no cudaMalloc/cudaFree.
struct Arena {
  helio_gpu_ctx* ctx;
  size_t off = 0;
  bool sizing = true;
  template <typename T>
  int take(T** p, size_t n) {
    const size_t bytes = (sizeof(T) * std::max<size_t>(n, 1) + 255) / 256 * 256;
    if (!sizing) *p = reinterpret_cast<T*>(static_cast<char*>(ctx->d_route) + off);
    off += bytes;
    return HELIO_OK;
  }
};

}  // namespace

extern "C" int helio_gpu_route_host(helio_gpu_ctx* ctx, const int16_t* h_pl,
                                    const helio_plan_edge* pe, int32_t ne, int64_t R,
                                    const int32_t* h_in, const int32_t* h_out, int32_t max_hops,
                                    int32_t* h_nh, int32_t* h_hn, int32_t* h_hs, int32_t* h_he,
                                    int64_t* h_deferred) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (!h_pl || (ne > 0 && !pe) || R < 0 || max_hops < 0 || (R > 0 && (!h_in || !h_out || !h_nh)) ||
      (R > 0 && max_hops > 0 && (!h_hn || (!h_hs) != (!h_he))))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  const int N = ctx->N, L = ctx->L;
  // Scheduler ctor (scheduler.cpp:58-98): vertex 0 = coordinator, then the
  // plan's non-empty nodes in id order.
  if (ne <= 0) return fail(ctx, HELIO_ERR_INVALID, "plan has no flow edges to schedule on");
  std::vector<int> order(N);
  for (int k = 0; k < N; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return ctx->h_lexrank[a] < ctx->h_lexrank[b]; });
  std::vector<int> vof(N, -1);
  std::vector<int32_t> node_of(1, -1);
  std::vector<double> kv_cap(1, 0.0);
  std::vector<int> vend(1, 0);
  for (int k : order) {
    const int s = h_pl[2 * k], e = h_pl[2 * k + 1];
    if (e <= s) continue;
    vof[k] = (int)node_of.size();
    node_of.push_back(k);
    const double held = e - s;
    const double cap = ctx->h_vram[k] - (e - s) * ctx->bytes_per_layer;
    (void)held;
    kv_cap.push_back(0.0 < cap ? cap : 0.0);
    vend.push_back(e);
  }
  const int nv = (int)node_of.size();
  std::vector<int> esrc(ne), edst(ne);
  for (int i = 0; i < ne; ++i) {
    const int a = pe[i].src_node, b = pe[i].dst_node;
    if (a < -1 || a >= N || b < -1 || b >= N)
      return fail(ctx, HELIO_ERR_INVALID, "plan edge endpoint out of range");
    const int va = a < 0 ? 0 : vof[a], vb = b < 0 ? 0 : vof[b];
    if (va < 0 || vb < 0) return fail(ctx, HELIO_ERR_INVALID, "plan edge references an unplaced node");
    esrc[i] = va;
    edst[i] = vb;
  }
  std::vector<int32_t> obeg(nv + 1, 0), odst(ne), oes(ne), oee(ne);
  std::vector<double> oflow(ne);
  for (int i = 0; i < ne; ++i) obeg[esrc[i] + 1]++;
  for (int x = 0; x < nv; ++x) obeg[x + 1] += obeg[x];
  if (obeg[1] == 0) return fail(ctx, HELIO_ERR_INVALID, "plan has no edge leaving the coordinator");
  {
    std::vector<int> fill(nv, 0);
    for (int i = 0; i < ne; ++i) {
      const int p = obeg[esrc[i]] + fill[esrc[i]]++;
      odst[p] = edst[i];
      oes[p] = pe[i].exec_start;
      oee[p] = pe[i].exec_end;
      oflow[p] = pe[i].flow;
    }
  }
  // Fast-path eligibility: node-consistent exec intervals, and no hop that
  // could ever be masked in the AC8 order.
  bool closed = true;
  // node-consistent exec ranges (every edge starts where its source vertex's
  // interval ends and ends where its target's does; coordinator edges only
  // leave vertices that end at L): the replay's tiling checks cannot fail
  bool consistent = true;
  for (int x = 0; x < nv; ++x)
    for (int p = obeg[x]; p < obeg[x + 1]; ++p) {
      const int d = odst[p];
      if (d == 0 ? vend[x] != L : (oes[p] != vend[x] || oee[p] != vend[d])) consistent = false;
    }
  int max_in = 0, max_out = 232;
  for (int64_t r = 0; r < R; ++r) {
    max_in = std::max(max_in, h_in[r]);
    max_out = std::max(max_out, h_out[r]);
  }
  const double tok_max = (double)max_in + (double)max_out * (1.0 + 1e-9) + 1.0;
  for (int x = 0; x < nv && closed; ++x)
    for (int p = obeg[x]; p < obeg[x + 1]; ++p) {
      const int d = odst[p];
      if (d == 0) continue;
      if (oee[p] != vend[d] || oes[p] != vend[x]) closed = false;
      const double charge = tok_max * ctx->kv_token_layer_bytes * (double)(oee[p] - oes[p]);
      if (!(charge * (1.0 + 1e-9) < 0.9 * kv_cap[d])) closed = false;
    }
  // weights / cycles: cycle length of x is sum(w) <= 32 * deg
  std::vector<int32_t> cyc_off(nv + 1, 0);
  for (int x = 0; x < nv; ++x) cyc_off[x + 1] = cyc_off[x] + 32 * (obeg[x + 1] - obeg[x]);

  cudaStream_t st = ctx->stream;
  int rc = HELIO_OK;
  int32_t *d_obeg = nullptr, *d_odst = nullptr, *d_oes = nullptr, *d_oee = nullptr, *d_node = nullptr,
          *d_cycoff = nullptr, *d_in = nullptr, *d_out = nullptr, *d_cur = nullptr, *d_nh = nullptr,
          *d_flag = nullptr, *d_rank = nullptr, *d_hn = nullptr, *d_hs = nullptr, *d_he = nullptr,
          *d_cyclen = nullptr;
  double *d_flow = nullptr, *d_kvcap = nullptr;
  long long *d_w = nullptr, *d_wmax = nullptr, *d_den = nullptr;
  int16_t *d_cyc = nullptr, *d_cov = nullptr;
  int* d_err = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0;
  const size_t HR = (size_t)R * std::max(max_hops, 1);
#define TRY(x)               \
  do {                       \
    if (!rc) rc = (x);       \
  } while (0)
  const bool want_se = h_hs != nullptr;
  const bool closed_path = closed && R > 0;
  if (closed_path) {
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)R, st);
  }
  Arena ar{ctx};
  for (int pass = 0; pass < 2 && !rc; ++pass) {
    ar.off = 0;
    ar.sizing = pass == 0;
    TRY(ar.take(&d_obeg, nv + 1));
    TRY(ar.take(&d_odst, ne));
    TRY(ar.take(&d_oes, ne));
    TRY(ar.take(&d_oee, ne));
    TRY(ar.take(&d_flow, ne));
    TRY(ar.take(&d_node, nv));
    TRY(ar.take(&d_kvcap, nv));
    TRY(ar.take(&d_w, ne));
    TRY(ar.take(&d_wmax, nv));
    TRY(ar.take(&d_cycoff, nv + 1));
    TRY(ar.take(&d_cyc, cyc_off[nv]));
    TRY(ar.take(&d_cyclen, nv));
    TRY(ar.take(&d_in, R));
    TRY(ar.take(&d_out, R));
    TRY(ar.take(&d_nh, R));
    TRY(ar.take(&d_hn, HR));
    TRY(ar.take(&d_hs, want_se ? HR : 1));
    TRY(ar.take(&d_he, want_se ? HR : 1));
    TRY(ar.take(&d_err, 1));
    TRY(ar.take(&d_den, 1));
    if (closed_path) {
      TRY(ar.take(&d_cur, R));
      TRY(ar.take(&d_cov, R));
      TRY(ar.take(&d_flag, R));
      TRY(ar.take(&d_rank, R));
      TRY(ar.take(reinterpret_cast<char**>(&d_tmp), tmp_bytes));
    }
    if (pass == 0 && ar.off > ctx->route_cap) {
      cudaFree(ctx->d_route);
      ctx->d_route = nullptr;
      ctx->route_cap = 0;
      if (cudaMalloc(&ctx->d_route, ar.off) != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "route arena alloc");
      else ctx->route_cap = ar.off;
    }
  }
  if (!rc) {
    auto H2D = [&](void* d, const void* h, size_t bytes) {
      if (bytes && !rc && cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = fail(ctx, HELIO_ERR_CUDA, "route H2D failed");
    };
    H2D(d_obeg, obeg.data(), 4 * (nv + 1));
    H2D(d_odst, odst.data(), 4 * ne);
    H2D(d_oes, oes.data(), 4 * ne);
    H2D(d_oee, oee.data(), 4 * ne);
    H2D(d_flow, oflow.data(), 8 * ne);
    H2D(d_node, node_of.data(), 4 * nv);
    H2D(d_kvcap, kv_cap.data(), 8 * nv);
    H2D(d_cycoff, cyc_off.data(), 4 * (nv + 1));
    H2D(d_in, h_in, 4 * R);
    H2D(d_out, h_out, 4 * R);
    if (!rc && (cudaMemsetAsync(d_err, 0, sizeof(int), st) != cudaSuccess ||
                cudaMemsetAsync(d_den, 0, sizeof(long long), st) != cudaSuccess))
      rc = fail(ctx, HELIO_ERR_CUDA, "route memset failed");
  }
  if (!rc) {
    route_setup<<<(nv + 63) / 64, 64, 0, st>>>(nv, d_obeg, d_flow, d_w, d_cycoff, d_cyc, d_wmax, d_cyclen);
    ctx->launches++;
    if (cudaGetLastError() != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "route_setup launch failed");
  }
  int64_t den = 0;
  if (!rc && closed && R > 0) {
    {
      const int grid = (int)std::min<int64_t>((R + 255) / 256, 8 * ctx->sm_count);
      route_init<<<grid, 256, 0, st>>>(R, d_cur, d_nh, d_cov);
      ctx->launches++;
      // vertices in end-layer order (coordinator first); sinks of routes
      // (end == L) never pick.
      std::vector<int> vorder;
      for (int x = 0; x < nv; ++x) vorder.push_back(x);
      std::stable_sort(vorder.begin(), vorder.end(), [&](int a, int b) { return vend[a] < vend[b]; });
      for (int x : vorder) {
        if (x != 0 && vend[x] >= L) continue;
        route_flag<<<grid, 256, 0, st>>>(R, x, d_cur, d_flag);
        cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_flag, d_rank, (int)R, st);
        route_apply<<<grid, 256, 0, st>>>(R, x, L, max_hops, d_obeg, d_odst, d_oes, d_oee, d_node,
                                           d_cycoff, d_cyclen, d_cyc, d_rank, d_cur, d_nh, d_cov, d_hn,
                                           want_se ? d_hs : nullptr, want_se ? d_he : nullptr,
                                           d_err);
        ctx->launches += 3;
      }
      if (cudaGetLastError() != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "route kernels failed");
    }
  } else if (!rc && R > 0) {
    {
      // slot records: 32 bytes per slot (int16 slot indices); every cycle
      // fits 32 slots per edge — when that bound does not fit shared memory,
      // read the actual cycle lengths back
      int64_t slots = cyc_off[nv];
      const size_t head = ((((size_t)4 * nv + 7) & ~size_t(7)) + 8 * (size_t)nv + 15) & ~size_t(15);
      if (head + (size_t)slots * sizeof(SlotRec) > 227 * 1024) {
        std::vector<int32_t> cl(nv);
        if (cudaMemcpyAsync(cl.data(), d_cyclen, 4 * nv, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
          rc = fail(ctx, HELIO_ERR_CUDA, "route: cycle lengths read-back failed");
        slots = 0;
        for (int x = 0; x < nv; ++x) slots += obeg[x + 1] > obeg[x] ? cl[x] : 0;
      }
      const size_t smem = head + (size_t)slots * sizeof(SlotRec) + 16;
      if (rc) {
      } else if (smem > 227 * 1024 || slots > 32767) {
        rc = fail(ctx, HELIO_ERR_TOO_LARGE, "plan too large for the masked routing kernel's shared memory");
      } else {
        auto kern = nv <= 32 ? (consistent ? route_masked_warp<true, false> : route_masked_warp<true, true>)
                             : (consistent ? route_masked_warp<false, false> : route_masked_warp<false, true>);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, 32, smem, st>>>(R, nv, L, max_hops, ctx->kv_token_layer_bytes, d_obeg, d_odst, d_oes, d_oee, d_node,
                                  d_kvcap, d_cyclen, d_cyc, d_in, d_out, d_nh, d_hn, want_se ? d_hs : nullptr,
                                  want_se ? d_he : nullptr, d_den, d_err);
      }
      if (cudaGetLastError() != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "route_masked_warp failed");
    }
  }
  int herr = 0;
  if (!rc && R > 0) {
    bool ok = cudaMemcpyAsync(h_nh, d_nh, 4 * R, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
              cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, st) == cudaSuccess;
    if (ok && max_hops > 0) ok = cudaMemcpyAsync(h_hn, d_hn, 4 * HR, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    if (ok && max_hops > 0 && want_se)
      ok = cudaMemcpyAsync(h_hs, d_hs, 4 * HR, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
           cudaMemcpyAsync(h_he, d_he, 4 * HR, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    long long dd = 0;
    if (ok && !closed) ok = cudaMemcpyAsync(&dd, d_den, sizeof(long long), cudaMemcpyDeviceToHost, st) == cudaSuccess;
    ok = ok && cudaStreamSynchronize(st) == cudaSuccess;
    if (!ok) rc = fail(ctx, HELIO_ERR_CUDA, std::string("route: ") + cudaGetErrorString(cudaGetLastError()));
    if (!rc && closed)
      for (int64_t r = 0; r < R; ++r) den += h_nh[r] < 0;
    else
      den = dd;
  }
  if (!rc && herr) rc = fail(ctx, HELIO_ERR_INVALID, "plan edges do not tile the layer range");
  if (!rc && h_deferred) *h_deferred = den;
#undef TRY
  return rc;
}

// ---------------------------------------------------------------------------
// Stand-alone iwrr_weights / IwrrPicker cycles / IwrrPicker::next on the
// device.  Buffers come from the context's host-entry arena (no per-call
// cudaMalloc/cudaFree).
namespace {

// iwrr_weights (scheduler.cpp:46-56) of list `l` = [off[l], off[l+1]).
__device__ void list_weights(const double* __restrict__ flow, long long* __restrict__ w, int b, int e) {
  long long wmax = 0;
  for (int i = b; i < e; ++i) {
    long long v = llround(1000.0 * flow[i]);
    w[i] = v > 1 ? v : 1;
    wmax = w[i] > wmax ? w[i] : wmax;
  }
  if (wmax > 32)
    for (int i = b; i < e; ++i) {
      long long v = llround(w[i] * 32.0 / wmax);
      w[i] = v > 1 ? v : 1;
    }
}

__global__ void iwrr_weights_kernel(int nlists, const int32_t* __restrict__ off, const double* __restrict__ flow,
                                    long long* __restrict__ w) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < nlists) list_weights(flow, w, off[l], off[l + 1]);
}

// One warp per candidate list: (flows -> weights, when flow != nullptr), then
// the IWRR cycle — the slots (round r, index i) with w_i >= r in (r, i) order,
// i.e. the order IwrrPicker::next (scheduler.cpp:28-44) visits them when
// every candidate is eligible.  cyc[cyc_off[l] + k] = candidate index of the
// k-th slot; cyc_len[l] = sum of the weights.
__global__ void iwrr_cycles_kernel(int nlists, const int32_t* __restrict__ off, const double* __restrict__ flow,
                                   long long* __restrict__ w, const int64_t* __restrict__ cyc_off,
                                   int32_t* __restrict__ cyc, int64_t* __restrict__ cyc_len) {
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (l >= nlists) return;
  const int b = off[l], e = off[l + 1];
  if (flow != nullptr && lane == 0) list_weights(flow, w, b, e);
  __syncwarp();
  long long wm = 1;  // IwrrPicker ctor: wmax_ starts at 1
  for (int i = b + lane; i < e; i += 32) wm = w[i] > wm ? w[i] : wm;
  for (int d = 16; d; d >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, wm, d);
    wm = o > wm ? o : wm;
  }
  int64_t p = cyc_off[l];
  for (long long r = 1; r <= wm; ++r)
    for (int base = b; base < e; base += 32) {
      const int i = base + lane;
      const bool take = i < e && w[i] >= r;
      const unsigned m = __ballot_sync(0xffffffffu, take);
      if (take) cyc[p + __popc(m & ((1u << lane) - 1u))] = i - b;
      p += __popc(m);
    }
  if (lane == 0) cyc_len[l] = p - cyc_off[l];
}

__global__ void iwrr_picks_kernel(int n, const long long* __restrict__ w, long long* state, int calls,
                                  const unsigned long long* __restrict__ masks, int* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  long long round = state[0], idx = state[1];
  long long wmax = 1;
  for (int i = 0; i < n; ++i) wmax = w[i] > wmax ? w[i] : wmax;
  const int words = (n + 63) / 64;
  for (int k = 0; k < calls; ++k) {
    int pick = -1;
    if (n > 0) {
      const long long positions = wmax * (long long)n;
      for (long long it = 0; it < positions; ++it) {
        if (idx == n) {
          idx = 0;
          round = round == wmax ? 1 : round + 1;
        }
        const int i = (int)idx++;
        if (w[i] >= round && ((masks[(size_t)k * words + (i >> 6)] >> (i & 63)) & 1ull)) {
          pick = i;
          break;
        }
      }
    }
    out[k] = pick;
  }
  state[0] = round;
  state[1] = idx;
}

}  // namespace

extern "C" int helio_gpu_iwrr_weights(helio_gpu_ctx* ctx, const double* h_flows, int32_t n, int64_t* h_w) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (n < 0 || (n > 0 && (!h_flows || !h_w))) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (n == 0) return HELIO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  auto carve = [&](Carve& c, int32_t*& off, double*& f, long long*& w) {
    off = c.take<int32_t>(2);
    f = c.take<double>(n);
    w = c.take<long long>(n);
  };
  int32_t* d_off;
  double* d_f;
  long long* d_w;
  Carve measure, c;
  carve(measure, d_off, d_f, d_w);
  int rc = host_arena(ctx, measure.off, &c.base);
  if (rc) return rc;
  carve(c, d_off, d_f, d_w);
  const int32_t off[2] = {0, n};
  CK(cudaMemcpyAsync(d_off, off, sizeof(off), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_f, h_flows, 8 * n, cudaMemcpyHostToDevice, st));
  iwrr_weights_kernel<<<1, 32, 0, st>>>(1, d_off, d_f, d_w);
  ctx->launches++;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h_w, d_w, 8 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HELIO_OK;
}

extern "C" int helio_gpu_iwrr_cycles(helio_gpu_ctx* ctx, int32_t nlists, const int32_t* h_off,
                                     const double* h_flows, int64_t* h_weights, const int64_t* h_cyc_off,
                                     int32_t* h_cycles, int64_t* h_cyc_len) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (nlists < 0 || (nlists > 0 && (!h_off || !h_weights || !h_cyc_off || !h_cyc_len)))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (nlists == 0) return HELIO_OK;
  const int32_t n = h_off[nlists];
  if (h_off[0] != 0 || n < 0) return fail(ctx, HELIO_ERR_INVALID, "list offsets must start at 0");
  for (int l = 0; l < nlists; ++l)
    if (h_off[l + 1] < h_off[l]) return fail(ctx, HELIO_ERR_INVALID, "list offsets must be non-decreasing");
  const int64_t total = h_cyc_off[nlists];
  if (h_cyc_off[0] != 0 || total < 0 || (total > 0 && !h_cycles))
    return fail(ctx, HELIO_ERR_INVALID, "bad cycle offsets");
  if (!h_flows)  // caller weights: every list's cycle (sum of its weights) must fit its slot range
    for (int l = 0; l < nlists; ++l) {
      long long sum = 0;
      for (int i = h_off[l]; i < h_off[l + 1]; ++i) sum += h_weights[i] > 0 ? h_weights[i] : 0;
      if (sum > h_cyc_off[l + 1] - h_cyc_off[l]) return fail(ctx, HELIO_ERR_INVALID, "cycle range too small");
    }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  auto carve = [&](Carve& c, int32_t*& off, double*& f, long long*& w, int64_t*& coff, int32_t*& cyc,
                   int64_t*& clen) {
    off = c.take<int32_t>(nlists + 1);
    f = c.take<double>(h_flows ? n : 1);
    w = c.take<long long>(n);
    coff = c.take<int64_t>(nlists + 1);
    cyc = c.take<int32_t>(total);
    clen = c.take<int64_t>(nlists);
  };
  int32_t *d_off, *d_cyc;
  double* d_f;
  long long* d_w;
  int64_t *d_coff, *d_clen;
  Carve measure, c;
  carve(measure, d_off, d_f, d_w, d_coff, d_cyc, d_clen);
  int rc = host_arena(ctx, measure.off, &c.base);
  if (rc) return rc;
  carve(c, d_off, d_f, d_w, d_coff, d_cyc, d_clen);
  CK(cudaMemcpyAsync(d_off, h_off, 4 * (nlists + 1), cudaMemcpyHostToDevice, st));
  if (h_flows)
    CK(cudaMemcpyAsync(d_f, h_flows, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
  else if (n > 0)
    CK(cudaMemcpyAsync(d_w, h_weights, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_coff, h_cyc_off, 8 * (nlists + 1), cudaMemcpyHostToDevice, st));
  const int warps = 4;
  iwrr_cycles_kernel<<<(nlists + warps - 1) / warps, 32 * warps, 0, st>>>(nlists, d_off, h_flows ? d_f : nullptr,
                                                                          d_w, d_coff, d_cyc, d_clen);
  ctx->launches++;
  CK(cudaGetLastError());
  if (h_flows && n > 0) CK(cudaMemcpyAsync(h_weights, d_w, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
  if (total > 0) CK(cudaMemcpyAsync(h_cycles, d_cyc, 4 * (size_t)total, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_cyc_len, d_clen, 8 * (size_t)nlists, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HELIO_OK;
}

extern "C" int helio_gpu_iwrr_picks(helio_gpu_ctx* ctx, const int64_t* h_w, int32_t n, int64_t* h_round,
                                    int64_t* h_idx, int32_t calls, const uint64_t* h_masks, int32_t* h_out) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (n < 0 || calls < 0 || !h_round || !h_idx || (n > 0 && !h_w) || (calls > 0 && (!h_out || (n > 0 && !h_masks))))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (calls == 0) return HELIO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int words = (n + 63) / 64;
  auto carve = [&](Carve& c, long long*& w, long long*& state, unsigned long long*& m, int*& out) {
    w = c.take<long long>(n);
    state = c.take<long long>(2);
    m = c.take<unsigned long long>((size_t)calls * words);
    out = c.take<int>(calls);
  };
  long long *d_w, *d_state;
  unsigned long long* d_m;
  int* d_out;
  Carve measure, c;
  carve(measure, d_w, d_state, d_m, d_out);
  int rc = host_arena(ctx, measure.off, &c.base);
  if (rc) return rc;
  carve(c, d_w, d_state, d_m, d_out);
  long long stt[2] = {(long long)*h_round, (long long)*h_idx};
  if (n > 0) CK(cudaMemcpyAsync(d_w, h_w, 8 * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_state, stt, 16, cudaMemcpyHostToDevice, st));
  if (n > 0) CK(cudaMemcpyAsync(d_m, h_masks, 8 * (size_t)calls * words, cudaMemcpyHostToDevice, st));
  iwrr_picks_kernel<<<1, 32, 0, st>>>(n, d_w, d_state, calls, d_m, d_out);
  ctx->launches++;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h_out, d_out, 4 * calls, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(stt, d_state, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *h_round = stt[0];
  *h_idx = stt[1];
  return HELIO_OK;
}

extern "C" int helio_gpu_check_division(helio_gpu_ctx* ctx, int64_t count, uint64_t seed, int64_t* mismatches) {
  if (!ctx || !mismatches || count < 0) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
  CK(cudaSetDevice(ctx->device));
  char* base = nullptr;
  int rc = host_arena(ctx, 64, &base);
  if (rc) return rc;
  unsigned long long* d = reinterpret_cast<unsigned long long*>(base);
  CK(api_begin(ctx, ctx->stream));
  CK(cudaMemsetAsync(d, 0, 8, ctx->stream));
  check_division_kernel<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(count, seed, d);
  CK(cudaGetLastError());
  CK(api_end(ctx, ctx->stream));
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *mismatches = (int64_t)h;
  ctx->launches++;
  return HELIO_OK;
}
