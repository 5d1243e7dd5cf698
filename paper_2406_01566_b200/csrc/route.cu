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
// for node-consistent plans the chunked parallel replay (route_masked_spec),
// otherwise one warp walking the device-built cycles with the state in shared
// memory (route_masked_warp).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
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

// ---------------------------------------------------------------------------
// The masked replay in parallel (plans with node-consistent exec ranges).
//
// Requests are taken in chunks of kSpecChunk.  Inside a chunk the serial
// coupling is (1) each vertex's picker position and (2) the running output
// mean, which depends on which requests get deferred.  A pass routes the
// chunk for a GUESSED set of deferrals:
//  * warp 0 runs the division chain from the guess and publishes every
//    request's tokens, 32 requests (a "group") at a time;
//  * every other warp owns plan vertices and walks them group by group: a
//    vertex may take group g once the chain and every vertex with an edge into
//    it have finished g (a plan edge always ends at a later layer than it
//    starts, so this is a wavefront over the plan DAG).  Inside a group the
//    arrivals pick in request order.
// If the deferrals found equal the guess, every token was right and the chunk
// is the reference's.  Otherwise let f be the first request whose guess was
// wrong: everything before f was exact (tokens and positions), so the next
// pass guesses the deferrals found and restarts from f's group with the
// positions and chain state saved at that group's start; f moves forward every
// pass, and after kSpecPasses the chunk is replayed serially instead.
//
// The first pass of a chunk is approximate: every token comes from the
// chunk-start mean (the mean drifts by a fraction of a token over a chunk), so
// the vertex warps run without waiting for the chain, and warp 0 runs the
// exact chain right behind them on the deferrals they found (it waits on the
// DAG's leaves).  Verification is then parallel: a request whose exact tokens
// give the same class at every vertex it visited picks the same slots (by
// induction over the requests), so the pass stands up to the first request
// where a class differs, and exact passes take over from that request's group.
// On bench.py's plan 97% of chunks are done after the approximate pass.
//
// Picks.  Eligibility of an edge, RN(tk * len) <= thr, is monotone in tk, so
// each edge has an exact cut-off te (the largest double passing; bisection
// over the bit patterns) and the eligible edges of a vertex are always the c
// edges of largest te — its "class" c, counted per arrival in parallel.  A
// class-deg arrival takes the current slot; a masked one (0 < c < deg) takes
// nxt[c][p], a per-vertex table of the first slot at or after p whose edge is
// among the top c (built at launch); class 0 is deferred with the position
// unchanged.  So a pick is one shared-memory load whatever the mask.  The
// coordinator, which every request passes, also gets a two-step table
// (two arrivals per load) and, in the approximate pass, its classes are
// computed for the whole chunk before the pass.
constexpr int kSpecChunk = 2048, kSpecGroups = kSpecChunk / 32, kSpecThreads = 1024, kSpecPasses = 8;

// Frontier flags live in shared memory: relaxed CTA-scope loads/stores on
// the shared window (plain LDS/STS) ordered by acq_rel fences — the fence
// pattern of the PTX memory model, without the generic-address strong loads
// cuda::atomic_ref compiles to.
__device__ __forceinline__ int spec_load(const int* p) {
  int v;
  asm volatile("ld.relaxed.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void spec_fence() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }
// Spin until *p >= need.  The wavefront cannot deadlock (every wait is on a
// vertex earlier in end-layer order, or on the chain); the bound turns a bug
// into a launch error instead of a hung device.
#ifndef SPEC_SLEEP
#define SPEC_SLEEP 32
#endif
// (the caller fences once after its waits)
template <bool SLEEP = true>
__device__ __forceinline__ void spec_wait(const int* p, int need) {
  // vertex warps back off between polls so waiting warps leave the issue
  // slots to the working ones; the chain polls tightly
  for (unsigned n = 0; spec_load(p) < need; ++n) {
    if (SLEEP && SPEC_SLEEP) __nanosleep(SPEC_SLEEP);
    if (n > (1u << 30)) __trap();
  }
}
__device__ __forceinline__ void spec_release(int* p, int v) {
  spec_fence();
  asm volatile("st.relaxed.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

#ifdef SPEC_PROFILE
__device__ long long spec_prof[8192];
#define SPEC_PROF(idx) \
  do {                 \
    if (c0 == 3 * C) spec_prof[idx] = clock64(); \
  } while (0)
#else
#define SPEC_PROF(idx) \
  do {                 \
  } while (0)
#endif

// One pick on a cycle [base, base + W) from relative position p (serial
// fallback): the first eligible slot in one full cycle; returns its absolute
// slot (p advanced past it) or -1 (p unchanged).
__device__ __forceinline__ int spec_pick(const SlotRec* rec, int base, int W, int& p, double tk) {
  for (int k = 0; k < W; ++k) {
    int q = p + k;
    q -= q >= W ? W : 0;
    const SlotRec& r = rec[base + q];
    if (tk * r.len <= r.thr) {
      p = q + 1 == W ? 0 : q + 1;
      return base + q;
    }
  }
  return -1;
}

// meta = [vorder: nvo vertex ids, end-layer order, the coordinator first]
//        [pred_beg: nvo + 1] [pred: order indices of the vertices with an edge into each]
//        [nleaves] [leaves: order indices of the vertices no routed vertex follows]
__global__ void __launch_bounds__(kSpecThreads, 1) route_masked_spec(
    int64_t R, int nv, int L, int max_hops, double kvb, const int32_t* __restrict__ obeg,
    const int32_t* __restrict__ odst, const int32_t* __restrict__ oes, const int32_t* __restrict__ oee,
    const int32_t* __restrict__ node_of, const double* __restrict__ kv_cap, const int32_t* __restrict__ cyc_len,
    const int16_t* __restrict__ cyc, int nvo, const int32_t* __restrict__ meta, int nxt_cap, int pair_cap, int hmax,
    const int32_t* __restrict__ in_len, const int32_t* __restrict__ out_len, int32_t* nh, int32_t* hop_node,
    int32_t* hop_s, int32_t* hop_e, long long* deferred, int* passes_out) {
  extern __shared__ __align__(16) char sm[];
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, NW = T >> 5;
  constexpr int C = kSpecChunk, G1 = kSpecGroups + 1;
  const unsigned FULL = 0xffffffffu;
  const int32_t* vorder = meta;
  const int32_t* pred_beg = meta + nvo;
  const int32_t* pred = meta + 2 * nvo + 1;
  const int32_t* leaves = pred + pred_beg[nvo] + 1;
  const int nleaves = leaves[-1];
  size_t o = 0;
#define take(bytes) (sm + ((o += ((size_t)(bytes) + 15) & ~size_t(15)) - (((size_t)(bytes) + 15) & ~size_t(15))))
  double* tk = reinterpret_cast<double*>(take(8 * C));
  double* tk_exact = reinterpret_cast<double*>(take(8 * C));
  uint8_t* route_v = reinterpret_cast<uint8_t*>(take((size_t)C * hmax));  // approximate pass: vertices visited
  double* ytab = reinterpret_cast<double*>(take(8 * C));
  int32_t* in_s = reinterpret_cast<int32_t*>(take(4 * C));
  int32_t* out_s = reinterpret_cast<int32_t*>(take(4 * C));
  int16_t* cur = reinterpret_cast<int16_t*>(take(2 * C));  // vertex the request waits at; -1 = done
  int16_t* hcnt = reinterpret_cast<int16_t*>(take(2 * C));
  uint8_t* dguess = reinterpret_cast<uint8_t*>(take(C));
  uint8_t* dfound = reinterpret_cast<uint8_t*>(take(C));
  uint8_t* cls0 = reinterpret_cast<uint8_t*>(take(C));  // approximate pass: classes at the coordinator
  double* a_grp = reinterpret_cast<double*>(take(8 * G1));    // chain state at each group's start
  int32_t* adm_grp = reinterpret_cast<int32_t*>(take(4 * G1));
  int16_t* pos_g = reinterpret_cast<int16_t*>(take(2 * (size_t)nvo * G1));  // positions at group starts
  int32_t* front = reinterpret_cast<int32_t*>(take(4 * (nvo + 1)));         // groups done; [nvo] = chain
  int32_t* pcur = reinterpret_cast<int32_t*>(take(4 * nvo));
  int32_t* pos = reinterpret_cast<int32_t*>(take(4 * nv));  // committed relative positions
  int2* vgeo = reinterpret_cast<int2*>(take(8 * nv));
  const int ne = obeg[nv];
  const int deg0 = obeg[1] - obeg[0];  // vorder[0] is the coordinator (vertex 0, edges from 0)
  double* tes = reinterpret_cast<double*>(take(8 * (size_t)ne));      // cut-offs per vertex, descending
  double* te_raw = reinterpret_cast<double*>(take(8 * (size_t)ne));   // cut-off of each edge
  int16_t* erank = reinterpret_cast<int16_t*>(take(2 * (size_t)ne));  // edge's rank in its vertex
  int32_t* noff = reinterpret_cast<int32_t*>(take(4 * (nv + 1)));     // next-slot tables per vertex
  int16_t* nxt = reinterpret_cast<int16_t*>(take(2 * (size_t)nxt_cap));
  int32_t* wcls = reinterpret_cast<int32_t*>(take(4 * 32 * NW));  // per warp: class (* W) of each arrival
  int16_t* nxt2 = reinterpret_cast<int16_t*>(take(2 * (size_t)pair_cap));  // coordinator: two-step table
  double2* chain_ops = reinterpret_cast<double2*>(take(16 * 32));
  int32_t* scal = reinterpret_cast<int32_t*>(take(16));
  double* scal_d = reinterpret_cast<double*>(take(16));
  SlotRec* rec = reinterpret_cast<SlotRec*>(take(0));
#undef take
  if (tid == 0) {
    int toff = 0;
    for (int x = 0, base = 0; x < nv; ++x) {
      const int deg = obeg[x + 1] - obeg[x];
      const int W = deg > 0 ? cyc_len[x] : 0;
      vgeo[x] = make_int2(base, W);
      pos[x] = 0;
      base += W;
      noff[x] = toff;
      toff += (deg + 1) * W;
    }
    noff[nv] = toff;
    scal[2] = 0;  // deferrals of the chunks resolved in parallel
  }
  // each edge's cut-off te: the largest double t with RN(t * len) <= thr
  // (bisection over the bit patterns of the non-negative doubles)
  for (int e = tid; e < ne; e += T) {
    const int d = odst[e];
    const double thr = d == 0 ? 1.0e308 : 0.9 * kv_cap[d], len = (double)(oee[e] - oes[e]);
    unsigned long long lo = 0, hi = 0x7ff0000000000000ull;  // P(+0) holds (thr >= 0), P(+inf) fails
    while (hi - lo > 1) {
      const unsigned long long mid = lo + (hi - lo) / 2;
      if (__longlong_as_double((long long)mid) * len <= thr) lo = mid;
      else hi = mid;
    }
    te_raw[e] = __longlong_as_double((long long)lo);
  }
  __syncthreads();
  // ranks within each vertex by te descending (ties by edge order)
  for (int e = tid; e < ne; e += T) {
    int x = 0;
    while (obeg[x + 1] <= e) ++x;
    int r = 0;
    for (int f = obeg[x]; f < obeg[x + 1]; ++f) r += te_raw[f] > te_raw[e] || (te_raw[f] == te_raw[e] && f < e);
    erank[e] = (int16_t)r;
    tes[obeg[x] + r] = te_raw[e];
  }
  __syncthreads();
  if (noff[nv] > nxt_cap) __trap();  // the host sizes nxt_cap from 32 * deg >= W
  for (int x = wid; x < nv; x += NW) {
    const int2 geo = vgeo[x];
    const int b = obeg[x], deg = obeg[x + 1] - b, W = geo.y;
    for (int k = lane; k < W; k += 32) {
      const int e = b + cyc[32 * b + k];
      const int d = odst[e];
      SlotRec r;
      r.thr = d == 0 ? 1.0e308 : 0.9 * kv_cap[d];
      r.len = (double)(oee[e] - oes[e]);
      r.next = 0;
      r.dst = d;
      r.ee = oee[e];
      r.es_node = (oes[e] & 0xffff) | (node_of[d] << 16);
      rec[geo.x + k] = r;
    }
    // position table of class c (the c edges of largest te eligible), c = 0..deg:
    // nxt[c][p] = the position after the first slot at or after p (cyclically)
    // whose edge has rank < c; class 0 picks nothing (position unchanged)
    for (int c = lane; c <= deg; c += 32) {
      int16_t* t = nxt + noff[x] + c * W;
      int last = -1;
      for (int q2 = 2 * W - 1; q2 >= 0; --q2) {
        const int q = q2 < W ? q2 : q2 - W;
        if (erank[b + cyc[32 * b + q]] < c) last = q;
        if (q2 < W) t[q] = (int16_t)(c == 0 ? q : (last + 1 == W ? 0 : last + 1));
      }
    }
  }
  __syncthreads();
  // the coordinator (every request's first pick) also gets a two-step table:
  // nxt2[c1][c2][p] = nxt[c2][nxt[c1][p]], one load per two arrivals
  if (pair_cap > 0) {
    const int W0 = vgeo[0].y, D1 = deg0 + 1;
    if (D1 * D1 * W0 > pair_cap) __trap();  // the host sizes pair_cap
    const int16_t* t0 = nxt + noff[0];
    for (int idx = tid; idx < D1 * D1 * W0; idx += T) {
      const int p0 = idx % W0, cc = idx / W0, c2 = cc % D1, c1 = cc / D1;
      nxt2[idx] = t0[c2 * W0 + t0[c1 * W0 + p0]];
    }
  }
  __syncthreads();
  double avg = 232.0, samples = 1.0;  // thread 0: the committed running mean
  long long den = 0;
  int passes_total = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < R; c0 += C) {
    const int cn = R - c0 < C ? (int)(R - c0) : C;
    const int G = (cn + 31) >> 5;
    if (tid == 0) SPEC_PROF(0);
    for (int i = tid; i < cn; i += T) {
      in_s[i] = in_len[c0 + i];
      out_s[i] = out_len[c0 + i];
      dguess[i] = 0;
    }
    if (tid == 0) {
      a_grp[0] = avg;
      adm_grp[0] = 0;
      scal_d[0] = samples;
      scal[0] = 0;  // g0
    }
    for (int k = tid; k < nvo; k += T) pos_g[k * G1] = (int16_t)pos[vorder[k]];
    __syncthreads();
    const double samples0 = scal_d[0];
    for (int i = tid; i < cn; i += T) ytab[i] = __drcp_rn(samples0 + 1.0 + i);
    bool converged = false;
    __syncthreads();
    if (tid == 0) SPEC_PROF(1);
    for (int pass = 0; pass < kSpecPasses && !converged; ++pass) {
      const int g0 = scal[0];
      const bool approx = hmax > 0 && pass == 0;
      for (int i = (g0 << 5) + tid; i < cn; i += T) {
        cur[i] = 0;
        hcnt[i] = 0;
        dfound[i] = 0;
        if (approx) {  // every token from the chunk-start mean; the coordinator's classes up front
          const double t = ((double)in_s[i] + a_grp[0]) * kvb;
          tk[i] = t;
          int c = 0;
          for (int j = 0; j < deg0; ++j) c += t <= tes[j];
          cls0[i] = (uint8_t)c;
        }
      }
      for (int k = tid; k < nvo; k += T) {
        front[k] = g0;
        pcur[k] = pos_g[k * G1 + g0];
      }
      if (tid == 0) {
        front[nvo] = g0;
        scal[1] = 0x7fffffff;  // first mismatch
      }
      __syncthreads();
      if (wid == 0) {
        const unsigned lt = (1u << lane) - 1u;
        double a = a_grp[g0];
        int adm = adm_grp[g0];
        // the division chain over the admissions, 32 requests at a time.  An
        // exact pass takes the guessed deferrals and publishes its tokens for
        // the vertex warps; the approximate pass runs it right behind the
        // routing on the deferrals found (every vertex done with the group),
        // into tk_exact for the verification
        const uint8_t* dsrc = approx ? dfound : dguess;
        double* tout = approx ? tk_exact : tk;
        int done_upto = 0;
        for (int g = g0; g < G; ++g) {
          if (approx && done_upto <= g) {  // every vertex done with the group: every leaf is
            int lo = 0x7fffffff;
            for (int j = 0; j < nleaves; ++j) {
              spec_wait<false>(&front[leaves[j]], g + 1);
              lo = min(lo, spec_load(&front[leaves[j]]));
            }
            spec_fence();
            done_upto = lo;  // the leaves are done through group lo - 1: no polling until then
          }
          const int i0 = g << 5, i = i0 + lane;
          const bool valid = i < cn;
          const bool ad = valid && !dsrc[i];
          const unsigned am = __ballot_sync(FULL, ad);
          const double my_in = valid ? (double)in_s[i] : 0.0;
          // the group's admissions packed in order: (out, 1/n) per step,
          // so the loop below is only the 5 dependent FP64 ops per step
          const int rk = __popc(am & lt), m = __popc(am);
          if (ad) chain_ops[rk] = make_double2((double)out_s[i], ytab[adm + rk]);
          __syncwarp();
          double my_a = a;  // the mean before request i: after its rk admitted predecessors
#pragma unroll 4
          for (int k2 = 0; k2 < m; ++k2) {
            const double2 oy = chain_ops[k2];
            a += div_by_count(oy.x - a, samples0 + 1.0 + (adm + k2), oy.y);
            if (k2 + 1 == rk) my_a = a;
          }
          __syncwarp();
          if (valid) tout[i] = (my_in + my_a) * kvb;
          adm += m;
          __syncwarp();
          if (lane == 0) {
            if (pass < 2) SPEC_PROF(64 + pass * 2048 + 31 * 64 + g);
            a_grp[g + 1] = a;
            adm_grp[g + 1] = adm;
            if (!approx) spec_release(&front[nvo], g + 1);
          }
        }
      } else {
        // vertex warps: each owns vorder[k] for k = wid - 1 (mod NW - 1) and
        // walks its groups in order (deadlock-free: every wait is on a vertex
        // earlier in end-layer order, or on the chain)
        for (int k = wid - 1; k < nvo; k += NW - 1) {
          const int v = vorder[k];
          const int2 geo = vgeo[v];
          const int base = geo.x, W = geo.y;
          const int eb = obeg[v], deg = obeg[v + 1] - eb;
          const int pb = pred_beg[k], pe = pred_beg[k + 1];
          const int16_t* tb = nxt + noff[v];
          const unsigned lt = (1u << lane) - 1u;
          int32_t* wc = wcls + (wid << 5);
          int p = pcur[k];
          for (int g = g0; g < G; ++g) {
            const int need = g + 1;
            if (!approx) spec_wait(&front[nvo], need);  // (the approximate tokens are set before the pass)
            for (int j = pb; j < pe; ++j) spec_wait(&front[pred[j]], need);
            spec_fence();
            if (lane == 0) pos_g[k * G1 + g] = (int16_t)p;
            const int i = (g << 5) + lane;
            int hop_h = -1, hop_es_node = 0, hop_ee = 0;
            const bool arr = i < cn && cur[i] == v;
            const unsigned am = __ballot_sync(FULL, arr);
            if (am) {
              int slot = -1;
              if (approx && arr) {  // the route, for the verification
                const int h = hcnt[i];
                if (h < hmax) route_v[i * hmax + h] = (uint8_t)v;
              }
              if (W > 0) {
                // class: how many of the vertex's edges are eligible (a
                // prefix of the te-descending order)
                int c = 0;
                if (arr) {
                  if (approx && k == 0) {
                    c = cls0[i];
                  } else {
                    const double t = tk[i];
#pragma unroll 4
                    for (int j = 0; j < deg; ++j) c += t <= tes[eb + j];
                  }
                }
                const unsigned fm = __ballot_sync(FULL, arr && c == deg);
                if (fm == am) {  // every arrival takes the next slot
                  const int r = p + __popc(am & lt);
                  slot = r < W ? r : r % W;
                  const int n = p + __popc(am);
                  p = n < W ? n : n % W;
                } else {
                  // the picks in request order: one table load per arrival on
                  // the serial path (p -> nxt[c][p]); the whole warp walks it
                  // in lockstep, the class offsets come from shared memory
                  const int rank = __popc(am & lt), m = __popc(am);
                  if (k == 0 && pair_cap > 0) {
                    // the coordinator: two arrivals per load on the serial path;
                    // each lane then recovers its own pick from the position
                    // before it (or before the arrival ahead of it)
                    if (arr) wc[rank] = c;
                    __syncwarp();
                    const int D1 = deg + 1;
                    int my_pb = 0;
                    int k2 = 0;
#pragma unroll 4
                    for (; k2 + 1 < m; k2 += 2) {
                      const int o2 = (wc[k2] * D1 + wc[k2 + 1]) * W;
                      if (k2 == rank) my_pb = p;
                      if (k2 + 1 == rank) my_pb = -1 - p;
                      p = nxt2[o2 + p];
                    }
                    if (k2 < m) {
                      if (k2 == rank) my_pb = p;
                      p = tb[wc[k2] * W + p];
                    }
                    __syncwarp();
                    if (arr) {
                      const int pb = my_pb >= 0 ? my_pb : tb[wc[rank - 1] * W + (-1 - my_pb)];
                      const int pa = tb[c * W + pb];
                      slot = c == 0 ? -1 : (pa == 0 ? W - 1 : pa - 1);
                    }
                  } else {
                    if (arr) wc[rank] = c * W;
                    __syncwarp();
                    int my_p = 0;
#pragma unroll 4
                    for (int k2 = 0; k2 < m; ++k2) {
                      p = tb[wc[k2] + p];
                      if (k2 == rank) my_p = p;
                    }
                    __syncwarp();
                    if (arr) slot = c == 0 ? -1 : (my_p == 0 ? W - 1 : my_p - 1);
                  }
                }
              }
              if (arr) {
                if (slot < 0) {
                  dfound[i] = 1;
                  cur[i] = -1;
                } else {
                  const SlotRec& rc = rec[base + slot];
                  hop_h = hcnt[i];
                  hop_es_node = rc.es_node;
                  hop_ee = rc.ee;
                  hcnt[i] = (int16_t)(hcnt[i] + 1);
                  cur[i] = (int16_t)(rc.ee >= L ? -1 : rc.dst);
                }
              }
            }
            if (lane == 0 && pass < 2 && k < 31) SPEC_PROF(64 + pass * 2048 + k * 64 + g);
            __syncwarp();
            if (lane == 0) spec_release(&front[k], need);
            // the hops go to HBM after the release (no consumer reads them)
            if (hop_h >= 0 && hop_h < max_hops) {
              const int64_t at = (c0 + i) * max_hops + hop_h;
              hop_node[at] = hop_es_node >> 16;
              if (hop_s) {
                hop_s[at] = hop_es_node & 0xffff;
                hop_e[at] = hop_ee;
              }
            }
          }
          if (lane == 0) pcur[k] = p;
        }
      }
      __syncthreads();
      if (tid == 0 && pass < 4) SPEC_PROF(2 + 2 * pass);
      if (!approx)
        for (int i = (g0 << 5) + tid; i < cn; i += T)
          if (dfound[i] != dguess[i]) atomicMin(&scal[1], i);
      __syncthreads();
      if (tid == 0 && pass < 4) SPEC_PROF(3 + 2 * pass);
      if (approx) {
        // verification: the routing with the chunk-start mean is the exact
        // one up to the first request whose exact tokens put it in another
        // class at a vertex it visited (by induction over the requests: the
        // same classes at the same positions pick the same slots)
        for (int i = tid; i < cn; i += T) {
          const int nvis = hcnt[i] + dfound[i];
          bool bad = nvis > hmax;
          const double t0 = tk[i], t1 = tk_exact[i];
          for (int h = 0; h < nvis && !bad; ++h) {
            const int v = route_v[i * hmax + h], eb = obeg[v], deg = obeg[v + 1] - eb;
            int c0 = 0, c1 = 0;
            for (int j = 0; j < deg; ++j) {
              c0 += t0 <= tes[eb + j];
              c1 += t1 <= tes[eb + j];
            }
            bad = c0 != c1;
          }
          if (bad) atomicMin(&scal[1], i);
        }
        __syncthreads();
      }
      const int f = scal[1];
      if (approx && f != 0x7fffffff) {  // exact passes from f's group, guessing the deferrals found
        for (int i = tid; i < cn; i += T) dguess[i] = dfound[i];
        if (tid == 0) scal[0] = f >> 5;
      } else if (f == 0x7fffffff) {
        converged = true;
      } else {
        for (int i = f + tid; i < cn; i += T) dguess[i] = dfound[i];
        if (tid == 0) scal[0] = f >> 5;
      }
      ++passes_total;
      __syncthreads();
    }
    if (converged) {
      int local = 0;
      for (int i = tid; i < cn; i += T) {
        nh[c0 + i] = dfound[i] ? -1 : hcnt[i];
        local += dfound[i];
      }
      for (int k = tid; k < nvo; k += T) pos[vorder[k]] = pcur[k];
      for (int d = 16; d; d >>= 1) local += __shfl_xor_sync(FULL, local, d);
      if (lane == 0) atomicAdd(&scal[2], local);
      if (tid == 0) {
        avg = a_grp[G];
        samples = samples0 + adm_grp[G];
      }
    } else if (tid == 0) {
      // serial replay of the chunk from the committed state
      for (int i = 0; i < cn; ++i) {
        const double tki = ((double)in_s[i] + avg) * kvb;
        int v = 0, covered = 0, h = 0;
        bool ok = true;
        while (covered < L) {
          const int2 geo = vgeo[v];
          if (geo.y == 0) {
            ok = false;
            break;
          }
          int p = pos[v];
          const int s2 = spec_pick(rec, geo.x, geo.y, p, tki);
          if (s2 < 0) {
            ok = false;
            break;
          }
          pos[v] = p;
          const SlotRec& r = rec[s2];
          if (max_hops > 0 && h < max_hops) {
            const int64_t at = (c0 + i) * max_hops + h;
            hop_node[at] = r.es_node >> 16;
            if (hop_s) {
              hop_s[at] = r.es_node & 0xffff;
              hop_e[at] = r.ee;
            }
          }
          ++h;
          covered = r.ee;
          v = r.dst;
        }
        if (ok) {
          samples += 1.0;
          avg += ((double)out_s[i] - avg) / samples;
        } else {
          ++den;
        }
        nh[c0 + i] = ok ? h : -1;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    *deferred = den + scal[2];
    if (passes_out) *passes_out = passes_total;
  }
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
  int32_t *d_vord = nullptr, *d_passes = nullptr;
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
    TRY(ar.take(&d_vord, 3 * nv + 2 + ne));
    TRY(ar.take(&d_passes, 1));
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
  // pinned staging of the pageable request stream and outputs (large calls)
  char* pin = nullptr;
  const size_t out_bytes = 4 * (size_t)R + (max_hops > 0 ? 4 * HR * (want_se ? 3 : 1) : 0);
  const bool stage_io = !rc && R >= (int64_t(1) << 18) && !(is_pinned(h_in) && is_pinned(h_nh)) &&
                        host_pin(ctx, std::max<size_t>(8 * (size_t)R, out_bytes), &pin) == HELIO_OK;
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
    // large pageable request streams go through a pinned staging buffer
    // (threaded host copies, then full-speed DMA), the outputs likewise below
    if (stage_io && !rc) {
      stage_copy(pin, h_in, 4 * R);
      stage_copy(pin + 4 * R, h_out, 4 * R);
      H2D(d_in, pin, 4 * R);
      H2D(d_out, pin + 4 * R, 4 * R);
    } else {
      H2D(d_in, h_in, 4 * R);
      H2D(d_out, h_out, 4 * R);
    }
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
      std::vector<int32_t> cl;
      if (consistent || head + (size_t)slots * sizeof(SlotRec) > 227 * 1024) {
        cl.resize(nv);
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
        // node-consistent plans: the chunked parallel replay (route_masked_spec)
        // vertices routed from (the coordinator, then every vertex ending
        // before L) in end-layer order, and each one's predecessors
        std::vector<int32_t> vo, kof(nv, -1), meta;
        for (int x = 0; x < nv; ++x)
          if (x == 0 || vend[x] < L) vo.push_back(x);
        std::stable_sort(vo.begin(), vo.end(), [&](int a, int b) { return vend[a] < vend[b]; });
        const int nvo = (int)vo.size();
        for (int k = 0; k < nvo; ++k) kof[vo[k]] = k;
        std::vector<std::vector<int32_t>> preds(nvo);
        for (int x = 0; x < nv; ++x)
          for (int p = obeg[x]; p < obeg[x + 1]; ++p)
            if (kof[x] >= 0 && odst[p] != 0 && kof[odst[p]] >= 0) preds[kof[odst[p]]].push_back(kof[x]);
        meta = vo;
        meta.push_back(0);
        for (int k = 0; k < nvo; ++k) {
          std::sort(preds[k].begin(), preds[k].end());
          preds[k].erase(std::unique(preds[k].begin(), preds[k].end()), preds[k].end());
          meta.push_back(meta[nvo + k] + (int32_t)preds[k].size());
        }
        for (int k = 0; k < nvo; ++k) meta.insert(meta.end(), preds[k].begin(), preds[k].end());
        {  // leaves (no successor among the routed vertices): a group is done
           // everywhere once every leaf is done with it
          std::vector<char> has_succ(nvo, 0);
          for (int k = 0; k < nvo; ++k)
            for (int u : preds[k]) has_succ[u] = 1;
          std::vector<int32_t> leaves;
          for (int k = 0; k < nvo; ++k)
            if (!has_succ[k]) leaves.push_back(k);
          meta.push_back((int32_t)leaves.size());
          meta.insert(meta.end(), leaves.begin(), leaves.end());
        }
        constexpr int G1 = kSpecGroups + 1;
        auto a16 = [](size_t b) { return (b + 15) & ~size_t(15); };
        // longest route in picks (vertices of vorder along a path from the
        // coordinator): the approximate pass records the vertices visited
        int hmax = 0;
        {
          std::vector<int> picks(nvo, 0);
          for (int k = 0; k < nvo; ++k) {
            int best = 0;
            for (int j = meta[nvo + k]; j < meta[nvo + k + 1]; ++j) best = std::max(best, picks[meta[2 * nvo + 1 + j]]);
            picks[k] = best + 1;
            hmax = std::max(hmax, picks[k]);
          }
          const char* ap = getenv("HELIO_ROUTE_APPROX");
          if (hmax > 32 || nv > 256 || (ap && ap[0] == '0')) hmax = 0;  // exact passes only (route_v is 8-bit)
        }
        int pair_cap = 0;  // the coordinator's two-step table, when small
        if (!cl.empty()) {
          const int64_t d1 = obeg[1] - obeg[0] + 1;
          if (d1 * d1 * cl[0] <= 8192) pair_cap = (int)(d1 * d1 * cl[0]);
        }
        int64_t nxt_cap = 0;  // position tables: (deg + 1) * W per vertex
        for (int x = 0; x < nv && !cl.empty(); ++x) {
          const int deg = obeg[x + 1] - obeg[x];
          if (deg > 0) nxt_cap += (int64_t)(deg + 1) * cl[x];
        }
        const size_t spec_smem = a16(8 * kSpecChunk) + a16(kSpecChunk) + a16((size_t)kSpecChunk * hmax) + 2 * a16(8 * kSpecChunk) + 2 * a16(4 * kSpecChunk) + 2 * a16(2 * kSpecChunk) +
                                 2 * a16(kSpecChunk) + a16(8 * G1) + a16(4 * G1) + a16(2 * (size_t)nvo * G1) +
                                 a16(4 * (nvo + 1)) + a16(4 * nvo) + a16(4 * nv) + a16(8 * nv) +
                                 2 * a16(8 * (size_t)ne) + a16(2 * (size_t)ne) + a16(4 * (nv + 1)) +
                                 a16(2 * (size_t)nxt_cap) + a16(4 * kSpecThreads) + a16(2 * (size_t)pair_cap) + 16 * 32 + 32 + (size_t)slots * sizeof(SlotRec);
        const char* sp_env = getenv("HELIO_ROUTE_SPEC");
        const bool use_spec = consistent && !cl.empty() && spec_smem <= 227 * 1024 && obeg[1] - obeg[0] < 256 /* cls0 is 8-bit */ &&
                              (int)meta.size() <= 3 * nv + 2 + ne && !(sp_env && sp_env[0] == '0');
        if (use_spec) {
          if (cudaMemcpyAsync(d_vord, meta.data(), 4 * meta.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
            rc = fail(ctx, HELIO_ERR_CUDA, "route H2D failed");
          cudaFuncSetAttribute(route_masked_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)spec_smem);
          const bool diag = getenv("HELIO_ROUTE_DIAG") != nullptr;
          cudaEvent_t e0 = nullptr, e1 = nullptr;
          if (diag) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, st);
          }
          if (!rc)
            route_masked_spec<<<1, kSpecThreads, spec_smem, st>>>(
                R, nv, L, max_hops, ctx->kv_token_layer_bytes, d_obeg, d_odst, d_oes, d_oee, d_node, d_kvcap,
                d_cyclen, d_cyc, nvo, d_vord, (int)nxt_cap, pair_cap, hmax, d_in, d_out, d_nh, d_hn, want_se ? d_hs : nullptr,
                want_se ? d_he : nullptr, d_den, d_passes);
          ctx->launches++;
          if (diag) {  // kernel time and passes (tools/route_spec_probe.py)
            int passes = 0;
            float ms = 0.f;
            cudaEventRecord(e1, st);
            cudaMemcpyAsync(&passes, d_passes, 4, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            cudaEventElapsedTime(&ms, e0, e1);
            fprintf(stderr, "route_masked_spec: %lld requests, %d chunk passes, %.3f ms\n", (long long)R, passes, ms);
#ifdef SPEC_PROFILE
            {
              std::vector<long long> pr(8192);
              cudaMemcpyFromSymbol(pr.data(), spec_prof, 8 * 8192);
              fprintf(stderr, "SPECPROF nvo=%d", nvo);
              for (int q = 0; q < 8192; ++q) fprintf(stderr, " %lld", pr[q]);
              fprintf(stderr, "\n");
            }
#endif
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
          }
        } else {
        auto kern = nv <= 32 ? (consistent ? route_masked_warp<true, false> : route_masked_warp<true, true>)
                             : (consistent ? route_masked_warp<false, false> : route_masked_warp<false, true>);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, 32, smem, st>>>(R, nv, L, max_hops, ctx->kv_token_layer_bytes, d_obeg, d_odst, d_oes, d_oee, d_node,
                                  d_kvcap, d_cyclen, d_cyc, d_in, d_out, d_nh, d_hn, want_se ? d_hs : nullptr,
                                  want_se ? d_he : nullptr, d_den, d_err);
        ctx->launches++;
        }
      }
      if (cudaGetLastError() != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "route_masked_warp failed");
    }
  }
  int herr = 0;
  if (!rc && R > 0) {
    // destinations: the caller's buffers, or the pinned staging buffer
    int32_t* o_nh = stage_io ? reinterpret_cast<int32_t*>(pin) : h_nh;
    int32_t* o_hn = stage_io ? o_nh + R : h_hn;
    int32_t* o_hs = stage_io ? o_hn + HR : h_hs;
    int32_t* o_he = stage_io ? o_hs + HR : h_he;
    bool ok = cudaMemcpyAsync(o_nh, d_nh, 4 * R, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
              cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, st) == cudaSuccess;
    if (ok && max_hops > 0) ok = cudaMemcpyAsync(o_hn, d_hn, 4 * HR, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    if (ok && max_hops > 0 && want_se)
      ok = cudaMemcpyAsync(o_hs, d_hs, 4 * HR, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
           cudaMemcpyAsync(o_he, d_he, 4 * HR, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    long long dd = 0;
    if (ok && !closed) ok = cudaMemcpyAsync(&dd, d_den, sizeof(long long), cudaMemcpyDeviceToHost, st) == cudaSuccess;
    ok = ok && cudaStreamSynchronize(st) == cudaSuccess;
    if (!ok) rc = fail(ctx, HELIO_ERR_CUDA, std::string("route: ") + cudaGetErrorString(cudaGetLastError()));
    if (!rc && stage_io) {
      stage_copy(h_nh, o_nh, 4 * R);
      if (max_hops > 0) stage_copy(h_hn, o_hn, 4 * HR);
      if (max_hops > 0 && want_se) {
        stage_copy(h_hs, o_hs, 4 * HR);
        stage_copy(h_he, o_he, 4 * HR);
      }
    }
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
