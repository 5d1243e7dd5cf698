// helio_gpu.cu — B200 (sm_100a) engine behind include/helio_gpu.h.
//
// Kernels (SIMT; the path is FP64 min/add/compare graph work — no tensor
// cores):
//
//   K1+K2  score_kernel   placement rows -> split-node flow network in shared
//                         memory -> FIFO preflow-push max-flow -> value.
//                         One warp per graph, persistent CTAs pulling work from
//                         an atomic counter.  PARITY semantics: the discharge
//                         sequence of src/flow_graph.cpp:138-229 is replayed
//                         exactly (ballot = the sequential admissible-arc
//                         scan), so values AND per-edge flows are bit-identical
//                         to the reference's doubles.  Graphs whose arcs exceed
//                         the small slot are queued and finished by the same
//                         kernel launched with one warp per CTA and a large slot.
//   raw    raw_kernel     max_flow on caller-supplied raw graphs (AC1 style).
//   K4     argmax         (max value, min index) reduction (enumerate.hpp:59).
//   gen    gen_kernel     counter-based candidate generator (gen.h).
//   K3     route kernels  IWRR routing (scheduler.cpp:28-190), see route section.
//
// Everything is compiled with -fmad=false; the only FP operations on the path
// are min / + / - / compare on doubles (flow) and the iwrr_weights scaling,
// exactly the reference's operations in the reference's order.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
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

namespace {

Layout make_layout(int V, int A, int N, int M) {
  Layout l;
  l.V = V; l.A = A; l.N = N; l.M = M;
  int o = 0;
  auto take = [&](int bytes, int align) {
    o = (o + align - 1) / align * align;
    int r = o;
    o += bytes;
    return r;
  };
  l.o_cap = take(8 * A, 16);
  // 16 B per vertex: PARITY's packed VState; SCORE reuses the bytes as a
  // double array (bottleneck) followed by an int16 array (BFS parent arc).
  l.o_vs = take(16 * V, 16);
  l.o_ex = l.o_vs;
  l.o_h = l.o_vs + 8 * V;
  l.o_to = take(2 * A, 2);
  l.o_rv = take(2 * A, 2);
  l.o_abeg = take(2 * (V + 1), 2);
  l.o_cur = take(2 * V, 2);
  l.o_q = take(2 * V, 2);
  l.o_cnt = take(2 * (2 * V + 1), 2);
  l.o_ps = take(2 * N, 4);
  l.o_pe = take(2 * N, 2);
  l.o_vin = take(2 * N, 2);
  l.o_unode = take(2 * N, 2);
  l.o_efwd = take(2 * M, 2);
  l.o_inq = take(V, 1);
  l.bytes = (o + 15) / 16 * 16;
  return l;
}

// PARITY per-vertex solver state, one 16-byte shared-memory record so a
// discharge loads it with a single LDS.128.
struct __align__(16) VState {
  double ex;     // excess
  int16_t h;     // height
  int16_t cur;   // current-arc index (relative)
  int16_t b;     // first arc
  int16_t deg;   // arc count
};

// Per-warp view of a slot.
struct Gs {
  VState* vs;
  double* cap;
  double* ex;
  int16_t* to;
  int16_t* rv;
  int16_t* abeg;
  int16_t* h;
  int16_t* cur;
  int16_t* q;
  int16_t* cnt;
  uint8_t* inq;
  int16_t* ps;
  int16_t* pe;
  int16_t* vin;
  int16_t* unode;
  int16_t* efwd;
};

__device__ __forceinline__ Gs slot_view(char* base, const Layout& l) {
  Gs g;
  g.vs = reinterpret_cast<VState*>(base + l.o_vs);
  g.cap = reinterpret_cast<double*>(base + l.o_cap);
  g.ex = reinterpret_cast<double*>(base + l.o_ex);
  g.to = reinterpret_cast<int16_t*>(base + l.o_to);
  g.rv = reinterpret_cast<int16_t*>(base + l.o_rv);
  g.abeg = reinterpret_cast<int16_t*>(base + l.o_abeg);
  g.h = reinterpret_cast<int16_t*>(base + l.o_h);
  g.cur = reinterpret_cast<int16_t*>(base + l.o_cur);
  g.q = reinterpret_cast<int16_t*>(base + l.o_q);
  g.cnt = reinterpret_cast<int16_t*>(base + l.o_cnt);
  g.inq = reinterpret_cast<uint8_t*>(base + l.o_inq);
  g.ps = reinterpret_cast<int16_t*>(base + l.o_ps);
  g.pe = reinterpret_cast<int16_t*>(base + l.o_pe);
  g.vin = reinterpret_cast<int16_t*>(base + l.o_vin);
  g.unode = reinterpret_cast<int16_t*>(base + l.o_unode);
  g.efwd = reinterpret_cast<int16_t*>(base + l.o_efwd);
  return g;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// std::min(a, b) == (b < a) ? b : a
__device__ __forceinline__ double ref_min(double a, double b) { return b < a ? b : a; }

// ---------------------------------------------------------------------------
// FIFO preflow-push with the gap heuristic, warp-cooperative replay of
// max_flow (flow_graph.cpp:147-208).  Arcs for vertex x are
// [abeg[x], abeg[x+1]) in the reference's adjacency order; rv[] is the global
// index of the paired arc.  On return cap[] holds residual capacities.
//
// Replay argument: while vertex u discharges, nothing but u's own pushes
// changes state, and a push either drains u (loop ends, current stays on the
// arc) or saturates the arc to exactly 0.0 (the reference then re-tests it,
// fails, and advances).  So "first admissible arc at index >= current" — one
// ballot over 32 arcs — is exactly the arc the sequential scan reaches.
// Relabel is a warp min-reduce (:183-186); the gap sweep (:190-198) only moves
// integer counts, so it is done lane-parallel.  Queue order is preserved
// because enqueues happen in push order.
// (implemented by solve_fifo2 below)

// ---------------------------------------------------------------------------
// SCORE mode: value-only Edmonds-Karp (shortest augmenting paths), one warp
// per graph — see solve_ek_batched below.  Exact on integer capacities (every
// intermediate is an integer-valued double); on float capacities the value
// differs from the reference's FIFO preflow-push only by rounding (north_star
// tolerance 1e-6 relative; tests assert it).  Slot reuse: h = BFS parent arc,
// q = BFS queue, ex = bottleneck capacity from the source.

// ---------------------------------------------------------------------------
// PARITY solver (the replay argued above), with little bookkeeping per step: per-vertex state in one 16-byte VState (one LDS.128 per pop, one
// STS.128 per write-back), the in-queue set in registers when n <= 128
// (every lane holds the same two 64-bit words, so the enqueue test is a
// uniform register test), and a failed scan of the last arc chunk falls
// straight into the relabel instead of taking another loop trip.
__device__ void solve_fifo2(const Gs& g, const int n, const int s, const int t, const int lane) {
  VState* vs = g.vs;
  for (int x = lane; x < n; x += 32) {
    VState v;
    v.ex = 0.0;
    v.h = (x == s) ? (int16_t)n : (int16_t)0;
    v.cur = 0;
    v.b = g.abeg[x];
    v.deg = (int16_t)(g.abeg[x + 1] - g.abeg[x]);
    vs[x] = v;
    g.inq[x] = 0;
  }
  for (int x = lane; x <= 2 * n; x += 32) g.cnt[x] = 0;
  __syncwarp();
  if (lane == 0) {
    g.cnt[0] = (int16_t)(n - 1);
    g.cnt[n] += 1;
  }
  // in-queue flags: every lane writes them and every lane reads its own
  // write, so no cross-lane ordering is needed (a byte test beat a register
  // bitmask on issue slots)
  auto in_queue = [&](int x) -> bool { return g.inq[x] != 0; };
  auto mark = [&](int x, bool on) { g.inq[x] = on ? 1 : 0; };
  int tail = 0, qcount = 0;
  // saturate source arcs in adjacency order (:168-173): uniform loop, lane 0 stores
  __syncwarp();
  {
    const int b = g.abeg[s], e = g.abeg[s + 1];
    for (int a = b; a < e; ++a) {
      __syncwarp();
      const double c = g.cap[a];
      if (c > FLOW_EPS) {
        const int to = g.to[a];
        const int r = g.rv[a];
        double exs = vs[s].ex + c;
        const double amt = ref_min(exs, g.cap[a]);
        __syncwarp();
        if (lane == 0) {
          vs[s].ex = exs;
          g.cap[a] -= amt;
          g.cap[r] += amt;
          vs[s].ex -= amt;
          vs[to].ex += amt;
        }
        __syncwarp();
        if (to != s && to != t && !in_queue(to)) {
          mark(to, true);
          if (lane == 0) g.q[tail] = (int16_t)to;
          tail = tail + 1 == n ? 0 : tail + 1;
          ++qcount;
        }
      }
    }
  }
  int head = 0;
  const int two_n = 2 * n;
  while (qcount > 0) {
    __syncwarp();
    const int u = g.q[head];
    head = head + 1 == n ? 0 : head + 1;
    --qcount;
    const VState su = vs[u];
    double ex = su.ex;
    int hu = su.h;
    int cu = su.cur;
    const int b = su.b;
    const int deg = su.deg;
    mark(u, false);
    int kl = -1;
    bool inr = false;
    double ca = 0.0;
    int ta = 0, ra = 0, hta = 0;
    while (ex > FLOW_EPS) {
      if (cu < deg) {
        const int k = cu >> 5;
        if (k != kl) {
          const int jr = (k << 5) + lane;
          inr = jr < deg;
          if (inr) {
            const int a = b + jr;
            ca = g.cap[a];
            ta = g.to[a];
            ra = g.rv[a];
            hta = vs[ta].h;
          }
          kl = k;
        }
        const int jr = (k << 5) + lane;
        const bool adm = inr && jr >= cu && ca > FLOW_EPS && hu == hta + 1;
        const unsigned m = __ballot_sync(FULL, adm);
        if (m != 0u) {
          const int j = __ffs(m) - 1;
          cu = (k << 5) + j;
          const double cj = __shfl_sync(FULL, ca, j);
          const int tj = __shfl_sync(FULL, ta, j);
          const double amt = ref_min(ex, cj);  // push (:156-166)
          if (lane == j) {
            ca -= amt;
            g.cap[b + cu] = ca;
            g.cap[ra] += amt;
          }
          if (lane == 0) vs[tj].ex += amt;
          ex -= amt;
          if (tj != s && tj != t && !in_queue(tj)) {
            mark(tj, true);
            if (lane == 0) g.q[tail] = (int16_t)tj;
            tail = tail + 1 == n ? 0 : tail + 1;
            ++qcount;
          }
          continue;
        }
        cu = min(deg, (k + 1) << 5);
        if (cu < deg) continue;
      }
      // relabel (:180-199)
      const int old = hu;
      int best = two_n;
      const int nch = (deg + 31) >> 5;
      for (int k = 0; k < nch; ++k) {
        if (k != kl) {
          const int jr = (k << 5) + lane;
          inr = jr < deg;
          if (inr) {
            const int a = b + jr;
            ca = g.cap[a];
            ta = g.to[a];
            ra = g.rv[a];
            hta = vs[ta].h;
          }
          kl = k;
        }
        const int cand = (inr && ca > FLOW_EPS) ? hta + 1 : two_n;
        best = min(best, __reduce_min_sync(FULL, cand));
      }
      hu = best;
      cu = 0;
      int cold = 0;
      if (lane == 0) {
        vs[u].h = (int16_t)best;
        cold = g.cnt[old] - 1;
        g.cnt[old] = (int16_t)cold;
        g.cnt[best] += 1;
      }
      cold = __shfl_sync(FULL, cold, 0);
      __syncwarp();
      if (old < n && cold == 0) {
        int moved = 0;
        for (int x = lane; x < n; x += 32) {
          const int hx = vs[x].h;
          if (x != s && hx > old && hx < n) {
            vs[x].h = (int16_t)(n + 1);
            ++moved;
          }
        }
        moved = __reduce_add_sync(FULL, moved);
        for (int hh = old + 1 + lane; hh < n; hh += 32) g.cnt[hh] = 0;
        __syncwarp();
        if (lane == 0) g.cnt[n + 1] += (int16_t)moved;
        if (hu > old && hu < n) hu = n + 1;
        if (inr) hta = vs[ta].h;
      }
      if (inr && ta == u) hta = hu;  // self-loop arcs see u's new height
      if (best >= two_n) break;
    }
    if (lane == 0) {
      VState w;
      w.ex = ex;
      w.h = (int16_t)hu;
      w.cur = (int16_t)cu;
      w.b = (int16_t)b;
      w.deg = (int16_t)deg;
      vs[u] = w;
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// K1: build the reference's FlowGraph for one placement row into the slot.
// Vertex numbering (flow_graph.cpp:63-69): source 0, sink 1, then (in, out)
// pairs of the used nodes in byte-lexicographic id order.  Edge order: compute
// edges in that order (:71-84), then valid links in declaration order
// (:86-134).  Arc order per vertex = edge order (:140-145), which for these
// graphs is: the compute arc first, then link arcs in link order; so the
// position of a link's arc at a vertex is 1 (0 at source/sink) + the number of
// earlier valid links touching that vertex — a running counter per vertex,
// advanced per 32-link chunk with __match_any_sync.
//
// Returns status (0 ok, 1-3 validation, ST_OVERFLOW), V and E.

struct LinkEval {
  bool valid;
  int u, v;
};

__device__ __forceinline__ LinkEval eval_link(const ClusterDev& cd, const Gs& g, int l, int partial) {
  LinkEval r{false, 0, 0};
  const uint32_t pk = __ldg(cd.link_pack + l);
  const int a = (int)(pk & 0xffffu) - 1;
  const int bb = (int)(pk >> 16) - 1;
  if (a < 0) {  // coordinator -> bb (:89-101)
    const int vb = g.vin[bb];
    if (vb >= 0 && g.ps[bb] == 0) {
      r.valid = true;
      r.u = 0;
      r.v = vb;
    }
  } else if (bb < 0) {  // a -> coordinator (:102-114)
    const int va = g.vin[a];
    if (va >= 0 && g.pe[a] == cd.L) {
      r.valid = true;
      r.u = va + 1;
      r.v = 1;
    }
  } else {  // a -> bb (:115-133)
    const int va = g.vin[a], vb = g.vin[bb];
    if (va >= 0 && vb >= 0) {
      const int aend = g.pe[a], bs = g.ps[bb], be = g.pe[bb];
      const bool ok = partial ? (bs <= aend && aend < be) : (aend == bs);
      if (ok) {
        r.valid = true;
        r.u = va + 1;
        r.v = vb;
      }
    }
  }
  return r;
}

__device__ int build_graph(const ClusterDev& cd, const Gs& g, const Layout& lay, const int16_t* row,
                           int partial, int lane, int& V, int& E) {
  const int N = cd.N, L = cd.L;
  // placement + validation in id order (:52-61): first failing node in lex order
  int bad = INT_MAX;
  const int32_t* row32 = reinterpret_cast<const int32_t*>(row);
  for (int k = lane; k < N; k += 32) {
    const int32_t w = __ldg(row32 + k);
    const int s = (int16_t)(w & 0xffff);
    const int e = (int16_t)(w >> 16);
    g.ps[k] = (int16_t)s;
    g.pe[k] = (int16_t)e;
    g.vin[k] = -1;
    if (e > s) {
      int code = 0;
      if (s < 0 || e > L) code = 2;
      else if (e - s > __ldg(cd.kmax + k)) code = 3;
      if (code) bad = min(bad, __ldg(cd.lexrank + k) * 4 + code);
    }
  }
  bad = __reduce_min_sync(FULL, bad);
  if (bad != INT_MAX) return bad & 3;
  __syncwarp();
  // vertices in lex order (:63-69)
  int U = 0;
  for (int r0 = 0; r0 < N; r0 += 32) {
    const int r = r0 + lane;
    int k = -1;
    bool used = false;
    if (r < N) {
      k = __ldg(cd.lexnode + r);
      used = g.pe[k] > g.ps[k];
    }
    const unsigned m = __ballot_sync(FULL, used);
    if (used) {
      const int idx = U + __popc(m & lanemask_lt());
      g.vin[k] = (int16_t)(2 + 2 * idx);
      g.unode[idx] = (int16_t)k;
    }
    U += __popc(m);
  }
  V = 2 + 2 * U;
  // degree count: compute arc (1 per used vertex) + link arcs
  for (int x = lane; x < V; x += 32) g.cur[x] = x >= 2 ? 1 : 0;
  __syncwarp();
  int nvalid = 0;
  for (int l0 = 0; l0 < cd.Mv; l0 += 32) {
    const int l = l0 + lane;
    LinkEval le{false, 0, 0};
    if (l < cd.Mv) le = eval_link(cd, g, l, partial);
    const unsigned vm = __ballot_sync(FULL, le.valid);
    if (vm == 0u) continue;
    nvalid += __popc(vm);
    unsigned pu = 0, pv = 0;
    int cu = 0, cv = 0;
    if (le.valid) {
      pu = __match_any_sync(vm, le.u);
      pv = __match_any_sync(vm, le.v);
      cu = g.cur[le.u];
      cv = g.cur[le.v];
    }
    __syncwarp();
    if (le.valid) {
      const unsigned lt = lanemask_lt();
      if ((pu & lt) == 0u) g.cur[le.u] = (int16_t)(cu + __popc(pu));
      if ((pv & lt) == 0u) g.cur[le.v] = (int16_t)(cv + __popc(pv));
    }
    __syncwarp();
  }
  E = U + nvalid;
  if (V > lay.V || 2 * E > lay.A) return ST_OVERFLOW;
  // arc offsets: exclusive scan of degrees
  int run = 0;
  for (int x0 = 0; x0 < V; x0 += 32) {
    const int x = x0 + lane;
    const int d = x < V ? g.cur[x] : 0;
    int incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (x < V) g.abeg[x] = (int16_t)(run + incl - d);
    run += __shfl_sync(FULL, incl, 31);
  }
  if (lane == 0) g.abeg[V] = (int16_t)run;
  __syncwarp();
  // compute arcs (edge j = in_j -> out_j, cap compute_edge_capacity)
  for (int j = lane; j < U; j += 32) {
    const int k = g.unode[j];
    const int vi = 2 + 2 * j, vo = vi + 1;
    const int ai = g.abeg[vi], ao = g.abeg[vo];
    g.to[ai] = (int16_t)vo;
    g.rv[ai] = (int16_t)ao;
    g.cap[ai] = __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (g.pe[k] - g.ps[k]) - 1);
    g.to[ao] = (int16_t)vi;
    g.rv[ao] = (int16_t)ai;
    g.cap[ao] = 0.0;
  }
  for (int x = lane; x < V; x += 32) g.cur[x] = x >= 2 ? 1 : 0;
  __syncwarp();
  // link arcs at their ranked positions
  for (int l0 = 0; l0 < cd.Mv; l0 += 32) {
    const int l = l0 + lane;
    LinkEval le{false, 0, 0};
    if (l < cd.Mv) le = eval_link(cd, g, l, partial);
    const unsigned vm = __ballot_sync(FULL, le.valid);
    if (vm == 0u) continue;
    unsigned pu = 0, pv = 0;
    int cu = 0, cv = 0;
    if (le.valid) {
      pu = __match_any_sync(vm, le.u);
      pv = __match_any_sync(vm, le.v);
      cu = g.cur[le.u];
      cv = g.cur[le.v];
    }
    __syncwarp();
    if (le.valid) {
      const unsigned lt = lanemask_lt();
      const int fa = g.abeg[le.u] + cu + __popc(pu & lt);
      const int ra = g.abeg[le.v] + cv + __popc(pv & lt);
      g.to[fa] = (int16_t)le.v;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + l);
      g.to[ra] = (int16_t)le.u;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
      if ((pu & lt) == 0u) g.cur[le.u] = (int16_t)(cu + __popc(pu));
      if ((pv & lt) == 0u) g.cur[le.v] = (int16_t)(cv + __popc(pv));
    }
    __syncwarp();
  }
  return 0;
}

// SCORE-mode builder.  Same graph as build_graph up to vertex numbering and
// arc order, which the value does not depend on: node k owns vertices
// in = 2 + 2k, out = 3 + 2k (unused nodes keep no arcs), and each lane walks
// its node's precomputed out-/in-link lists instead of scanning every link
// of the cluster.  Validation and status codes are shared with build_graph.
__device__ __forceinline__ bool edge_ok(int aend, int bs, int be, int partial) {
  return partial ? (bs <= aend && aend < be) : (aend == bs);
}

__device__ int build_graph_score(const ClusterDev& cd, const Gs& g, const Layout& lay, const int16_t* row,
                                 int partial, int lane, int& V, int& E) {
  const int N = cd.N, L = cd.L;
  int bad = INT_MAX;
  const int32_t* row32 = reinterpret_cast<const int32_t*>(row);
  for (int k = lane; k < N; k += 32) {
    const int32_t w = __ldg(row32 + k);
    const int s = (int16_t)(w & 0xffff);
    const int e = (int16_t)(w >> 16);
    g.ps[k] = (int16_t)s;
    g.pe[k] = (int16_t)e;
    if (e > s) {
      int code = 0;
      if (s < 0 || e > L) code = 2;
      else if (e - s > __ldg(cd.kmax + k)) code = 3;
      if (code) bad = min(bad, __ldg(cd.lexrank + k) * 4 + code);
    }
  }
  bad = __reduce_min_sync(FULL, bad);
  if (bad != INT_MAX) return bad & 3;
  V = 2 + 2 * N;
  if (V > lay.V) return ST_OVERFLOW;
  __syncwarp();
  // degrees: in_k = compute + valid in-links + source arc; out_k = compute +
  // valid out-links + sink arc.
  int nedges = 0, dsrc = 0, dsink = 0;
  int* fill = reinterpret_cast<int*>(g.ex);  // int counters per vertex during the build
  for (int k = lane; k < N; k += 32) {
    const int s = g.ps[k], e = g.pe[k];
    int din = 0, dout = 0;
    if (e > s) {
      din = 1;
      dout = 1;
      ++nedges;
      for (int p = __ldg(cd.out_beg + k), pe_ = __ldg(cd.out_beg + k + 1); p < pe_; ++p) {
        const int j = __ldg(&cd.out_list[p].x);
        const int sj = g.ps[j], ej = g.pe[j];
        if (ej > sj && edge_ok(e, sj, ej, partial)) ++dout;
      }
      for (int p = __ldg(cd.in_beg + k), pe_ = __ldg(cd.in_beg + k + 1); p < pe_; ++p) {
        const int i = __ldg(&cd.in_list[p].x);
        const int si = g.ps[i], ei = g.pe[i];
        if (ei > si && edge_ok(ei, s, e, partial)) ++din;
      }
      nedges += dout - 1;  // each link edge counted once, at its source
      if (s == 0 && __ldg(cd.cout_link + k) >= 0) {
        ++din;
        ++dsrc;
        ++nedges;
      }
      if (e == L && __ldg(cd.cin_link + k) >= 0) {
        ++dout;
        ++dsink;
        ++nedges;
      }
    }
    g.cur[2 + 2 * k] = (int16_t)din;
    g.cur[3 + 2 * k] = (int16_t)dout;
  }
  nedges = __reduce_add_sync(FULL, nedges);
  dsrc = __reduce_add_sync(FULL, dsrc);
  dsink = __reduce_add_sync(FULL, dsink);
  E = nedges;
  if (2 * E > lay.A) return ST_OVERFLOW;
  if (lane == 0) {
    g.cur[0] = (int16_t)dsrc;
    g.cur[1] = (int16_t)dsink;
  }
  __syncwarp();
  int run = 0;
  for (int x0 = 0; x0 < V; x0 += 32) {
    const int x = x0 + lane;
    const int d = x < V ? g.cur[x] : 0;
    int incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (x < V) {
      g.abeg[x] = (int16_t)(run + incl - d);
      fill[x] = 0;
    }
    run += __shfl_sync(FULL, incl, 31);
  }
  if (lane == 0) g.abeg[V] = (int16_t)run;
  __syncwarp();
  // arcs: each lane places its node's compute pair and every edge it
  // sources; the paired reverse arc takes the next free slot at its head.
  for (int k = lane; k < N; k += 32) {
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    const int vi = 2 + 2 * k, vo = vi + 1;
    const int ai = g.abeg[vi] + atomicAdd(&fill[vi], 1);
    const int ao = g.abeg[vo] + atomicAdd(&fill[vo], 1);
    g.to[ai] = (int16_t)vo;
    g.rv[ai] = (int16_t)ao;
    g.cap[ai] = __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (e - s) - 1);
    g.to[ao] = (int16_t)vi;
    g.rv[ao] = (int16_t)ai;
    g.cap[ao] = 0.0;
    for (int p = __ldg(cd.out_beg + k), pe_ = __ldg(cd.out_beg + k + 1); p < pe_; ++p) {
      const int2 jl = __ldg(&cd.out_list[p]);
      const int sj = g.ps[jl.x], ej = g.pe[jl.x];
      if (!(ej > sj && edge_ok(e, sj, ej, partial))) continue;
      const int vj = 2 + 2 * jl.x;
      const int fa = g.abeg[vo] + atomicAdd(&fill[vo], 1);
      const int ra = g.abeg[vj] + atomicAdd(&fill[vj], 1);
      g.to[fa] = (int16_t)vj;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + jl.y);
      g.to[ra] = (int16_t)vo;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
    const int lc = __ldg(cd.cout_link + k);
    if (s == 0 && lc >= 0) {
      const int fa = g.abeg[0] + atomicAdd(&fill[0], 1);
      const int ra = g.abeg[vi] + atomicAdd(&fill[vi], 1);
      g.to[fa] = (int16_t)vi;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + lc);
      g.to[ra] = 0;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
    const int lk = __ldg(cd.cin_link + k);
    if (e == L && lk >= 0) {
      const int fa = g.abeg[vo] + atomicAdd(&fill[vo], 1);
      const int ra = g.abeg[1] + atomicAdd(&fill[1], 1);
      g.to[fa] = 1;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + lk);
      g.to[ra] = (int16_t)vo;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
  }
  __syncwarp();
  return 0;
}

// SCORE builder for N <= 64: node sets are 64-bit words.  cover[l] = nodes
// whose interval contains layer l, start[l] = nodes starting at l.  Node i's
// valid successors are (partial ? cover[e_i] : start[e_i]) & out_mask[i]
// (flow_graph.cpp:121: s_j <= e_i < e_j, resp. e_i == s_j), so each node
// visits only its ~2-3 actual edges instead of every link of the cluster.
__device__ int build_graph_score_small(const ClusterDev& cd, const Gs& g, const Layout& lay, const int16_t* row,
                                       int partial, int lane, int& V, int& E) {
  const int N = cd.N, L = cd.L;
  unsigned long long* cover = reinterpret_cast<unsigned long long*>(g.cap);  // [L] then start[L]; scratch
  unsigned long long* start = cover + L;
  int bad = INT_MAX;
  const int32_t* row32 = reinterpret_cast<const int32_t*>(row);
  for (int k = lane; k < N; k += 32) {
    const int32_t w = __ldg(row32 + k);
    const int s = (int16_t)(w & 0xffff);
    const int e = (int16_t)(w >> 16);
    g.ps[k] = (int16_t)s;
    g.pe[k] = (int16_t)e;
    if (e > s) {
      int code = 0;
      if (s < 0 || e > L) code = 2;
      else if (e - s > __ldg(cd.kmax + k)) code = 3;
      if (code) bad = min(bad, __ldg(cd.lexrank + k) * 4 + code);
    }
  }
  bad = __reduce_min_sync(FULL, bad);
  if (bad != INT_MAX) return bad & 3;
  V = 2 + 2 * N;
  if (V > lay.V || 2 * L > lay.A) return ST_OVERFLOW;  // cover/start scratch lives in cap[]
  for (int l = lane; l < 2 * L; l += 32) cover[l] = 0ull;
  __syncwarp();
  for (int k = lane; k < N; k += 32) {
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    const unsigned long long bit = 1ull << k;
    atomicOr(&start[s], bit);
    for (int l = s; l < e; ++l) atomicOr(&cover[l], bit);
  }
  __syncwarp();
  // successor sets (kept in registers; lanes own nodes lane, lane+32)
  unsigned long long T[2] = {0ull, 0ull};
  int* fill = reinterpret_cast<int*>(g.vs);
  for (int x = lane; x < V; x += 32) fill[x] = 0;
  __syncwarp();
  int nedges = 0, dsrc = 0, dsink = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = lane + 32 * q;
    if (k >= N) continue;
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    unsigned long long t = 0ull;
    if (e < L) t = (partial ? cover[e] : start[e]) & __ldg(cd.out_mask + k);
    T[q] = t;
    const int nt = __popcll(t);
    nedges += 1 + nt;
    int dout = 1 + nt, din = 1;
    if (s == 0 && __ldg(cd.cout_link + k) >= 0) {
      ++din;
      ++dsrc;
      ++nedges;
    }
    if (e == L && __ldg(cd.cin_link + k) >= 0) {
      ++dout;
      ++dsink;
      ++nedges;
    }
    atomicAdd(&fill[2 + 2 * k], din);
    atomicAdd(&fill[3 + 2 * k], dout);
    for (unsigned long long m = t; m; m &= m - 1) atomicAdd(&fill[2 + 2 * (__ffsll(m) - 1)], 1);  // in_j
  }
  nedges = __reduce_add_sync(FULL, nedges);
  dsrc = __reduce_add_sync(FULL, dsrc);
  dsink = __reduce_add_sync(FULL, dsink);
  E = nedges;
  if (2 * E > lay.A) return ST_OVERFLOW;
  __syncwarp();
  if (lane == 0) {
    fill[0] = dsrc;
    fill[1] = dsink;
  }
  __syncwarp();
  int run = 0;
  for (int x0 = 0; x0 < V; x0 += 32) {
    const int x = x0 + lane;
    const int d = x < V ? fill[x] : 0;
    int incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (x < V) g.abeg[x] = (int16_t)(run + incl - d);
    run += __shfl_sync(FULL, incl, 31);
  }
  if (lane == 0) g.abeg[V] = (int16_t)run;
  __syncwarp();
  for (int x = lane; x < V; x += 32) fill[x] = 0;
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = lane + 32 * q;
    if (k >= N) continue;
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    const int vi = 2 + 2 * k, vo = vi + 1;
    const int ai = g.abeg[vi] + atomicAdd(&fill[vi], 1);
    const int ao = g.abeg[vo] + atomicAdd(&fill[vo], 1);
    g.to[ai] = (int16_t)vo;
    g.rv[ai] = (int16_t)ao;
    g.cap[ai] = __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (e - s) - 1);
    g.to[ao] = (int16_t)vi;
    g.rv[ao] = (int16_t)ai;
    g.cap[ao] = 0.0;
    for (unsigned long long m = T[q]; m; m &= m - 1) {
      const int j = __ffsll(m) - 1;
      const int vj = 2 + 2 * j;
      const int fa = g.abeg[vo] + atomicAdd(&fill[vo], 1);
      const int ra = g.abeg[vj] + atomicAdd(&fill[vj], 1);
      g.to[fa] = (int16_t)vj;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + __ldg(cd.pair_link + k * N + j));
      g.to[ra] = (int16_t)vo;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
    const int lc = __ldg(cd.cout_link + k);
    if (s == 0 && lc >= 0) {
      const int fa = g.abeg[0] + atomicAdd(&fill[0], 1);
      const int ra = g.abeg[vi] + atomicAdd(&fill[vi], 1);
      g.to[fa] = (int16_t)vi;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + lc);
      g.to[ra] = 0;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
    const int lk = __ldg(cd.cin_link + k);
    if (e == L && lk >= 0) {
      const int fa = g.abeg[vo] + atomicAdd(&fill[vo], 1);
      const int ra = g.abeg[1] + atomicAdd(&fill[1], 1);
      g.to[fa] = 1;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + lk);
      g.to[ra] = (int16_t)vo;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
  }
  __syncwarp();
  return 0;
}

// Edmonds-Karp with a batched BFS: each step takes as many queued vertices as
// have <= 32 arcs between them and gives every lane one arc.  Lanes are in
// queue order, and a vertex reached twice in one step keeps its lowest lane,
// so the BFS tree — hence every augmenting path — is exactly that of the
// one-vertex-at-a-time BFS.
__device__ double solve_ek_batched(const Gs& g, const int n, const int s, const int t, const int lane) {
  double value = 0.0;
  const unsigned lt = lanemask_lt();
  const unsigned le = lt | (1u << lane);
  for (;;) {
    for (int x = lane; x < n; x += 32) g.h[x] = -1;
    __syncwarp();
    if (lane == 0) {
      g.h[s] = -2;
      g.q[0] = (int16_t)s;
      g.ex[s] = 1.0e300;
    }
    __syncwarp();
    int qh = 0, qt = 1;
    bool found = false;
    while (qh < qt) {
      const int avail = min(32, qt - qh);
      int vi = 0, bi = 0, di = 0;
      if (lane < avail) {
        vi = g.q[qh + lane];
        bi = g.abeg[vi];
        di = g.abeg[vi + 1] - bi;
      }
      int incl = di;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int d0 = __shfl_sync(FULL, di, 0);
      if (d0 > 32) {
        // a wide vertex: scan it alone, 32 arcs at a time
        const int u = vi, b = bi;
        const double bu = g.ex[__shfl_sync(FULL, u, 0)];
        const int ub = __shfl_sync(FULL, b, 0);
        for (int a0 = ub; a0 < ub + d0; a0 += 32) {
          const int a = a0 + lane;
          bool ok = false;
          int v = 0;
          double c = 0.0;
          if (a < ub + d0) {
            c = g.cap[a];
            if (c > FLOW_EPS) {
              v = g.to[a];
              ok = g.h[v] == -1;
            }
          }
          const unsigned m = __ballot_sync(FULL, ok);
          if (ok) {
            g.h[v] = (int16_t)a;
            g.q[qt + __popc(m & lt)] = (int16_t)v;
            g.ex[v] = ref_min(bu, c);
          }
          qt += __popc(m);
          if (__any_sync(FULL, ok && v == t)) {
            found = true;
            break;
          }
        }
        qh += 1;
      } else {
        const unsigned fit = __ballot_sync(FULL, lane < avail && incl <= 32);
        const int k = __popc(fit);  // >= 1: lane 0 fits (d0 <= 32)
        const int start = incl - di;
        const unsigned sm = __reduce_or_sync(FULL, (lane < k && di > 0) ? (1u << start) : 0u);
        const int total = __shfl_sync(FULL, incl, k - 1);
        const int slot = __popc(sm & le) - 1;
        const int su = slot < 0 ? 0 : slot;
        const int u_b = __shfl_sync(FULL, bi, su);
        const int u_st = __shfl_sync(FULL, start, su);
        const int u_v = __shfl_sync(FULL, vi, su);
        bool ok = false;
        int v = 0;
        double c = 0.0;
        if (lane < total) {
          const int a = u_b + (lane - u_st);
          c = g.cap[a];
          if (c > FLOW_EPS) {
            v = g.to[a];
            ok = g.h[v] == -1;
          }
        }
        const unsigned cand = __ballot_sync(FULL, ok);
        if (ok) {
          const unsigned peers = __match_any_sync(cand, v);
          ok = (peers & lt) == 0u;
        }
        const unsigned m = __ballot_sync(FULL, ok);
        if (ok) {
          const int a = u_b + (lane - u_st);
          g.h[v] = (int16_t)a;
          g.q[qt + __popc(m & lt)] = (int16_t)v;
          g.ex[v] = ref_min(g.ex[u_v], c);
        }
        qt += __popc(m);
        qh += k;
        if (__any_sync(FULL, ok && v == t)) found = true;
      }
      __syncwarp();
      if (found) break;
    }
    if (!found) break;
    const double f = g.ex[t];
    if (lane == 0) {
      int x = t;
      while (x != s) {
        const int a = g.h[x];
        const int r = g.rv[a];
        g.cap[a] -= f;
        g.cap[r] += f;
        x = g.to[r];
      }
    }
    __syncwarp();
    value += f;
  }
  return value;
}

// SCORE solver for n <= 128: Edmonds-Karp with a level-synchronous bitset
// BFS.  Lane l owns vertices l, l+32, l+64, l+96 and keeps, in registers, the
// set of their residual out-neighbours (two 64-bit words per vertex).  One
// BFS level is: OR the rows of owned frontier vertices, REDUX.OR across the
// warp, mask with the visited set.  Only BFS levels are stored; the
// augmenting path is recovered backwards from the sink (at each step the
// first arc, in adjacency order, from a vertex one level closer to the
// source with residual capacity).  Deterministic; exact on integer
// capacities like every SCORE path.
__device__ __forceinline__ bool bit128(unsigned long long w0, unsigned long long w1, int x) {
  return ((x < 64 ? w0 : w1) >> (x & 63)) & 1ull;
}

__device__ __forceinline__ unsigned long long warp_or64(unsigned long long v) {
  const unsigned lo = __reduce_or_sync(FULL, (unsigned)(v & 0xffffffffull));
  const unsigned hi = __reduce_or_sync(FULL, (unsigned)(v >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

// Pair closure: in this numbering a node's vertices are v and v^1 (in = 2+2k,
// out = 3+2k), joined by its compute arc.  When a BFS level reaches one half
// of a node whose pair arc has residual capacity, the other half joins the
// same level (a shift on the 128-bit frontier), so the BFS walks nodes rather
// than split vertices and needs about half the levels.  Paths remain valid
// augmenting paths and the choice stays deterministic.
__device__ __forceinline__ unsigned long long swap_pairs(unsigned long long x) {
  return ((x & 0x5555555555555555ull) << 1) | ((x & 0xAAAAAAAAAAAAAAAAull) >> 1);
}

__device__ double solve_ek_bits(const Gs& g, const int n, const int s, const int t, const int lane) {
  // rows R[x] (residual out-neighbours of x, 128 bits) in the VState region;
  // per-vertex BFS code (2*level, +1 if added by the pair closure) in the
  // count region; canonical parent arc per vertex in `cur`; the augmenting
  // path in the queue region.
  ulonglong2* R = reinterpret_cast<ulonglong2*>(g.vs);
  int16_t* dist = g.cnt;
  int16_t* par = g.cur;
  int16_t* path = g.q;
  for (int x = lane; x < n; x += 32) {
    unsigned long long r0 = 0ull, r1 = 0ull;
    for (int a = g.abeg[x], e = g.abeg[x + 1]; a < e; ++a) {
      if (g.cap[a] > FLOW_EPS) {
        const int y = g.to[a];
        if (y < 64) r0 |= 1ull << y;
        else r1 |= 1ull << (y - 64);
      }
    }
    R[x] = make_ulonglong2(r0, r1);
  }
  __syncwarp();
  double value = 0.0;
  for (;;) {
    // pair arcs with residual capacity: bit v set iff R[v] holds v^1 (v >= 2)
    unsigned long long P0, P1;
    {
      unsigned b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int v = lane + 32 * i;
        bool pr = false;
        if (v >= 2 && v < n) {
          const ulonglong2 r = R[v];
          const int w = v ^ 1;
          pr = ((w < 64 ? r.x : r.y) >> (w & 63)) & 1ull;
        }
        b[i] = __ballot_sync(FULL, pr);
      }
      P0 = ((unsigned long long)b[1] << 32) | b[0];
      P1 = ((unsigned long long)b[3] << 32) | b[2];
    }
    for (int x = lane; x < n; x += 32) dist[x] = (int16_t)(x == s ? 0 : -1);
    unsigned long long F0 = s < 64 ? (1ull << s) : 0ull, F1 = s < 64 ? 0ull : (1ull << (s - 64));
    unsigned long long V0 = F0, V1 = F1;
    int d = 0;
    bool found = false;
    for (;;) {
      unsigned long long a0 = 0ull, a1 = 0ull;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const unsigned long long w = (i < 2) ? F0 : F1;
        if ((w >> (lane + 32 * (i & 1))) & 1ull) {
          const ulonglong2 r = R[lane + 32 * i];
          a0 |= r.x;
          a1 |= r.y;
        }
      }
      unsigned long long n0 = warp_or64(a0) & ~V0;
      unsigned long long n1 = warp_or64(a1) & ~V1;
      if ((n0 | n1) == 0ull) break;
      ++d;
      const unsigned long long c0 = swap_pairs(n0 & P0) & ~V0 & ~n0;
      const unsigned long long c1 = swap_pairs(n1 & P1) & ~V1 & ~n1;
      n0 |= c0;
      n1 |= c1;
      V0 |= n0;
      V1 |= n1;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int sh = lane + 32 * (i & 1);
        const unsigned long long w = (i < 2) ? n0 : n1;
        const unsigned long long cw = (i < 2) ? c0 : c1;
        if ((w >> sh) & 1ull) dist[lane + 32 * i] = (int16_t)(2 * d + (int)((cw >> sh) & 1ull));
      }
      F0 = n0;
      F1 = n1;
      if (bit128(n0, n1, t)) {
        found = true;
        break;
      }
    }
    if (!found) break;
    __syncwarp();
    // canonical parent of every visited vertex: a closure vertex takes its
    // pair arc; otherwise the first arc, in adjacency order, back to a vertex
    // of the previous level with residual capacity
    for (int x = lane; x < n; x += 32) {
      const int cx = dist[x];
      if (cx <= 0) continue;
      const int want = (cx >> 1) - 1;
      for (int a = g.abeg[x], e = g.abeg[x + 1]; a < e; ++a) {
        const int u = g.to[a];
        const int r = g.rv[a];
        const bool ok = (cx & 1) ? (u == (x ^ 1)) : (dist[u] >= 0 && (dist[u] >> 1) == want && g.cap[r] > FLOW_EPS);
        if (ok) {
          par[x] = (int16_t)r;
          break;
        }
      }
    }
    __syncwarp();
    int len = 0;
    if (lane == 0) {
      int x = t;
      while (x != s) {
        const int a = par[x];
        path[len++] = (int16_t)a;
        x = g.to[g.rv[a]];
      }
    }
    len = __shfl_sync(FULL, len, 0);
    __syncwarp();
    double f = 1.0e300;
    for (int k = lane; k < len; k += 32) f = ref_min(f, g.cap[path[k]]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f = ref_min(f, __shfl_xor_sync(FULL, f, o));
    for (int k = lane; k < len; k += 32) {
      const int a = path[k];
      const int r = g.rv[a];
      const int v = g.to[a];
      const int u = g.to[r];
      const double ca = g.cap[a] - f;
      g.cap[a] = ca;
      g.cap[r] += f;
      if (ca <= FLOW_EPS) {
        if (v < 64) atomicAnd(&R[u].x, ~(1ull << v));
        else atomicAnd(&R[u].y, ~(1ull << (v - 64)));
      }
      if (u < 64) atomicOr(&R[v].x, 1ull << u);
      else atomicOr(&R[v].y, 1ull << (u - 64));
    }
    value += f;
    __syncwarp();
  }
  return value;
}

// PARITY builder for N <= 64: the reference's exact graph (vertex numbering in
// id order, edge order, per-vertex arc order) without scanning every link.
// Valid interconnects come from the per-layer cover/start masks as in the
// SCORE builder; an arc's position in its vertex's list is its link's rank
// among that vertex's valid links in declaration order, counted pairwise
// over the ~2-3 valid links (pair_link holds compacted = declaration-ordered
// link indices) and, for coordinator links, with the less_cout / less_cin
// masks.  Produces exactly what build_graph produces (same vin/unode/abeg/
// to/rv/cap), so solve_fifo2 and built_value are unchanged.
__device__ int build_graph_small(const ClusterDev& cd, const Gs& g, const Layout& lay, const int16_t* row,
                                 int partial, int lane, int& V, int& E) {
  const int N = cd.N, L = cd.L;
  unsigned long long* cover = reinterpret_cast<unsigned long long*>(g.cap);  // scratch until arcs are written
  unsigned long long* start = cover + L;
  unsigned long long* inmask = reinterpret_cast<unsigned long long*>(g.vs);  // [N] sources of valid links into node
  int bad = INT_MAX;
  const int32_t* row32 = reinterpret_cast<const int32_t*>(row);
  for (int k = lane; k < N; k += 32) {
    const int32_t w = __ldg(row32 + k);
    const int s = (int16_t)(w & 0xffff);
    const int e = (int16_t)(w >> 16);
    g.ps[k] = (int16_t)s;
    g.pe[k] = (int16_t)e;
    g.vin[k] = -1;
    if (e > s) {
      int code = 0;
      if (s < 0 || e > L) code = 2;
      else if (e - s > __ldg(cd.kmax + k)) code = 3;
      if (code) bad = min(bad, __ldg(cd.lexrank + k) * 4 + code);
    }
  }
  bad = __reduce_min_sync(FULL, bad);
  if (bad != INT_MAX) return bad & 3;
  if (2 * L > lay.A) return ST_OVERFLOW;
  for (int l = lane; l < 2 * L; l += 32) cover[l] = 0ull;
  for (int k = lane; k < N; k += 32) inmask[k] = 0ull;
  __syncwarp();
  // vertices in id order (:63-69)
  int U = 0;
  for (int r0 = 0; r0 < N; r0 += 32) {
    const int r = r0 + lane;
    int k = -1;
    bool used = false;
    if (r < N) {
      k = __ldg(cd.lexnode + r);
      used = g.pe[k] > g.ps[k];
    }
    const unsigned m = __ballot_sync(FULL, used);
    if (used) {
      const int idx = U + __popc(m & lanemask_lt());
      g.vin[k] = (int16_t)(2 + 2 * idx);
      g.unode[idx] = (int16_t)k;
    }
    U += __popc(m);
  }
  V = 2 + 2 * U;
  for (int k = lane; k < N; k += 32) {
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    const unsigned long long bit = 1ull << k;
    atomicOr(&start[s], bit);
    for (int l = s; l < e; ++l) atomicOr(&cover[l], bit);
  }
  __syncwarp();
  // successor sets T (registers; lanes own nodes lane, lane + 32) and the
  // coordinator-link sets SRC (coord -> node valid) / SNK (node -> coord valid)
  unsigned long long T[2] = {0ull, 0ull};
  bool src_ok[2] = {false, false}, snk_ok[2] = {false, false};
  int nedges = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = lane + 32 * q;
    if (k >= N) continue;
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    unsigned long long t = 0ull;
    if (e < L) t = (partial ? cover[e] : start[e]) & __ldg(cd.out_mask + k);
    T[q] = t;
    for (unsigned long long m = t; m; m &= m - 1) atomicOr(&inmask[__ffsll(m) - 1], 1ull << k);
    src_ok[q] = s == 0 && __ldg(cd.cout_link + k) >= 0;
    snk_ok[q] = e == L && __ldg(cd.cin_link + k) >= 0;
    nedges += 1 + __popcll(t) + (src_ok[q] ? 1 : 0) + (snk_ok[q] ? 1 : 0);
  }
  const unsigned long long SRC =
      ((unsigned long long)__ballot_sync(FULL, src_ok[1]) << 32) | __ballot_sync(FULL, src_ok[0]);
  const unsigned long long SNK =
      ((unsigned long long)__ballot_sync(FULL, snk_ok[1]) << 32) | __ballot_sync(FULL, snk_ok[0]);
  E = __reduce_add_sync(FULL, nedges);
  if (V > lay.V || 2 * E > lay.A) return ST_OVERFLOW;
  __syncwarp();
  // degrees -> arc offsets
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = lane + 32 * q;
    if (k >= N || g.vin[k] < 0) continue;
    const int vi = g.vin[k];
    g.cur[vi] = (int16_t)(1 + __popcll(inmask[k]) + (src_ok[q] ? 1 : 0));
    g.cur[vi + 1] = (int16_t)(1 + __popcll(T[q]) + (snk_ok[q] ? 1 : 0));
  }
  if (lane == 0) {
    g.cur[0] = (int16_t)__popcll(SRC);
    g.cur[1] = (int16_t)__popcll(SNK);
  }
  __syncwarp();
  int run = 0;
  for (int x0 = 0; x0 < V; x0 += 32) {
    const int x = x0 + lane;
    const int d = x < V ? g.cur[x] : 0;
    int incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (x < V) g.abeg[x] = (int16_t)(run + incl - d);
    run += __shfl_sync(FULL, incl, 31);
  }
  if (lane == 0) g.abeg[V] = (int16_t)run;
  __syncwarp();
  // rank of link (src -> dst) among dst's valid incoming links, after the compute arc
  auto in_rank = [&](int dst, int lidx) -> int {
    int r = 1;
    for (unsigned long long m = inmask[dst]; m; m &= m - 1) {
      const int i = __ffsll(m) - 1;
      r += __ldg(cd.pair_link + i * N + dst) < lidx;
    }
    const int lc = __ldg(cd.cout_link + dst);
    if (g.ps[dst] == 0 && lc >= 0 && lc < lidx) ++r;
    return r;
  };
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = lane + 32 * q;
    if (k >= N || g.vin[k] < 0) continue;
    const int s = g.ps[k], e = g.pe[k];
    const int vi = g.vin[k], vo = vi + 1;
    const int ai = g.abeg[vi], ao = g.abeg[vo];
    // compute edge: forward first at in, reverse first at out (:140-145)
    g.to[ai] = (int16_t)vo;
    g.rv[ai] = (int16_t)ao;
    g.cap[ai] = __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (e - s) - 1);
    g.to[ao] = (int16_t)vi;
    g.rv[ao] = (int16_t)ai;
    g.cap[ao] = 0.0;
    const int lk = __ldg(cd.cin_link + k);
    // node -> node links, ranked among this out-vertex's valid links
    for (unsigned long long m = T[q]; m; m &= m - 1) {
      const int j = __ffsll(m) - 1;
      const int lidx = __ldg(cd.pair_link + k * N + j);
      int ro = 1;
      for (unsigned long long m2 = T[q]; m2; m2 &= m2 - 1)
        ro += __ldg(cd.pair_link + k * N + (__ffsll(m2) - 1)) < lidx;
      if (snk_ok[q] && lk < lidx) ++ro;
      const int vj = g.vin[j];
      const int fa = ao + ro;
      const int ra = g.abeg[vj] + in_rank(j, lidx);
      g.to[fa] = (int16_t)vj;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + lidx);
      g.to[ra] = (int16_t)vo;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
    if (src_ok[q]) {  // coordinator -> k
      const int lc = __ldg(cd.cout_link + k);
      const int fa = g.abeg[0] + __popcll(SRC & __ldg(cd.less_cout + k));
      const int ra = ai + in_rank(k, lc);
      g.to[fa] = (int16_t)vi;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + lc);
      g.to[ra] = 0;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
    if (snk_ok[q]) {  // k -> coordinator
      int ro = 1;
      for (unsigned long long m2 = T[q]; m2; m2 &= m2 - 1)
        ro += __ldg(cd.pair_link + k * N + (__ffsll(m2) - 1)) < lk;
      const int fa = ao + ro;
      const int ra = g.abeg[1] + __popcll(SNK & __ldg(cd.less_cin + k));
      g.to[fa] = 1;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + lk);
      g.to[ra] = (int16_t)vo;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    }
  }
  __syncwarp();
  return 0;
}

// Net flow into the sink in edge order (:222-227).  In built graphs the only
// edges touching the sink are node->coordinator links, whose order in
// g.edges equals the order of the sink's arcs.
__device__ double built_value(const ClusterDev& cd, const Gs& g, int lane) {
  double value = 0.0;
  if (lane == 0) {
    const int b = g.abeg[1], e = g.abeg[2];
    for (int a = b; a < e; ++a) {
      const int fa = g.rv[a];
      const int node = g.unode[(g.to[a] - 2) >> 1];
      double f = __ldg(cd.cin_cap + node) - g.cap[fa];
      if (f < FLOW_EPS) f = 0.0;
      value += f;
    }
  }
  return __shfl_sync(FULL, value, 0);
}

// Per-edge records in g.edges order with flows (:210-221).
__device__ void emit_edges(const ClusterDev& cd, const Gs& g, int U, int partial, int lane,
                           helio_edge* out) {
  for (int j = lane; j < U; j += 32) {
    const int k = g.unode[j];
    const int vi = 2 + 2 * j;
    const int ai = g.abeg[vi];
    const double c0 = __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (g.pe[k] - g.ps[k]) - 1);
    double f = c0 - g.cap[ai];
    if (f < FLOW_EPS) f = 0.0;
    helio_edge ed;
    ed.u = vi; ed.v = vi + 1; ed.kind = HELIO_EDGE_COMPUTE;
    ed.exec_start = g.ps[k]; ed.exec_end = g.pe[k];
    ed.src_node = k; ed.dst_node = k; ed.pad = 0;
    ed.cap = c0; ed.flow = f;
    out[j] = ed;
  }
  for (int x = lane; x < 2 + 2 * U; x += 32) g.cur[x] = x >= 2 ? 1 : 0;
  __syncwarp();
  int eidx = U;
  for (int l0 = 0; l0 < cd.Mv; l0 += 32) {
    const int l = l0 + lane;
    LinkEval le{false, 0, 0};
    if (l < cd.Mv) le = eval_link(cd, g, l, partial);
    const unsigned vm = __ballot_sync(FULL, le.valid);
    if (vm == 0u) continue;
    unsigned pu = 0;
    int cu = 0;
    if (le.valid) {
      pu = __match_any_sync(vm, le.u);
      cu = g.cur[le.u];
    }
    __syncwarp();
    if (le.valid) {
      const unsigned lt = lanemask_lt();
      const int fa = g.abeg[le.u] + cu + __popc(pu & lt);
      const uint32_t pk = __ldg(cd.link_pack + l);
      const int a = (int)(pk & 0xffffu) - 1, bb = (int)(pk >> 16) - 1;
      const double c0 = __ldg(cd.link_cap + l);
      double f = c0 - g.cap[fa];
      if (f < FLOW_EPS) f = 0.0;
      helio_edge ed;
      ed.u = le.u; ed.v = le.v;
      ed.src_node = a; ed.dst_node = bb; ed.pad = 0;
      if (a < 0) {
        ed.kind = HELIO_EDGE_COORD_OUT; ed.exec_start = 0; ed.exec_end = g.pe[bb];
      } else if (bb < 0) {
        ed.kind = HELIO_EDGE_COORD_IN; ed.exec_start = cd.L; ed.exec_end = cd.L;
      } else {
        ed.kind = HELIO_EDGE_INTERCONNECT; ed.exec_start = g.pe[a]; ed.exec_end = g.pe[bb];
      }
      ed.cap = c0; ed.flow = f;
      out[eidx + __popc(vm & lt)] = ed;
      if ((pu & lt) == 0u) g.cur[le.u] = (int16_t)(cu + __popc(pu));
    }
    eidx += __popc(vm);
    __syncwarp();
  }
}

struct FlowOut {
  helio_edge* edges;  // [B][max_e] or nullptr
  int32_t* nv;
  int32_t* ne;
  int max_e;
};

// Persistent: every warp loops fetching candidate indices.  big == 0: all B
// candidates, overflowing graphs appended to ovf; big == 1: the ovf list.
template <int MODE>
__global__ void score_kernel(ClusterDev cd, Layout lay, const int16_t* __restrict__ pl, int64_t B,
                             int partial, double* __restrict__ values, int32_t* __restrict__ status,
                             unsigned long long* work, int64_t* ovf, unsigned int* ovf_count,
                             int big, FlowOut fo) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Gs g = slot_view(smem + wib * lay.bytes, lay);
  const int64_t total = big ? (int64_t)(*ovf_count) : B;
  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(work, 1ull);
    w = __shfl_sync(FULL, w, 0);
    if ((int64_t)w >= total) break;
    const int64_t b = big ? ovf[w] : (int64_t)w;
    int V = 0, E = 0;
    int st = MODE == HELIO_MODE_SCORE
                 ? (cd.out_mask ? build_graph_score_small(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E)
                                : build_graph_score(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E))
                 : (cd.less_cout && !fo.edges
                        ? build_graph_small(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E)
                        : build_graph(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E));
    if (st == ST_OVERFLOW) {
      if (!big) {
        if (lane == 0) ovf[atomicAdd(ovf_count, 1u)] = b;
        continue;
      }
      st = HELIO_CAND_TOO_LARGE;
    }
    double value = 0.0;
    if (st == 0 && MODE == HELIO_MODE_SCORE) {
      value = V <= 128 ? solve_ek_bits(g, V, 0, 1, lane) : solve_ek_batched(g, V, 0, 1, lane);
    } else if (st == 0) {
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
      if (fo.nv) {
        fo.nv[b] = V;
        fo.ne[b] = E;
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// max_flow on raw graphs.  Arc construction follows :140-145 literally (lane
// 0, edge order; a self-loop's forward arc gets rev = itself because adj[v].
// size() is read before the push_back).
__global__ void raw_kernel(Layout lay, int64_t G, const int32_t* __restrict__ gn,
                           const int32_t* __restrict__ gs, const int32_t* __restrict__ gt,
                           const int64_t* __restrict__ eoff, const int32_t* __restrict__ eu,
                           const int32_t* __restrict__ ev, const double* __restrict__ ecap,
                           double* __restrict__ values, double* __restrict__ flows,
                           unsigned long long* work) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Gs g = slot_view(smem + wib * lay.bytes, lay);
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
  // big slot.  Arc budget 2 * (4N + 16) edges: covering chains average E ~3.3N
  // (het42: mean 140, p99 159, max 165 of 184; geo24 p99 98 of 112).
  int a_small = 2 * (4 * N + 16);
  int a_struct = 2 * (N + ctx->Mv);
  if (a_small > a_struct) a_small = a_struct;
  if (a_small < 2) a_small = 2;
  ctx->small = make_layout(V, a_small, N, 0);
  int warps = 4;
  ctx->small_warps = warps;
  const size_t max_smem = 227 * 1024;
  if ((size_t)ctx->small.bytes * warps > max_smem) {
    warps = 1;
    ctx->small_warps = 1;
  }
  // Big slot: structural maximum (every declared link valid).
  int a_big = a_struct < 2 ? 2 : a_struct;
  if (a_big > 32766) a_big = 32766;
  ctx->big = make_layout(V, a_big, N, 0);
  ctx->big_ok = (size_t)ctx->big.bytes <= max_smem;
  if (!ctx->big_ok) {
    // largest arc count that still fits one CTA
    int lo = 2, hi = a_big;
    while (lo < hi) {
      int mid = (lo + hi + 1) / 2;
      if ((size_t)make_layout(V, mid, N, 0).bytes <= max_smem) lo = mid;
      else hi = mid - 1;
    }
    ctx->big = make_layout(V, lo, N, 0);
    ctx->big_ok = (size_t)ctx->big.bytes <= max_smem;
  }
  if ((size_t)ctx->small.bytes * ctx->small_warps > max_smem)
    return fail(ctx, HELIO_ERR_TOO_LARGE, "cluster too large: one graph slot exceeds shared memory");
  // occupancy of both instantiations (PARITY / SCORE)
  void* fns[2] = {reinterpret_cast<void*>(score_kernel<HELIO_MODE_PARITY>),
                  reinterpret_cast<void*>(score_kernel<HELIO_MODE_SCORE>)};
  for (int m = 0; m < 2; ++m) {
    CK(cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[m], 32 * ctx->small_warps,
                                                     ctx->small.bytes * ctx->small_warps));
    if (per_sm < 1) per_sm = 1;
    ctx->small_blocks[m] = per_sm * ctx->sm_count;
    int per_sm_big = 1;
    if (ctx->big_ok) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_big, fns[m], 32, ctx->big.bytes));
      if (per_sm_big < 1) per_sm_big = 1;
    }
    ctx->big_blocks[m] = per_sm_big * ctx->sm_count;
  }
  return HELIO_OK;
}

int ensure_ovf(helio_gpu_ctx* ctx, int set, int64_t B) {
  if (ctx->ovf_cap[set] >= B) return HELIO_OK;
  if (ctx->d_ovf[set]) cudaFree(ctx->d_ovf[set]);
  int64_t cap = std::max<int64_t>(B, 1 << 16);
  CK(cudaMalloc(&ctx->d_ovf[set], sizeof(int64_t) * cap));
  ctx->ovf_cap[set] = cap;
  return HELIO_OK;
}

template <int MODE>
void launch_score_mode(helio_gpu_ctx* ctx, int set, const int16_t* d_pl, int64_t B, int partial, double* d_val,
                       int32_t* d_st, cudaStream_t st, FlowOut fo, bool timed) {
  unsigned long long* work = ctx->d_work + 2 * set;
  unsigned int* oc = ctx->d_ovf_count + set;
  if (timed) cudaEventRecord(ctx->ev0, st);
  const int grid = (int)std::min<int64_t>(ctx->small_blocks[MODE], (B + ctx->small_warps - 1) / ctx->small_warps);
  score_kernel<MODE><<<grid, 32 * ctx->small_warps, ctx->small.bytes * ctx->small_warps, st>>>(
      ctx->cd, ctx->small, d_pl, B, partial, d_val, d_st, work, ctx->d_ovf[set], oc, 0, fo);
  if (timed) cudaEventRecord(ctx->ev1, st);
  // graphs that overflowed the small slot: same kernel, one warp per CTA, big slot
  const Layout& bl = ctx->big_ok ? ctx->big : ctx->small;
  score_kernel<MODE><<<ctx->big_blocks[MODE], 32, bl.bytes, st>>>(ctx->cd, bl, d_pl, B, partial, d_val, d_st,
                                                                   work + 1, ctx->d_ovf[set], oc, 1, fo);
}

int launch_score(helio_gpu_ctx* ctx, int set, const int16_t* d_pl, int64_t B, int partial,
                 double* d_val, int32_t* d_st, cudaStream_t st, FlowOut fo, bool timed, int mode) {
  if (B <= 0) return HELIO_OK;
  int rc = ensure_ovf(ctx, set, B);
  if (rc) return rc;
  CK(cudaMemsetAsync(ctx->d_work + 2 * set, 0, 2 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(ctx->d_ovf_count + set, 0, sizeof(unsigned int), st));
  if (mode == HELIO_MODE_SCORE && fo.edges == nullptr)
    launch_score_mode<HELIO_MODE_SCORE>(ctx, set, d_pl, B, partial, d_val, d_st, st, fo, timed);
  else
    launch_score_mode<HELIO_MODE_PARITY>(ctx, set, d_pl, B, partial, d_val, d_st, st, fo, timed);
  CK(cudaGetLastError());
  ctx->launches += 2;
  if (timed) ctx->timed = true;
  return HELIO_OK;
}

}  // namespace

// PARITY scoring of device rows on `st` (used by search.cu).
int helio_engine_score_parity(helio_gpu_ctx* ctx, const int16_t* d_pl, int64_t B, int partial, double* d_val,
                              int32_t* d_st, cudaStream_t st) {
  FlowOut fo{nullptr, nullptr, nullptr, 0};
  return launch_score(ctx, 0, d_pl, B, partial, d_val, d_st, st, fo, false, HELIO_MODE_PARITY);
}

namespace {

int ensure_stage(helio_gpu_ctx* ctx, int64_t chunk) {
  if (ctx->stage_cap >= chunk) return HELIO_OK;
  for (int i = 0; i < 2; ++i) {
    if (ctx->d_pl[i]) cudaFree(ctx->d_pl[i]);
    if (ctx->d_val[i]) cudaFree(ctx->d_val[i]);
    if (ctx->d_st[i]) cudaFree(ctx->d_st[i]);
    if (ctx->h_pl_pin[i]) cudaFreeHost(ctx->h_pl_pin[i]);
    if (ctx->h_val_pin[i]) cudaFreeHost(ctx->h_val_pin[i]);
    if (ctx->h_st_pin[i]) cudaFreeHost(ctx->h_st_pin[i]);
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

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

}  // namespace

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
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
      cudaMalloc(&ctx->d_work, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&ctx->d_ovf_count, 2 * sizeof(unsigned int)) != cudaSuccess ||
      cudaMalloc(&ctx->d_pv, 3 * 4096 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ctx->d_pi, 3 * 4096 * sizeof(long long)) != cudaSuccess ||
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
  for (int i = 0; i < 2; ++i) {
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
    cudaFree(ctx->d_ovf[i]);
  }
  cudaFree(ctx->d_cluster);
  cudaFree(ctx->d_kmax32);
  cudaFree(ctx->d_work);
  cudaFree(ctx->d_ovf_count);
  cudaFree(ctx->d_pv);
  cudaFree(ctx->d_pi);
  cudaFree(ctx->d_best);
  cudaFree(ctx->d_bidx);
  cudaFree(ctx->d_route);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* helio_gpu_last_error(const helio_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int helio_gpu_sync(helio_gpu_ctx* ctx) {
  if (!ctx) return HELIO_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaStreamSynchronize(ctx->pipe[0]));
  CK(cudaStreamSynchronize(ctx->pipe[1]));
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
  if (mode != HELIO_MODE_PARITY && mode != HELIO_MODE_SCORE) return fail(ctx, HELIO_ERR_INVALID, "unknown mode");
  ctx->mode = mode;
  return HELIO_OK;
}

int helio_gpu_get_mode(const helio_gpu_ctx* ctx) { return ctx ? ctx->mode : -1; }

int helio_gpu_compute_edge_capacity(const helio_gpu_ctx* ctx, int32_t node, int32_t j, double* out) {
  if (!ctx || !ctx->has_cluster || !out) return HELIO_ERR_NO_CLUSTER;
  if (node < 0 || node >= ctx->N || j < 1 || j > ctx->h_kmax[node]) return HELIO_ERR_INVALID;
  *out = ctx->h_cap_tab[ctx->h_cap_off[node] + j - 1];
  return HELIO_OK;
}

int helio_gpu_score(helio_gpu_ctx* ctx, const int16_t* d_pl, int64_t B, int allow_partial,
                    double* d_values, int32_t* d_status, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (B < 0 || (B > 0 && (!d_pl || !d_values || !d_status))) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  FlowOut fo{nullptr, nullptr, nullptr, 0};
  return launch_score(ctx, 0, d_pl, B, allow_partial ? 1 : 0, d_values, d_status, st, fo, true, ctx->mode);
}

}  // extern "C"

namespace {
int argmax_on(helio_gpu_ctx* ctx, int scratch, const double* d_values, const int32_t* d_status, int64_t B,
              int64_t index_base, double* d_best, int64_t* d_index, cudaStream_t st);

// Host-buffer scoring, pipelined over two streams in chunks: H2D of chunk c+1
// and D2H of chunk c-1 overlap the kernels of chunk c.  With pinned caller
// buffers everything is enqueued up front (no host waits until the end);
// pageable buffers go through pinned staging.  Optionally reduces the first
// maximum on the device per chunk (best/index).
int score_host_impl(helio_gpu_ctx* ctx, const int16_t* h_pl, int64_t B, int allow_partial, double* h_values,
                    int32_t* h_status, double* h_best, int64_t* h_index) {
  if (!ctx) return HELIO_ERR_INVALID;
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (B < 0 || (B > 0 && (!h_pl || (!h_values) != (!h_status) || (!h_values && !h_best))))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (B == 0) {
    if (h_best) *h_best = 0.0;
    if (h_index) *h_index = -1;
    return HELIO_OK;
  }
  CK(cudaSetDevice(ctx->device));
  const int64_t chunk = std::min<int64_t>(B, 1 << 18);
  const int64_t nchunks = (B + chunk - 1) / chunk;
  if (h_best && nchunks > 2 * 4096) return fail(ctx, HELIO_ERR_TOO_LARGE, "batch too large for the best reduction");
  int rc = ensure_stage(ctx, chunk);
  if (rc) return rc;
  const bool pin_in = is_pinned(h_pl);
  const bool want_vals = h_values != nullptr;
  const bool pin_out = want_vals && is_pinned(h_values) && is_pinned(h_status);
  const size_t row = sizeof(int16_t) * 2 * ctx->N;
  FlowOut fo{nullptr, nullptr, nullptr, 0};
  for (int64_t c = 0; c < nchunks; ++c) {
    const int s = (int)(c & 1);
    cudaStream_t st = ctx->pipe[s];
    const int64_t lo = c * chunk, n = std::min(chunk, B - lo);
    if (c >= 2 && (!pin_in || (want_vals && !pin_out))) {
      // staging buffers of chunk c-2 are reused: retire it first
      CK(cudaStreamSynchronize(st));
      if (want_vals && !pin_out) {
        const int64_t plo = (c - 2) * chunk, pn = std::min(chunk, B - plo);
        std::memcpy(h_values + plo, ctx->h_val_pin[s], sizeof(double) * pn);
        std::memcpy(h_status + plo, ctx->h_st_pin[s], sizeof(int32_t) * pn);
      }
    }
    const void* src = h_pl + lo * 2 * ctx->N;
    if (!pin_in) {
      std::memcpy(ctx->h_pl_pin[s], src, row * n);
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
  const int64_t first_tail = (pin_in && (!want_vals || pin_out)) ? 0 : std::max<int64_t>(0, nchunks - 2);
  for (int64_t c = first_tail; c < nchunks; ++c) {
    const int s = (int)(c & 1);
    CK(cudaStreamSynchronize(ctx->pipe[s]));
    if (want_vals && !pin_out) {
      const int64_t lo = c * chunk, n = std::min(chunk, B - lo);
      std::memcpy(h_values + lo, ctx->h_val_pin[s], sizeof(double) * n);
      std::memcpy(h_status + lo, ctx->h_st_pin[s], sizeof(int32_t) * n);
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
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (K <= 0) return HELIO_OK;
  if (!h_pl || !h_nv || !h_ne || !h_values || !h_status || max_edges < 0 || (max_edges > 0 && !h_edges))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t row = sizeof(int16_t) * 2 * ctx->N;
  int16_t* d_pl = nullptr;
  double* d_val = nullptr;
  int32_t *d_st = nullptr, *d_nv = nullptr, *d_ne = nullptr;
  helio_edge* d_ed = nullptr;
  int rc = HELIO_OK;
  const size_t edge_bytes = sizeof(helio_edge) * (size_t)K * std::max(max_edges, 1);
  if (cudaMalloc(&d_pl, row * K) != cudaSuccess || cudaMalloc(&d_val, 8 * K) != cudaSuccess ||
      cudaMalloc(&d_st, 4 * K) != cudaSuccess || cudaMalloc(&d_nv, 4 * K) != cudaSuccess ||
      cudaMalloc(&d_ne, 4 * K) != cudaSuccess || cudaMalloc(&d_ed, edge_bytes) != cudaSuccess) {
    rc = fail(ctx, HELIO_ERR_CUDA, "cudaMalloc failed in flows");
  }
  if (!rc && cudaMemcpyAsync(d_pl, h_pl, row * K, cudaMemcpyHostToDevice, st) != cudaSuccess)
    rc = fail(ctx, HELIO_ERR_CUDA, "H2D failed in flows");
  if (!rc) {
    FlowOut fo{d_ed, d_nv, d_ne, max_edges};
    rc = launch_score(ctx, 0, d_pl, K, allow_partial ? 1 : 0, d_val, d_st, st, fo, false, HELIO_MODE_PARITY);
  }
  if (!rc) {
    bool ok = cudaMemcpyAsync(h_values, d_val, 8 * K, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
              cudaMemcpyAsync(h_status, d_st, 4 * K, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
              cudaMemcpyAsync(h_nv, d_nv, 4 * K, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
              cudaMemcpyAsync(h_ne, d_ne, 4 * K, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
              (max_edges == 0 || cudaMemcpyAsync(h_edges, d_ed, sizeof(helio_edge) * (size_t)K * max_edges,
                                                 cudaMemcpyDeviceToHost, st) == cudaSuccess) &&
              cudaStreamSynchronize(st) == cudaSuccess;
    if (!ok) rc = fail(ctx, HELIO_ERR_CUDA, std::string("flows: ") + cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(d_pl); cudaFree(d_val); cudaFree(d_st); cudaFree(d_nv); cudaFree(d_ne); cudaFree(d_ed);
  return rc;
}

int helio_gpu_maxflow_raw_host(helio_gpu_ctx* ctx, int64_t G, const int32_t* h_n, const int32_t* h_s,
                               const int32_t* h_t, const int64_t* h_off, const int32_t* h_u,
                               const int32_t* h_v, const double* h_cap, double* h_values,
                               double* h_flows) {
  if (!ctx) return HELIO_ERR_INVALID;
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
  if ((size_t)lay.bytes > max_smem)
    return fail(ctx, HELIO_ERR_TOO_LARGE, "raw graph does not fit one SM's shared memory");
  int warps = (int)std::max<size_t>(1, std::min<size_t>(4, max_smem / lay.bytes));
  CK(cudaFuncSetAttribute(raw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raw_kernel, 32 * warps, lay.bytes * warps));
  if (per_sm < 1) per_sm = 1;
  cudaStream_t st = ctx->stream;
  int32_t *d_n, *d_s, *d_t, *d_u = nullptr, *d_v = nullptr;
  int64_t* d_off;
  double *d_cap = nullptr, *d_val, *d_fl = nullptr;
  const int64_t Ea = std::max<int64_t>(Etot, 1);
  CK(cudaMalloc(&d_n, 4 * G));
  CK(cudaMalloc(&d_s, 4 * G));
  CK(cudaMalloc(&d_t, 4 * G));
  CK(cudaMalloc(&d_off, 8 * (G + 1)));
  CK(cudaMalloc(&d_u, 4 * Ea));
  CK(cudaMalloc(&d_v, 4 * Ea));
  CK(cudaMalloc(&d_cap, 8 * Ea));
  CK(cudaMalloc(&d_val, 8 * G));
  if (h_flows) CK(cudaMalloc(&d_fl, 8 * Ea));
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
  int grid = (int)std::min<int64_t>((int64_t)per_sm * ctx->sm_count, (G + warps - 1) / warps);
  raw_kernel<<<grid, 32 * warps, lay.bytes * warps, st>>>(lay, G, d_n, d_s, d_t, d_off, d_u, d_v, d_cap,
                                                           d_val, d_fl, ctx->d_work);
  CK(cudaGetLastError());
  ctx->launches++;
  CK(cudaMemcpyAsync(h_values, d_val, 8 * G, cudaMemcpyDeviceToHost, st));
  if (h_flows && Etot > 0) CK(cudaMemcpyAsync(h_flows, d_fl, 8 * Etot, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(d_n); cudaFree(d_s); cudaFree(d_t); cudaFree(d_off); cudaFree(d_u); cudaFree(d_v);
  cudaFree(d_cap); cudaFree(d_val); cudaFree(d_fl);
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

extern "C" {

int helio_gpu_argmax(helio_gpu_ctx* ctx, const double* d_values, const int32_t* d_status, int64_t B,
                     int64_t index_base, double* d_best, int64_t* d_index, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  if (!d_best || !d_index || (B > 0 && (!d_values || !d_status))) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return argmax_on(ctx, 2, d_values, d_status, B, index_base, d_best, d_index, st);
}

int helio_gpu_generate(helio_gpu_ctx* ctx, uint64_t seed, int64_t first, int64_t B, uint32_t ppm,
                       int16_t* d_out, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
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
  if (!ctx || !ctx->has_cluster || (B > 0 && !h_out)) return HELIO_ERR_INVALID;
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
