// solve_parity.cuh — K2 PARITY: bit-exact replay of the reference's FIFO
// preflow-push, plus the value / per-edge-flow read-out.
#pragma once

namespace {

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

// ---------------------------------------------------------------------------
// PARITY solver (the replay argued above), with little bookkeeping per step: per-vertex state in one 16-byte VState (one LDS.128 per pop, one
// STS.128 per write-back), the in-queue set in registers when n <= 128
// (every lane holds the same two 64-bit words, so the enqueue test is a
// uniform register test), and a failed scan of the last arc chunk falls
// straight into the relabel instead of taking another loop trip.
// HELIO_BOUNDS (diagnostic builds only): trap on an out-of-range slot index.
#ifdef HELIO_BOUNDS
#define HB_CHECK(idx, lim, tag)                                                                    \
  do {                                                                                             \
    if ((unsigned)(idx) >= (unsigned)(lim)) {                                                      \
      printf("HELIO_BOUNDS %s idx=%d lim=%d block=%d lane=%d\n", tag, (int)(idx), (int)(lim),       \
             (int)blockIdx.x, (int)(threadIdx.x & 31));                                            \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
#else
#define HB_CHECK(idx, lim, tag) \
  do {                          \
  } while (0)
#endif

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
#ifdef HELIO_BOUNDS
  for (int x = lane; x < n; x += 32) g.q[x] = -7;  // sentinel: a slot read before any write shows -7
#endif
  __syncwarp();
  if (lane == 0) {
    g.cnt[0] = (int16_t)(n - 1);
    g.cnt[n] += 1;
  }
  // In-queue flags and the queue array are written by lane 0 only, and the
  // flag is tested by all lanes between two warp barriers.  (Round 1 let
  // every lane test and set the flag itself; under independent thread
  // scheduling the "uniform" code after a divergent push can run at different
  // times in different lanes, so one lane could see another's fresh flag and
  // skip an enqueue the others counted — the queue then read a slot lane 0
  // never wrote.  Found with the HELIO_BOUNDS diagnostic build.)
  int tail = 0, qcount = 0;
#if !defined(HELIO_ENQ_SHFL)
  // every lane tests the flag between two warp barriers (so all lanes see the
  // same state), lane 0 alone sets it and stores the entry
  auto enqueue = [&](int x) {
    __syncwarp();
    const bool fresh = x != s && x != t && !g.inq[x];
    __syncwarp();
    if (fresh) {
      if (lane == 0) {
        g.inq[x] = 1;
        g.q[tail] = (int16_t)x;
      }
      tail = tail + 1 == n ? 0 : tail + 1;
      ++qcount;
    }
  };
#else
  auto enqueue = [&](int x) {
    int fresh = 0;
    if (lane == 0 && x != s && x != t && !g.inq[x]) {
      g.inq[x] = 1;
      g.q[tail] = (int16_t)x;
      fresh = 1;
    }
    if (__shfl_sync(FULL, fresh, 0)) {
      tail = tail + 1 == n ? 0 : tail + 1;
      ++qcount;
    }
  };
#endif
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
        enqueue(to);
      }
    }
  }
  int head = 0;
  const int two_n = 2 * n;
  while (qcount > 0) {
    __syncwarp();
    const int u = g.q[head];
#ifdef HELIO_BOUNDS
    if ((unsigned)u >= (unsigned)n) {
      printf("HELIO_BOUNDS queue vertex u=%d n=%d head=%d tail=%d qcount=%d deg_b=%d q[h-1]=%d q[h+1]=%d\n", u, n,
             head, tail, qcount, (int)g.abeg[n], (int)g.q[head ? head - 1 : n - 1], (int)g.q[head + 1 < n ? head + 1 : 0]);
      __trap();
    }
#endif
    head = head + 1 == n ? 0 : head + 1;
    --qcount;
    const VState su = vs[u];
    double ex = su.ex;
    int hu = su.h;
    int cu = su.cur;
    const int b = su.b;
    const int deg = su.deg;
    if (lane == 0) g.inq[u] = 0;
    if (deg <= 32) {
      // Single-chunk fast path (almost every vertex): lane j holds arc b + j for
      // the whole discharge.  A failed ballot means the scan reached the end of
      // the list, i.e. the reference's relabel (:180).
      const bool inr = lane < deg;
      double ca = 0.0;
      int ta = 0, ra = 0, hp1 = 0;  // hp1 = height[to] + 1
      if (inr) {
        const int a = b + lane;
        ca = g.cap[a];
        ta = g.to[a];
        ra = g.rv[a];
        HB_CHECK(ta, n, "fast arc head");
        hp1 = vs[ta].h + 1;
      }
      bool live = inr && ca > FLOW_EPS;  // residual arc: changes only when this lane pushes
      while (ex > FLOW_EPS) {
        const bool adm = live && lane >= cu && hu == hp1;
        const unsigned m = __ballot_sync(FULL, adm);
        if (m != 0u) {
          const int j = __ffs(m) - 1;
          cu = j;
          const double cj = __shfl_sync(FULL, ca, j);
          const int tj = __shfl_sync(FULL, ta, j);
          const double amt = ref_min(ex, cj);  // push (:156-166)
          if (lane == j) {
            ca -= amt;
            live = ca > FLOW_EPS;
            g.cap[b + j] = ca;
            g.cap[ra] += amt;
          }
          HB_CHECK(tj, n, "fast push target");
          if (lane == 0) vs[tj].ex += amt;
          ex -= amt;
          enqueue(tj);
          continue;
        }
        // relabel (:180-199)
        const int old = hu;
        const int best = __reduce_min_sync(FULL, live ? hp1 : two_n);
        HB_CHECK(best, two_n + 1, "fast best");
        HB_CHECK(old, two_n + 1, "fast old");
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
          if (inr) hp1 = vs[ta].h + 1;
        }
        if (inr && ta == u) hp1 = hu + 1;  // self-loop arcs see u's new height
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
      continue;
    }
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
          enqueue(tj);
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
  // link_pack a few batches ahead: one warp scans every link, and each
  // batch's evaluation would otherwise wait on its own global load
  constexpr int kAhead = 2;
  uint32_t ahead[kAhead];
#pragma unroll
  for (int q = 0; q < kAhead; ++q) ahead[q] = 32 * q + lane < cd.Mv ? __ldg(cd.link_pack + 32 * q + lane) : 0u;
  for (int l0 = 0; l0 < cd.Mv; l0 += 32) {
    const int l = l0 + lane;
    uint32_t pk = ahead[0];
#pragma unroll
    for (int q = 0; q + 1 < kAhead; ++q) ahead[q] = ahead[q + 1];
    {
      const int ln = l + 32 * kAhead;
      ahead[kAhead - 1] = ln < cd.Mv ? __ldg(cd.link_pack + ln) : 0u;
    }
    LinkEval le{false, 0, 0};
    if (l < cd.Mv) le = eval_link_pk(cd, g, pk, partial);
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
}  // namespace
