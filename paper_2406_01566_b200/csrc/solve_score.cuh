// solve_score.cuh — K2 SCORE: value-only Edmonds-Karp solvers.
#pragma once

namespace {

// ---------------------------------------------------------------------------
// SCORE mode: value-only Edmonds-Karp (shortest augmenting paths), one warp
// per graph — see solve_ek_batched below.  Exact on integer capacities (every
// intermediate is an integer-valued double); on float capacities the value
// differs from the reference's FIFO preflow-push only by rounding (north_star
// tolerance 1e-6 relative; tests assert it).  Slot reuse: h = BFS parent arc,
// q = BFS queue, ex = bottleneck capacity from the source.

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

// ---------------------------------------------------------------------------
// SCORE solver for n > 128 (deep sparse networks such as syn256's link walks,
// ~500 vertices, ~40 augmenting paths of ~60 arcs each): synchronous
// push-relabel, preflow phase only, with periodic global relabels.  The
// preflow phase ends with a minimum cut and the sink's excess equals the
// max-flow value, so the excess-return phase is never run.
//
// Batches: live vertices with excess (height < n, not s/t) wait in a FIFO
// (each at most once); a batch pops up to 32 of them, one lane each.  Push rounds: every lane pushes along
// its next admissible arc (h[u] == h[v] + 1, residual > eps, current-arc
// order).  Lanes whose target another lower lane also pushes to this round
// wait one round, so every vertex receives at most one deposit per round and
// no FP addition order depends on timing; pushes into the sink accumulate in
// the pushing lane's register and are reduced at the end; receivers join the
// FIFO tail in lane order.  Then every batch vertex with excess left relabels to 1 + min height over its residual arcs
// (capped at n = dead: it cannot reach the sink) and rejoins the FIFO.
// Every gr_every batches a global relabel runs: backward
// BFS from the sink over residual arcs (warp-cooperative, arc-parallel over
// the queue, lowest lane wins = exact BFS distances); unreached vertices get
// n.  Everything is deterministic; on integer capacities every intermediate
// is an integer-valued double, so the value is exact.
// Global relabel: exact BFS distances to t over residual arcs into h.  The
// BFS stops as soon as every live vertex holding excess is labelled: at that
// point every vertex at distance <= hd (the level of the queue head) is
// labelled, so hd + 1 is a valid (lower-bound) label for the rest.  Dead
// vertices (h >= n: distance >= n, i.e. unreachable) stay dead; anything the
// exhausted BFS never reached becomes dead.  q: n-entry queue scratch.
__device__ void pr_global_relabel(const Gs& g, int16_t* q, const int n, const int s, const int t, const int lane) {
  const unsigned lt = lanemask_lt();
  const unsigned le = lt | (1u << lane);
  int need = 0;
  for (int x = lane; x < n; x += 32) {
    const int hx = g.h[x];
    const bool dead = x == s || hx >= n;
    if (!dead && x != t && g.ex[x] > 0.0) ++need;
    g.h[x] = (int16_t)(dead ? n : -1);
  }
  need = __reduce_add_sync(FULL, need);
  __syncwarp();
  if (lane == 0) {
    g.h[t] = 0;
    q[0] = (int16_t)t;
  }
  __syncwarp();
  // the queue's arcs form one stream; each step gives lane j stream arc j.
  // off = arcs of q[qh] already scanned (a vertex with > 32 arcs spans steps)
  int qh = 0, qt = 1, off = 0;
  while (qh < qt) {
    const int avail = min(32, qt - qh);
    int vi = 0, bi = 0, di = 0;
    if (lane < avail) {
      vi = q[qh + lane];
      bi = g.abeg[vi];
      di = g.abeg[vi + 1] - bi;
      if (lane == 0) {
        bi += off;
        di -= off;
      }
    }
    int incl = di;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int start = incl - di;
    const unsigned sm = __reduce_or_sync(FULL, (lane < avail && di > 0 && start < 32) ? (1u << start) : 0u);
    const int total = min(32, __shfl_sync(FULL, incl, avail - 1));
    const int slot = __popc(sm & le) - 1;
    const int su = slot < 0 ? 0 : slot;
    const int u_b = __shfl_sync(FULL, bi, su);
    const int u_st = __shfl_sync(FULL, start, su);
    const int u_v = __shfl_sync(FULL, vi, su);
    const int kfull = __popc(__ballot_sync(FULL, lane < avail && incl <= 32));
    const int p_st = __shfl_sync(FULL, start, kfull & 31);
    bool ok = false;
    int x = 0;
    if (lane < total) {
      const int a = u_b + (lane - u_st);
      x = g.to[a];
      // arc x -> u_v is residual (the reverse of a); x not yet labelled
      ok = g.h[x] == -1 && g.cap[g.rv[a]] > FLOW_EPS;
    }
    const unsigned cand = __ballot_sync(FULL, ok);
    if (ok) ok = (__match_any_sync(cand, x) & lt) == 0u;
    const unsigned m = __ballot_sync(FULL, ok);
    if (ok) {
      g.h[x] = (int16_t)(g.h[u_v] + 1);
      q[qt + __popc(m & lt)] = (int16_t)x;
    }
    qt += __popc(m);
    need -= __popc(__ballot_sync(FULL, ok && g.ex[x] > 0.0));
    if (kfull < avail) {  // q[qh + kfull] continues into the next step
      off = (kfull == 0 ? off : 0) + (32 - p_st);
    } else {
      off = 0;
    }
    qh += kfull;
    __syncwarp();
    if (need == 0 && qh < qt) break;
  }
  const int rest = qh < qt ? g.h[q[qh]] + 1 : n;
  for (int x = lane; x < n; x += 32)
    if (g.h[x] == -1) g.h[x] = (int16_t)rest;
  __syncwarp();
}

// ILP (the dedicated large-graph kernel): the admissible-arc scan and the
// relabel take four arcs per step (independent loads); otherwise one arc per
// step — the code the combined small-cluster kernel is register-tuned with.
template <bool ILP>
__device__ double solve_pr(const Gs& g, const int n, const int s, const int t, const int lane, const int gr_every) {
  const unsigned lt = lanemask_lt();
  int16_t* fq = g.q;     // circular FIFO of live vertices with excess (<= n entries)
  uint8_t* inq = g.inq;  // FIFO membership
  int16_t* bq = g.cur;   // global-relabel queue
  for (int x = lane; x < n; x += 32) {
    g.ex[x] = 0.0;
    g.h[x] = 0;  // live until the first global relabel
    inq[x] = 0;
  }
  __syncwarp();
  int head = 0, cnt = 0;
  if (lane == 0) {  // saturate the source's arcs in adjacency order
    for (int a = g.abeg[s], e = g.abeg[s + 1]; a < e; ++a) {
      const double c = g.cap[a];
      if (c > 0.0) {
        const int v = g.to[a];
        g.cap[a] = 0.0;
        g.cap[g.rv[a]] += c;
        g.ex[v] += c;
        if (v != t && v != s && !inq[v]) {
          inq[v] = 1;
          fq[cnt++] = (int16_t)v;
        }
      }
    }
  }
  cnt = __shfl_sync(FULL, cnt, 0);
  __syncwarp();
  double sink = 0.0;  // this lane's pushes into t
  int since = gr_every;
  while (cnt > 0) {
    if (since >= gr_every) {
      pr_global_relabel(g, bq, n, s, t, lane);
      since = 0;
    }
    ++since;
    // pop up to 32 (FIFO order); entries that died since they were queued drop out
    const int take = min(32, cnt);
    int u = -1, a = 0, ae = 0, hu = 0;
    if (lane < take) {
      int p = head + lane;
      if (p >= n) p -= n;
      u = fq[p];
      inq[u] = 0;
      hu = g.h[u];
      if (hu < n && g.ex[u] > 0.0) {
        a = g.abeg[u];
        ae = g.abeg[u + 1];
      } else {
        u = -1;
      }
    }
    head += take;
    if (head >= n) head -= n;
    cnt -= take;
    int tail = head + cnt;
    if (tail >= n) tail -= n;
    __syncwarp();
    for (;;) {
      double e = 0.0, c = 0.0;
      int v = -1, r = -1;  // ILP: r = the chosen arc's reverse, loaded with the scan
      if (u >= 0) {
        e = g.ex[u];
        if (e > 0.0 && !ILP) {
          for (; a < ae; ++a) {
            const int w = g.to[a];
            if (g.h[w] == hu - 1) {
              c = g.cap[a];
              if (c > FLOW_EPS) {
                v = w;
                break;
              }
            }
          }
        } else if (e > 0.0) {
          // the first admissible arc at or after `a`, four arcs per step:
          // their loads are independent, so one step costs two shared-memory
          // round trips instead of two per arc
          const int hw = hu - 1;
          while (a < ae) {
            const int n4 = min(4, ae - a);
            int w[4], hh[4];
            double cc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              w[k] = k < n4 ? g.to[a + k] : 0;
              cc[k] = k < n4 ? g.cap[a + k] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) hh[k] = k < n4 ? g.h[w[k]] : -2;
            int rr[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) rr[k] = k < n4 ? g.rv[a + k] : 0;
            int kk = -1, vk = -1, rk = -1;
            double ck = 0.0;
#pragma unroll
            for (int k = 3; k >= 0; --k)
              if (hh[k] == hw && cc[k] > FLOW_EPS) {
                kk = k;
                vk = w[k];
                ck = cc[k];
                rk = rr[k];
              }
            if (kk >= 0) {
              a += kk;
              v = vk;
              c = ck;
              r = rk;
              break;
            }
            a += n4;
          }
        }
      }
      // ILP: the reverse arc's residual and the target's queue flag are read
      // before the ballots — within a round only this lane touches that arc
      // (lowest lane per target; v cannot push back along it, h[v] < h[u]),
      // and only the lane depositing into v appends it
      double rc = 0.0;
      bool vq = false;
      if (ILP && v >= 0) {
        rc = g.cap[r];
        vq = v != t && inq[v];
      }
      const unsigned pm = __ballot_sync(FULL, v >= 0);
      if (pm == 0u) break;
      const unsigned nm = __ballot_sync(FULL, v >= 0 && v != t);
      bool go = v >= 0;
      if (v >= 0 && v != t) go = (__match_any_sync(nm, v) & lt) == 0u;  // lowest lane per target
      double d = 0.0;
      if (go) {
        d = ref_min(e, c);
        g.cap[a] = c - d;
        if (ILP)
          g.cap[r] = rc + d;
        else
          g.cap[g.rv[a]] += d;
        g.ex[u] = e - d;
        if (v == t) sink += d;
        if (d == c) ++a;  // saturated (else u is drained)
      }
      __syncwarp();
      const bool app = go && v != t && (ILP ? !vq : !inq[v]);
      if (go && v != t) g.ex[v] += d;
      const unsigned am = __ballot_sync(FULL, app);
      if (app) {
        int p = tail + __popc(am & lt);
        if (p >= n) p -= n;
        fq[p] = (int16_t)v;
        inq[v] = 1;
      }
      tail += __popc(am);
      if (tail >= n) tail -= n;
      cnt += __popc(am);
      __syncwarp();
    }
    // relabel what still has excess: every arc was scanned, none admissible
    int nl = -1;
    if (u >= 0 && g.ex[u] > 0.0) {
      int best = n;
      if (!ILP) {
        for (int b2 = g.abeg[u]; b2 < ae; ++b2)
          if (g.cap[b2] > FLOW_EPS) best = min(best, g.h[g.to[b2]] + 1);
      } else {
      for (int b2 = g.abeg[u]; b2 < ae; b2 += 4) {  // four independent arcs per step
        const int n4 = min(4, ae - b2);
        int w[4];
        double cc[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          w[k] = k < n4 ? g.to[b2 + k] : 0;
          cc[k] = k < n4 ? g.cap[b2 + k] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (cc[k] > FLOW_EPS) best = min(best, g.h[w[k]] + 1);
      }
      }
      nl = best;
    }
    __syncwarp();
    const bool app = nl >= 0 && nl < n && !inq[u];
    if (nl >= 0) g.h[u] = (int16_t)nl;
    const unsigned am = __ballot_sync(FULL, app);
    if (app) {
      int p = tail + __popc(am & lt);
      if (p >= n) p -= n;
      fq[p] = (int16_t)u;
      inq[u] = 1;
    }
    cnt += __popc(am);
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sink += __shfl_xor_sync(FULL, sink, o);
  return g.ex[t] + sink;
}

// SCORE solver for n <= 128: Edmonds-Karp with a level-synchronous bitset
// BFS.  Vertex sets are four 32-bit words (vertex v = bit v & 31 of word
// v >> 5), so lane l owns vertices l, l+32, l+64, l+96 and its bit in every
// word is simply bit l.  R[v] (shared memory) is the set of residual
// out-neighbours of v, kept exact by the augmentations.
//
// Pair closure: in this numbering a node's two vertices are v and v^1 (in =
// 2+2k, out = 3+2k), joined by its compute arc.  When a level reaches one
// half of a node whose pair arc has residual capacity, the other half joins
// the same level, so the BFS walks nodes rather than split vertices and needs
// about half the levels.  It is folded into each lane's rows once per
// augmentation: Q[v] = R[v] | swap(R[v] & P), P = vertices whose pair arc has
// residual capacity.  A level is then: OR the Q rows of owned frontier
// vertices, four REDUX.OR, mask with the visited set.
//
// Path recovery: a vertex at level d takes the first arc (adjacency order)
// from a level d-1 vertex with residual capacity; a vertex without one was
// added through its partner's pair arc.  Paths are valid augmenting paths,
// chosen deterministically.
__device__ __forceinline__ unsigned swap_pairs32(unsigned x) {
  return ((x & 0x55555555u) << 1) | ((x >> 1) & 0x55555555u);
}

// NW = 32-bit words per vertex set = ceil(n / 32): lane l owns vertices l + 32i
// for i < NW, so every loop below is unrolled to exactly the words in use.
template <int NW>
__device__ double solve_ek_bits_w(const Gs& g, const int n, const int s, const int t, const int lane,
                                  const double cut) {
  // R in the VState region; BFS level per vertex (int8, n <= 128 levels) in
  // the in-queue bytes; parent arc | parent vertex << 16 per vertex in the
  // count region (4V + 2 bytes); the augmenting path in the queue region.
  uint4* R = reinterpret_cast<uint4*>(g.vs);
  int8_t* dist = reinterpret_cast<int8_t*>(g.inq);
  int32_t* par = reinterpret_cast<int32_t*>(g.cnt);
  int16_t* path = g.q;
  const unsigned lb = 1u << lane;
  for (int x = lane; x < n; x += 32) {
    unsigned r[4] = {0u, 0u, 0u, 0u};
    for (int a = g.abeg[x], e = g.abeg[x + 1]; a < e; ++a)
      if (g.cap[a] > FLOW_EPS) {
        const int y = g.to[a];
        r[y >> 5] |= 1u << (y & 31);
      }
    R[x] = make_uint4(r[0], r[1], r[2], r[3]);
  }
  __syncwarp();
  double value = 0.0;
  for (;;) {
    // P: vertices v >= 2 whose pair arc v -> v^1 has residual capacity (v^1
    // is bit lane^1 of v's own word); then this lane's closure rows Q
    unsigned Q[NW][NW];
    unsigned P[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const int v = lane + 32 * i;
      bool pr = false;
#pragma unroll
      for (int w = 0; w < NW; ++w) Q[i][w] = 0u;
      if (v < n) {
        const uint4 r = R[v];
        const unsigned rw[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int w = 0; w < NW; ++w) Q[i][w] = rw[w];
        pr = v >= 2 && ((Q[i][i] >> (lane ^ 1)) & 1u);
      }
      P[i] = __ballot_sync(FULL, pr);
    }
#pragma unroll
    for (int i = 0; i < NW; ++i)
#pragma unroll
      for (int w = 0; w < NW; ++w) Q[i][w] |= swap_pairs32(Q[i][w] & P[w]);
    // BFS levels from s
    unsigned F[NW], Vs[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      F[w] = (s >> 5) == w ? 1u << (s & 31) : 0u;
      Vs[w] = F[w];
    }
    int dl[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) dl[i] = (lane + 32 * i == s) ? 0 : -1;
    int d = 0;
    bool found = false;
    for (;;) {
      unsigned a[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) a[w] = 0u;
#pragma unroll
      for (int i = 0; i < NW; ++i)
        if (F[i] & lb)
#pragma unroll
          for (int w = 0; w < NW; ++w) a[w] |= Q[i][w];
      unsigned any = 0u;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        F[w] = __reduce_or_sync(FULL, a[w]) & ~Vs[w];
        any |= F[w];
      }
      if (any == 0u) break;
      ++d;
#pragma unroll
      for (int w = 0; w < NW; ++w) Vs[w] |= F[w];
#pragma unroll
      for (int i = 0; i < NW; ++i) dl[i] = (F[i] & lb) ? d : dl[i];
      if ((F[t >> 5] >> (t & 31)) & 1u) {
        found = true;
        break;
      }
    }
    if (!found) break;
#pragma unroll
    for (int i = 0; i < NW; ++i)
      if (lane + 32 * i < n) dist[lane + 32 * i] = (int8_t)dl[i];
    __syncwarp();
    // parent of every visited vertex
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const int x = lane + 32 * i;
      const int dx = dl[i];
      if (x >= n || dx <= 0) continue;
      int pick = -1, pu = -1;
      for (int a = g.abeg[x], e = g.abeg[x + 1]; a < e; ++a) {
        const int u = g.to[a];
        const int r = g.rv[a];
        if (dist[u] == dx - 1 && g.cap[r] > FLOW_EPS) {
          pick = r;
          pu = u;
          break;
        }
      }
      if (pick < 0) {  // reached through its partner's pair arc at the same level
        pick = g.rv[g.abeg[x]];  // the builder puts the compute pair in slot 0
        pu = x ^ 1;
      }
      par[x] = (int32_t)(uint16_t)pick | (pu << 16);
    }
    __syncwarp();
    int len = 0;
    if (lane == 0) {
      int x = t;
      while (x != s) {
        const int32_t w = par[x];
        path[len++] = (int16_t)(w & 0xffff);
        x = w >> 16;
      }
    }
    len = __shfl_sync(FULL, len, 0);
    __syncwarp();
    double f = 1.0e300;
    for (int k = lane; k < len; k += 32) f = ref_min(f, g.cap[path[k]]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f = ref_min(f, __shfl_xor_sync(FULL, f, o));
    unsigned* Rw = reinterpret_cast<unsigned*>(R);
    for (int k = lane; k < len; k += 32) {
      const int a = path[k];
      const int r = g.rv[a];
      const int v = g.to[a];
      const int u = g.to[r];
      const double ca = g.cap[a] - f;
      g.cap[a] = ca;
      g.cap[r] += f;
      if (ca <= FLOW_EPS) atomicAnd(&Rw[4 * u + (v >> 5)], ~(1u << (v & 31)));
      atomicOr(&Rw[4 * v + (u >> 5)], 1u << (u & 31));
    }
    value += f;
    __syncwarp();
    if (value >= cut) break;  // a flow as large as a cut is maximum: skip the proving BFS
  }
  return value;
}

// cut: the capacity of any s-t cut (the builder's layer cut), or +inf
__device__ double solve_ek_bits(const Gs& g, const int n, const int s, const int t, const int lane,
                                const double cut) {
  if (n <= 32) return solve_ek_bits_w<1>(g, n, s, t, lane, cut);
  if (n <= 64) return solve_ek_bits_w<2>(g, n, s, t, lane, cut);
  if (n <= 96) return solve_ek_bits_w<3>(g, n, s, t, lane, cut);
  return solve_ek_bits_w<4>(g, n, s, t, lane, cut);
}

}  // namespace
