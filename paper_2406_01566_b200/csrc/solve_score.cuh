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

}  // namespace
