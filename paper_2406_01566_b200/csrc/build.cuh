// build.cuh — K1: placement row -> the reference's flow network in a warp's
// shared-memory slot (PARITY builders keep the reference's vertex/edge/arc
// order; SCORE builders only its graph).
#pragma once

namespace {

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

__device__ __forceinline__ LinkEval eval_link_pk(const ClusterDev& cd, const Gs& g, uint32_t pk, int partial);
__device__ __forceinline__ LinkEval eval_link(const ClusterDev& cd, const Gs& g, int l, int partial) {
  return eval_link_pk(cd, g, __ldg(cd.link_pack + l), partial);
}
// (pk = link_pack[l], loaded ahead by callers that scan many links)
__device__ __forceinline__ LinkEval eval_link_pk(const ClusterDev& cd, const Gs& g, uint32_t pk, int partial) {
  LinkEval r{false, 0, 0};
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

// Valid out-links of node k (end e): calls f(j, link) for every declared
// link k -> j whose head's interval chains from e (flow_graph.cpp:121), in
// out-list order.  Four links per step: their global and shared loads are
// independent, so a step costs one round trip of each instead of one per link.
template <class F>
__device__ __forceinline__ void for_valid_out_links(const ClusterDev& cd, const int32_t* pse, int k, int e,
                                                    int partial, F&& f) {
  const int pb = __ldg(cd.out_beg + k), pend = __ldg(cd.out_beg + k + 1);
  for (int p = pb; p < pend; p += 4) {
    const int n4 = min(4, pend - p);
    int2 jl[4];
    int32_t iv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) jl[q] = q < n4 ? __ldg(&cd.out_list[p + q]) : make_int2(0, -1);
#pragma unroll
    for (int q = 0; q < 4; ++q) iv[q] = q < n4 ? pse[jl[q].x] : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int sj = (int16_t)(iv[q] & 0xffff), ej = (int16_t)(iv[q] >> 16);
      if (q < n4 && ej > sj && edge_ok(e, sj, ej, partial)) f(jl[q].x, jl[q].y);
    }
  }
}

// SCORE builder for N > 64 (sparse interconnects): per used node, one pass
// over its compiled out-link list.  Intervals are kept packed (start | end <<
// 16, the row's own int32 words) over the ps/pe scratch.
__device__ int build_graph_score(const ClusterDev& cd, const Gs& g, const Layout& lay, const int16_t* row,
                                 int partial, int lane, int& V, int& E) {
  const int N = cd.N, L = cd.L;
  int32_t* pse = reinterpret_cast<int32_t*>(g.ps);  // ps/pe: 4N contiguous bytes, 4-aligned
  int bad = INT_MAX;
  const int32_t* row32 = reinterpret_cast<const int32_t*>(row);
  for (int k = lane; k < N; k += 32) {
    const int32_t w = __ldg(row32 + k);
    const int s = (int16_t)(w & 0xffff);
    const int e = (int16_t)(w >> 16);
    pse[k] = w;
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
  // valid out-links + sink arc.  One pass over the out-lists: a valid link
  // k -> j adds to out_k here and to in_j through a shared atomic.
  int nedges = 0, dsrc = 0, dsink = 0;
  int* fill = reinterpret_cast<int*>(g.ex);  // int counters per vertex during the build
  for (int x = lane; x < V; x += 32) fill[x] = 0;
  __syncwarp();
  for (int k = lane; k < N; k += 32) {
    const int32_t w = pse[k];
    const int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
    if (e <= s) continue;
    int din = 1, dout = 1;
    ++nedges;
    for_valid_out_links(cd, pse, k, e, partial, [&](int j, int) {
      ++dout;
      atomicAdd(&fill[2 + 2 * j], 1);
    });
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
    atomicAdd(&fill[2 + 2 * k], din);
    fill[3 + 2 * k] = dout;  // only this lane touches an out-vertex's count
  }
  nedges = __reduce_add_sync(FULL, nedges);
  dsrc = __reduce_add_sync(FULL, dsrc);
  dsink = __reduce_add_sync(FULL, dsink);
  E = nedges;
  if (2 * E > lay.A) return ST_OVERFLOW;
  if (lane == 0) {
    fill[0] = dsrc;
    fill[1] = dsink;
  }
  __syncwarp();
  // arc ranges; each used node's compute pair takes slot 0 of both its
  // vertices (so the pair arc of x >= 2 is arc abeg[x]), the rest fill in.
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
    if (x < V) {
      g.abeg[x] = (int16_t)(run + incl - d);
      fill[x] = (x >= 2 && d > 0) ? 1 : 0;
    }
    run += __shfl_sync(FULL, incl, 31);
  }
  if (lane == 0) g.abeg[V] = (int16_t)run;
  __syncwarp();
  // arcs: each lane places its node's compute pair and every edge it
  // sources; the paired reverse arc takes the next free slot at its head.
  for (int k = lane; k < N; k += 32) {
    const int32_t w = pse[k];
    const int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
    if (e <= s) continue;
    const int vi = 2 + 2 * k, vo = vi + 1;
    const int ai = g.abeg[vi];
    const int ao = g.abeg[vo];
    g.to[ai] = (int16_t)vo;
    g.rv[ai] = (int16_t)ao;
    g.cap[ai] = __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (e - s) - 1);
    g.to[ao] = (int16_t)vi;
    g.rv[ao] = (int16_t)ai;
    g.cap[ao] = 0.0;
    for_valid_out_links(cd, pse, k, e, partial, [&](int j, int link) {
      const int vj = 2 + 2 * j;
      const int fa = ao + atomicAdd(&fill[vo], 1);
      const int ra = g.abeg[vj] + atomicAdd(&fill[vj], 1);
      g.to[fa] = (int16_t)vj;
      g.rv[fa] = (int16_t)ra;
      g.cap[fa] = __ldg(cd.link_cap + link);
      g.to[ra] = (int16_t)vo;
      g.rv[ra] = (int16_t)fa;
      g.cap[ra] = 0.0;
    });
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

// ---------------------------------------------------------------------------
// SCORE builder for large sparse networks (GEN kernel): the split network with
// every series vertex contracted away.  A vertex other than s, t with exactly
// one in-arc and one out-arc (an in-vertex with one in-edge — its only
// out-edge is the compute edge; an out-vertex with one out-edge) carries the
// same flow on both, so u -> x -> w becomes u -> w with capacity min of the
// two; chains of such vertices collapse into one edge.  The max-flow value is
// unchanged (min is exact), so SCORE's guarantees hold.  On syn256 link walks
// this takes V 514 -> ~248 and E 699 -> ~433, and the push-relabel solver's
// global-relabel BFS depth with it (367 -> 128 BFS steps per graph, modelled).
//
// din/dout: in-degree of in_k / out-degree of out_k (links + source / sink
// arcs); vin/vout: contracted vertex ids (-1 = contracted away); succ: the
// unique out-link of out_k when dout == 1 (the node -> coordinator link for
// the sink arc).
__device__ __forceinline__ int contract_walk(const ClusterDev& cd, const int32_t* pse, const int16_t* vin,
                                             const int16_t* vout, const int32_t* succ, int j, bool at_out,
                                             double& c) {
  for (int guard = 0; guard < 2 * cd.N + 2; ++guard) {
    if (!at_out) {
      const int x = vin[j];
      if (x >= 0) return x;
      const int32_t w = pse[j];  // in_j contracted away: through its compute edge
      const int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
      c = ref_min(c, __ldg(cd.cap_tab + __ldg(cd.cap_off + j) + (e - s) - 1));
      at_out = true;
    } else {
      const int x = vout[j];
      if (x >= 0) return x;
      const int link = succ[j];  // out_j contracted away: its unique out-edge
      c = ref_min(c, __ldg(cd.link_cap + link));
      const int m = (int)(__ldg(cd.link_pack + link) >> 16) - 1;
      if (m < 0) return 1;  // the sink
      j = m;
      at_out = false;
    }
  }
  return -1;  // unreachable on a DAG
}

__device__ int build_graph_score_contract(const ClusterDev& cd, const Gs& g, const Layout& lay, const int16_t* row,
                                          int partial, int lane, int& V, int& E) {
  const int N = cd.N, L = cd.L;
  int32_t* pse = reinterpret_cast<int32_t*>(g.ps);
  int32_t* din = reinterpret_cast<int32_t*>(g.efwd);
  int32_t* dout = din + N;
  int16_t* vin = g.vin;
  int16_t* vout = g.vin + N;
  int32_t* succ = reinterpret_cast<int32_t*>(g.unode);
  int bad = INT_MAX;
  const int32_t* row32 = reinterpret_cast<const int32_t*>(row);
  for (int k = lane; k < N; k += 32) {
    const int32_t w = __ldg(row32 + k);
    const int s = (int16_t)(w & 0xffff);
    const int e = (int16_t)(w >> 16);
    pse[k] = w;
    din[k] = 0;
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
  // degrees, and each out-vertex's last valid out-link (its only one when dout == 1)
  for (int k = lane; k < N; k += 32) {
    const int32_t w = pse[k];
    const int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
    if (e <= s) continue;
    int nout = 0, last = -1;
    for_valid_out_links(cd, pse, k, e, partial, [&](int j, int link) {
      ++nout;
      last = link;
      atomicAdd(&din[j], 1);
    });
    if (s == 0 && __ldg(cd.cout_link + k) >= 0) atomicAdd(&din[k], 1);
    const int lk = __ldg(cd.cin_link + k);
    const bool snk = e == L && lk >= 0;
    dout[k] = nout + (snk ? 1 : 0);
    succ[k] = snk ? lk : last;
  }
  __syncwarp();
  // kept vertices, numbered in node order after s = 0, t = 1
  int run = 2;
  for (int k0 = 0; k0 < N; k0 += 32) {
    const int k = k0 + lane;
    bool kin = false, kout = false;
    if (k < N) {
      const int32_t w = pse[k];
      const bool used = (int16_t)(w >> 16) > (int16_t)(w & 0xffff);
      kin = used && din[k] != 1;
      kout = used && dout[k] != 1;
    }
    const int cnt = (kin ? 1 : 0) + (kout ? 1 : 0);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (k < N) {
      const int base = run + incl - cnt;
      vin[k] = (int16_t)(kin ? base : -1);
      vout[k] = (int16_t)(kout ? base + (kin ? 1 : 0) : -1);
    }
    run += __shfl_sync(FULL, incl, 31);
  }
  V = run;
  if (V > lay.V) return ST_OVERFLOW;
  int* fill = reinterpret_cast<int*>(g.ex);  // per contracted vertex: degree, then slot counter
  // Degrees need no walks: every original edge into a kept vertex ends
  // exactly one contracted edge there, and every contracted edge starts at a
  // kept vertex — s (source arcs), a kept in-vertex (its compute edge) or a
  // kept out-vertex (its dout out-edges).  So deg(in_k) = din + 1,
  // deg(out_k) = 1 + dout, deg(s) = #source arcs, deg(t) = #sink arcs.
  // Arc order is fixed by construction (no atomic order): at every vertex
  // its forward arcs first — the source's in node order, an in-vertex's one
  // compute/contracted edge, an out-vertex's out-links in list order then the
  // sink arc — and then its reverse arcs sorted by their partners' positions.
  int16_t* nf = g.h;  // forward arcs per contracted vertex (h is the solver's; free while building)
  int nedges = 0, nsrc = 0, nsnk = 0;
  for (int k = lane; k < N; k += 32) {
    const int32_t w = pse[k];
    const int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
    if (e <= s) continue;
    if (s == 0 && __ldg(cd.cout_link + k) >= 0) {
      ++nsrc;
      ++nedges;
    }
    if (e == L && __ldg(cd.cin_link + k) >= 0) ++nsnk;
    const int xi = vin[k], xo = vout[k];
    if (xi >= 0) {
      fill[xi] = din[k] + 1;
      nf[xi] = 1;
      ++nedges;
    }
    if (xo >= 0) {
      fill[xo] = 1 + dout[k];
      nf[xo] = (int16_t)dout[k];
      nedges += dout[k];
    }
  }
  nedges = __reduce_add_sync(FULL, nedges);
  nsrc = __reduce_add_sync(FULL, nsrc);
  nsnk = __reduce_add_sync(FULL, nsnk);
  if (2 * nedges > lay.A) return ST_OVERFLOW;
  // the source's arcs in node order: rank of k among the source-fed nodes
  // (din is free once the degrees are in)
  {
    int run2 = 0;
    for (int k0 = 0; k0 < N; k0 += 32) {
      const int k = k0 + lane;
      bool f = false;
      if (k < N) {
        const int32_t w = pse[k];
        const int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
        f = e > s && s == 0 && __ldg(cd.cout_link + k) >= 0;
      }
      const unsigned m = __ballot_sync(FULL, f);
      if (f) din[k] = run2 + __popc(m & ((1u << lane) - 1u));
      run2 += __popc(m);
    }
  }
  if (lane == 0) {
    fill[0] = nsrc;
    fill[1] = nsnk;
    nf[0] = (int16_t)nsrc;
    nf[1] = 0;
  }
  __syncwarp();
  int* rfill = fill + V;  // reverse-arc counters (the ex region holds 2V ints)
  {
    int r2 = 0;
    for (int x0 = 0; x0 < V; x0 += 32) {
      const int x = x0 + lane;
      const int d = x < V ? fill[x] : 0;
      int incl = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      if (x < V) {
        g.abeg[x] = (int16_t)(r2 + incl - d);
        rfill[x] = 0;
      }
      r2 += __shfl_sync(FULL, incl, 31);
    }
    if (lane == 0) g.abeg[V] = (int16_t)r2;
  }
  __syncwarp();
  // one walk per contracted edge: forward arc at its start (slot given),
  // reverse at its end (claimed, sorted below)
  auto emit = [&](int a, int fslot, int b, double c) {
    const int fa = g.abeg[a] + fslot;
    const int ra = g.abeg[b] + nf[b] + atomicAdd(&rfill[b], 1);
    g.to[fa] = (int16_t)b;
    g.rv[fa] = (int16_t)ra;
    g.cap[fa] = c;
    g.to[ra] = (int16_t)a;
    g.rv[ra] = (int16_t)fa;
    g.cap[ra] = 0.0;
  };
  for (int k = lane; k < N; k += 32) {
    const int32_t w = pse[k];
    const int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
    if (e <= s) continue;
    const int lc = __ldg(cd.cout_link + k);
    if (s == 0 && lc >= 0) {
      double c = __ldg(cd.link_cap + lc);
      const int b = contract_walk(cd, pse, vin, vout, succ, k, false, c);
      emit(0, din[k], b, c);
    }
    const int xi = vin[k];
    if (xi >= 0) {
      double c = __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (e - s) - 1);
      const int b = contract_walk(cd, pse, vin, vout, succ, k, true, c);
      emit(xi, 0, b, c);
    }
    const int xo = vout[k];
    if (xo >= 0) {
      int fo = 0;
      for_valid_out_links(cd, pse, k, e, partial, [&](int j, int link) {
        double c = __ldg(cd.link_cap + link);
        const int b = contract_walk(cd, pse, vin, vout, succ, j, false, c);
        emit(xo, fo++, b, c);
      });
      const int lk = __ldg(cd.cin_link + k);
      if (e == L && lk >= 0) emit(xo, fo, 1, __ldg(cd.link_cap + lk));
    }
  }
  __syncwarp();
  // reverse arcs by partner position (partners are forward arcs, which stay
  // put), then each partner pointed back at its reverse arc's final slot
  for (int x = lane; x < V; x += 32) {
    const int b0 = g.abeg[x] + nf[x], b1 = g.abeg[x + 1];
    for (int i = b0 + 1; i < b1; ++i) {
      const int16_t ti = g.to[i], ri = g.rv[i];
      int j = i - 1;
      while (j >= b0 && g.rv[j] > ri) {
        g.to[j + 1] = g.to[j];
        g.rv[j + 1] = g.rv[j];
        --j;
      }
      g.to[j + 1] = ti;
      g.rv[j + 1] = ri;
    }
    for (int i = b0; i < b1; ++i) g.rv[g.rv[i]] = (int16_t)i;
  }
  __syncwarp();
  E = nedges;
  return 0;
}

// The round-1 general builder (one out-link per step), kept for the combined
// small-cluster kernel, whose register allocation is tuned with it.
__device__ int build_graph_score_r1(const ClusterDev& cd, const Gs& g, const Layout& lay, const int16_t* row,
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
  // valid out-links + sink arc.  One pass over the out-lists: a valid link
  // k -> j adds to out_k here and to in_j through a shared atomic.
  int nedges = 0, dsrc = 0, dsink = 0;
  int* fill = reinterpret_cast<int*>(g.ex);  // int counters per vertex during the build
  for (int x = lane; x < V; x += 32) fill[x] = 0;
  __syncwarp();
  for (int k = lane; k < N; k += 32) {
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    int din = 1, dout = 1;
    ++nedges;
    for (int p = __ldg(cd.out_beg + k), pe_ = __ldg(cd.out_beg + k + 1); p < pe_; ++p) {
      const int j = __ldg(&cd.out_list[p].x);
      const int sj = g.ps[j], ej = g.pe[j];
      if (ej > sj && edge_ok(e, sj, ej, partial)) {
        ++dout;
        atomicAdd(&fill[2 + 2 * j], 1);
      }
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
    atomicAdd(&fill[2 + 2 * k], din);
    fill[3 + 2 * k] = dout;  // only this lane touches an out-vertex's count
  }
  nedges = __reduce_add_sync(FULL, nedges);
  dsrc = __reduce_add_sync(FULL, dsrc);
  dsink = __reduce_add_sync(FULL, dsink);
  E = nedges;
  if (2 * E > lay.A) return ST_OVERFLOW;
  if (lane == 0) {
    fill[0] = dsrc;
    fill[1] = dsink;
  }
  __syncwarp();
  // arc ranges; each used node's compute pair takes slot 0 of both its
  // vertices (so the pair arc of x >= 2 is arc abeg[x]), the rest fill in.
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
    if (x < V) {
      g.abeg[x] = (int16_t)(run + incl - d);
      fill[x] = (x >= 2 && d > 0) ? 1 : 0;
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
    const int ai = g.abeg[vi];
    const int ao = g.abeg[vo];
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
                                       int partial, int lane, int& V, int& E, double& cut) {
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
  // Layer cut: every source -> sink path crosses the compute edge of some node
  // covering layer l (intervals chain from 0 to L), so those compute edges are
  // an s-t cut for each l; cut = the smallest one (summed in node order) bounds
  // the max-flow value, and a solver that reaches it can stop.
  {
    double c = 1.0e300;
    for (int l = lane; l < L; l += 32) {
      double sum = 0.0;
      for (unsigned long long m = cover[l]; m; m &= m - 1) {
        const int k = __ffsll(m) - 1;
        sum += __ldg(cd.cap_tab + __ldg(cd.cap_off + k) + (g.pe[k] - g.ps[k]) - 1);
      }
      c = ref_min(c, sum);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c = ref_min(c, __shfl_xor_sync(FULL, c, o));
    cut = c;
  }
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
  // each used node's compute pair takes slot 0 of both its vertices
  for (int x = lane; x < V; x += 32) fill[x] = (x >= 2 && g.abeg[x + 1] > g.abeg[x]) ? 1 : 0;
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = lane + 32 * q;
    if (k >= N) continue;
    const int s = g.ps[k], e = g.pe[k];
    if (e <= s) continue;
    const int vi = 2 + 2 * k, vo = vi + 1;
    const int ai = g.abeg[vi];
    const int ao = g.abeg[vo];
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

}  // namespace
