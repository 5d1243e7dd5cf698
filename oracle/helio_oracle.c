/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * Used by tests/ (as the checker for the CUDA path), __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg.  The product never links or calls it.
 * Parity of this restatement is pinned two ways: against the compiled
 * reference (oracle/_ref/libhelio_ref.so, built from /root/reference by
 * oracle/Makefile) on seeded inputs, and against the golden vectors committed
 * in tests/golden/ (generated from that same compiled reference by
 * tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Arithmetic is kept in the reference's exact
 * operation order so doubles match bit for bit; compile with
 * -ffp-contract=off. */
#include "helio_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FLOW_EPS 1e-12 /* kFlowEps, flow_graph.cpp:15 */

static double dmin(double a, double b) { return b < a ? b : a; } /* std::min */
static double dmax(double a, double b) { return a < b ? b : a; } /* std::max */

/* ClusterSpec::max_layers, cluster.cpp:62-68 */
int ora_max_layers(const ora_cluster* c, int k) {
  double usable = c->vram_bytes[k] * (1.0 - c->kv_reserve[k]);
  double bpl = c->param_bytes / c->num_layers;
  int kk = (int)floor(usable / bpl);
  int tl = c->table_off[k + 1] - c->table_off[k];
  if (tl > 0 && tl < kk) kk = tl;
  return kk < c->num_layers ? kk : c->num_layers;
}

/* ClusterSpec::throughput, cluster.cpp:70-76 (caller guarantees 1<=j<=k_i) */
static double ora_throughput(const ora_cluster* c, int k, int j) {
  int tl = c->table_off[k + 1] - c->table_off[k];
  if (tl > 0) return c->table_val[c->table_off[k] + j - 1];
  return c->peak_layer_tokens[k] / j;
}

/* ClusterSpec::nic_in / nic_out, cluster.cpp:82-96 */
static double ora_nic(const ora_cluster* c, int k, double explicit_bps) {
  if (explicit_bps > 0) return explicit_bps;
  double best = 0;
  for (int l = 0; l < c->num_links; ++l)
    if (c->link_src[l] == k || c->link_dst[l] == k) best = dmax(best, c->link_bw[l]);
  return best;
}

/* compute_edge_capacity, flow_graph.cpp:38-43 */
double ora_compute_edge_capacity(const ora_cluster* c, int k, int j) {
  double rate = ora_throughput(c, k, j);
  double act = c->activation_bytes;
  double nic_rate = dmin(ora_nic(c, k, c->nic_in_bps[k]), ora_nic(c, k, c->nic_out_bps[k])) / (8.0 * act);
  return dmin(rate, nic_rate);
}

typedef struct {
  int nv, ne;
  int32_t *u, *v, *kind, *es, *ee, *sn, *dn; /* sn/dn: node index, -1 coordinator */
  double* cap;
  int max_e;
} graph_buf;

/* add_merged_edge, flow_graph.cpp:25-34 (linear dedup; graphs are small) */
static int add_edge(graph_buf* g, int u, int v, double cap, int kind, int sn, int dn, int es, int ee) {
  for (int i = 0; i < g->ne && i < g->max_e; ++i)
    if (g->u[i] == u && g->v[i] == v) {
      g->cap[i] += cap;
      return 0;
    }
  if (g->ne < g->max_e) {
    int i = g->ne;
    g->u[i] = u; g->v[i] = v; g->cap[i] = cap; g->kind[i] = kind;
    g->sn[i] = sn; g->dn[i] = dn; g->es[i] = es; g->ee[i] = ee;
  }
  g->ne++;
  return 0;
}

static const ora_cluster* g_sort_c;
static int cmp_lex(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return g_sort_c->lex_rank[x] - g_sort_c->lex_rank[y];
}

/* build_flow_graph, flow_graph.cpp:45-136.  Nodes are visited in the
 * byte-lexicographic order of their ids (std::map<std::string,...>, :51). */
static int build(const ora_cluster* c, const int16_t* pl, int partial, graph_buf* g, int* vin) {
  const int N = c->num_nodes, L = c->num_layers;
  int* order = (int*)malloc(sizeof(int) * (N > 0 ? N : 1));
  int nu = 0;
  for (int k = 0; k < N; ++k) order[k] = k;
  g_sort_c = c;
  qsort(order, N, sizeof(int), cmp_lex);
  /* validation in map order, :52-61 */
  for (int r = 0; r < N; ++r) {
    int k = order[r];
    int s = pl[2 * k], e = pl[2 * k + 1];
    if (e <= s) continue; /* iv.empty() */
    if (s < 0 || e > L) { free(order); return 2; }
    if (e - s > ora_max_layers(c, k)) { free(order); return 3; }
  }
  g->nv = 2;
  g->ne = 0;
  for (int k = 0; k < N; ++k) vin[k] = -1;
  /* vertices, :63-69 */
  for (int r = 0; r < N; ++r) {
    int k = order[r];
    if (pl[2 * k + 1] <= pl[2 * k]) continue;
    vin[k] = g->nv;
    g->nv += 2;
    ++nu;
  }
  /* compute edges, :71-84 */
  for (int r = 0; r < N; ++r) {
    int k = order[r];
    int s = pl[2 * k], e = pl[2 * k + 1];
    if (e <= s) continue;
    add_edge(g, vin[k], vin[k] + 1, ora_compute_edge_capacity(c, k, e - s), 0, k, k, s, e);
  }
  /* links in declaration order, :86-134 */
  for (int l = 0; l < c->num_links; ++l) {
    int a = c->link_src[l], b = c->link_dst[l];
    if (a == -1) {
      if (b < 0 || vin[b] < 0 || pl[2 * b] != 0) continue;
      add_edge(g, 0, vin[b], c->link_bw[l] / (8.0 * c->token_bytes), 1, -1, b, 0, pl[2 * b + 1]);
    } else if (b == -1) {
      if (a < 0 || vin[a] < 0 || pl[2 * a + 1] != L) continue;
      add_edge(g, vin[a] + 1, 1, c->link_bw[l] / (8.0 * c->token_bytes), 2, a, -1, L, L);
    } else {
      if (a < 0 || b < 0 || vin[a] < 0 || vin[b] < 0) continue;
      int aend = pl[2 * a + 1], bs = pl[2 * b], be = pl[2 * b + 1];
      int valid = partial ? (bs <= aend && aend < be) : (aend == bs);
      if (!valid) continue;
      add_edge(g, vin[a] + 1, vin[b], c->link_bw[l] / (8.0 * c->activation_bytes), 3, a, b, aend, be);
    }
  }
  (void)nu;
  free(order);
  return 0;
}

int ora_build(const ora_cluster* c, const int16_t* pl, int allow_partial, int max_e, int32_t* nv,
              int32_t* ne, int32_t* u, int32_t* v, int32_t* kind, int32_t* es, int32_t* ee,
              double* cap) {
  int N = c->num_nodes;
  int* vin = (int*)malloc(sizeof(int) * (N > 0 ? N : 1));
  int32_t* sn = (int32_t*)malloc(sizeof(int32_t) * (max_e > 0 ? max_e : 1));
  int32_t* dn = (int32_t*)malloc(sizeof(int32_t) * (max_e > 0 ? max_e : 1));
  graph_buf g = {0, 0, u, v, kind, es, ee, sn, dn, cap, max_e};
  int st = build(c, pl, allow_partial, &g, vin);
  free(vin); free(sn); free(dn);
  if (st) return st;
  *nv = g.nv;
  *ne = g.ne;
  return g.ne > max_e ? -2 : 0;
}

/* max_flow, flow_graph.cpp:138-229: FIFO preflow-push with the gap heuristic. */
typedef struct { int to; double cap; int rev; int edge_id; } arc_t;

double ora_max_flow(int n, int s, int t, int m, const int32_t* eu, const int32_t* ev,
                    const double* ecap, double* flow) {
  int* deg = (int*)calloc(n + 1, sizeof(int));
  for (int i = 0; i < m; ++i) { deg[eu[i]]++; deg[ev[i]]++; }
  int* beg = (int*)malloc(sizeof(int) * (n + 1));
  int* fill = (int*)calloc(n, sizeof(int));
  beg[0] = 0;
  for (int x = 0; x < n; ++x) beg[x + 1] = beg[x] + deg[x];
  arc_t* arcs = (arc_t*)malloc(sizeof(arc_t) * (2 * m + 1));
  /* residual arcs per vertex in edge order, :140-145 (rev is evaluated
   * before the push_back, so a self-loop's forward arc points at itself) */
  for (int i = 0; i < m; ++i) {
    int a = eu[i], b = ev[i];
    int pa = fill[a];
    arc_t fa = {b, ecap[i], fill[b], i};
    arcs[beg[a] + fill[a]++] = fa;
    arc_t ra = {a, 0.0, pa, -1};
    arcs[beg[b] + fill[b]++] = ra;
  }
  double* excess = (double*)calloc(n, sizeof(double));
  int* height = (int*)calloc(n, sizeof(int));
  int* count = (int*)calloc(2 * n + 1, sizeof(int));
  int* current = (int*)calloc(n, sizeof(int));
  int* queue = (int*)malloc(sizeof(int) * (n + 1));
  char* inq = (char*)calloc(n, 1);
  int qh = 0, qt = 0, qn = 0; /* ring of capacity n+1 */
  height[s] = n;
  count[0] = n - 1;
  count[n] = 1;
#define PUSH(U, A)                                                         \
  do {                                                                     \
    arc_t* a_ = (A);                                                       \
    double amt = dmin(excess[U], a_->cap);                                 \
    a_->cap -= amt;                                                        \
    arcs[beg[a_->to] + a_->rev].cap += amt;                                \
    excess[U] -= amt;                                                      \
    excess[a_->to] += amt;                                                 \
    if (a_->to != s && a_->to != t && !inq[a_->to]) {                      \
      queue[qt] = a_->to; qt = (qt + 1) % (n + 1); qn++;                   \
      inq[a_->to] = 1;                                                     \
    }                                                                      \
  } while (0)
  /* saturate source arcs, :168-173 */
  for (int j = beg[s]; j < beg[s + 1]; ++j) {
    if (arcs[j].cap > FLOW_EPS) {
      excess[s] += arcs[j].cap;
      PUSH(s, &arcs[j]);
    }
  }
  /* discharge loop, :175-208 */
  while (qn > 0) {
    int u = queue[qh];
    qh = (qh + 1) % (n + 1);
    qn--;
    inq[u] = 0;
    int du = beg[u + 1] - beg[u];
    while (excess[u] > FLOW_EPS) {
      if (current[u] == du) {
        int old = height[u];
        int best = 2 * n;
        for (int j = beg[u]; j < beg[u + 1]; ++j)
          if (arcs[j].cap > FLOW_EPS && height[arcs[j].to] + 1 < best) best = height[arcs[j].to] + 1;
        height[u] = best;
        current[u] = 0;
        count[old]--;
        count[best]++;
        if (old < n && count[old] == 0) {
          for (int x = 0; x < n; ++x) {
            if (x != s && height[x] > old && height[x] < n) {
              count[height[x]]--;
              height[x] = n + 1;
              count[height[x]]++;
            }
          }
        }
        if (best >= 2 * n) break;
      } else {
        arc_t* a = &arcs[beg[u] + current[u]];
        if (a->cap > FLOW_EPS && height[u] == height[a->to] + 1)
          PUSH(u, a);
        else
          ++current[u];
      }
    }
  }
#undef PUSH
  /* flows from residuals, :210-221; value in edge order, :222-227 */
  double value = 0;
  double* fl = (double*)malloc(sizeof(double) * (m > 0 ? m : 1));
  for (int x = 0; x < n; ++x)
    for (int j = beg[x]; j < beg[x + 1]; ++j)
      if (arcs[j].edge_id >= 0) {
        int i = arcs[j].edge_id;
        fl[i] = ecap[i] - arcs[j].cap;
        if (fl[i] < FLOW_EPS) fl[i] = 0;
      }
  for (int i = 0; i < m; ++i) {
    if (ev[i] == t) value += fl[i];
    if (eu[i] == t) value -= fl[i];
  }
  if (flow) memcpy(flow, fl, sizeof(double) * m);
  free(fl); free(deg); free(beg); free(fill); free(arcs); free(excess); free(height);
  free(count); free(current); free(queue); free(inq);
  return value;
}

int ora_score(const ora_cluster* c, const int16_t* pl, int64_t B, int allow_partial,
              double* values, int32_t* status) {
  int N = c->num_nodes;
  int max_e = N + c->num_links + 1;
  int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * 7 * max_e);
  double* cap = (double*)malloc(sizeof(double) * max_e);
  int* vin = (int*)malloc(sizeof(int) * (N > 0 ? N : 1));
  for (int64_t b = 0; b < B; ++b) {
    graph_buf g = {0, 0, buf, buf + max_e, buf + 2 * max_e, buf + 3 * max_e, buf + 4 * max_e,
                   buf + 5 * max_e, buf + 6 * max_e, cap, max_e};
    int st = build(c, pl + b * 2 * N, allow_partial, &g, vin);
    status[b] = st;
    values[b] = st ? 0.0 : ora_max_flow(g.nv, 0, 1, g.ne, g.u, g.v, g.cap, NULL);
  }
  free(buf); free(cap); free(vin);
  return 0;
}

/* iwrr_weights, scheduler.cpp:46-56 */
void ora_iwrr_weights(const double* flows, int n, int64_t* w) {
  int64_t wmax = 0;
  for (int i = 0; i < n; ++i) {
    int64_t x = llround(1000.0 * flows[i]);
    w[i] = x > 1 ? x : 1;
    if (w[i] > wmax) wmax = w[i];
  }
  if (wmax > 32)
    for (int i = 0; i < n; ++i) {
      int64_t x = llround(w[i] * 32.0 / wmax);
      w[i] = x > 1 ? x : 1;
    }
}

/* fill_plan_edges / plan_from_placement, placement.cpp:440-469 */
int ora_plan(const ora_cluster* c, const int16_t* pl, int allow_partial, int max_edges,
             int32_t* src, int32_t* dst, double* flow, int32_t* es, int32_t* ee,
             double* objective) {
  int N = c->num_nodes;
  int max_e = N + c->num_links + 1;
  int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * 7 * max_e);
  double* cap = (double*)malloc(sizeof(double) * max_e);
  double* fl = (double*)malloc(sizeof(double) * max_e);
  int* vin = (int*)malloc(sizeof(int) * (N > 0 ? N : 1));
  graph_buf g = {0, 0, buf, buf + max_e, buf + 2 * max_e, buf + 3 * max_e, buf + 4 * max_e,
                 buf + 5 * max_e, buf + 6 * max_e, cap, max_e};
  int st = build(c, pl, allow_partial, &g, vin);
  int out = 0;
  if (st) {
    out = -st;
  } else {
    *objective = ora_max_flow(g.nv, 0, 1, g.ne, g.u, g.v, g.cap, fl);
    for (int i = 0; i < g.ne; ++i) {
      if (g.kind[i] == 0 || fl[i] <= 1e-9) continue;
      if (out < max_edges) {
        src[out] = g.kind[i] == 1 ? -1 : g.sn[i];
        dst[out] = g.kind[i] == 2 ? -1 : g.dn[i];
        flow[out] = fl[i];
        es[out] = g.es[i];
        ee[out] = g.ee[i];
      }
      ++out;
    }
  }
  free(buf); free(cap); free(fl); free(vin);
  return out;
}

/* IwrrPicker, scheduler.cpp:28-44 */
typedef struct { int64_t* w; int n; int64_t wmax, round; int idx; } picker_t;

/* Scheduler (IWRR policy): ctor scheduler.cpp:58-98, hop_charge :100-103,
 * hop_eligible :105-108, admit :157-181, complete :183-190, driven by the AC8
 * loop (acceptance_main.cpp:529-537): admit(r, in[r]); if admitted,
 * complete(r, out[r]).  Returns the number of deferred requests, -1 on a plan
 * that the reference Scheduler would reject. */
int64_t ora_route(const ora_cluster* c, const int16_t* pl, int allow_partial, int64_t R,
                  const int32_t* in_len, const int32_t* out_len, int max_hops, int32_t* nhops,
                  int32_t* hop_node, int32_t* hop_s, int32_t* hop_e) {
  const int N = c->num_nodes, L = c->num_layers;
  int max_e = N + c->num_links + 1;
  int32_t* src = (int32_t*)malloc(sizeof(int32_t) * max_e);
  int32_t* dst = (int32_t*)malloc(sizeof(int32_t) * max_e);
  int32_t* es = (int32_t*)malloc(sizeof(int32_t) * max_e);
  int32_t* ee = (int32_t*)malloc(sizeof(int32_t) * max_e);
  double* fl = (double*)malloc(sizeof(double) * max_e);
  double obj = 0;
  int ne = ora_plan(c, pl, allow_partial, max_e, src, dst, fl, es, ee, &obj);
  if (ne <= 0) { free(src); free(dst); free(es); free(ee); free(fl); return -1; }
  /* vertices: 0 = coordinator, then used nodes in id order */
  int* order = (int*)malloc(sizeof(int) * N);
  int* vof = (int*)malloc(sizeof(int) * N);
  int* node_of = (int*)malloc(sizeof(int) * (N + 1));
  for (int k = 0; k < N; ++k) { order[k] = k; vof[k] = -1; }
  g_sort_c = c;
  qsort(order, N, sizeof(int), cmp_lex);
  int nvtx = 1;
  node_of[0] = -1;
  for (int r = 0; r < N; ++r) {
    int k = order[r];
    if (pl[2 * k + 1] <= pl[2 * k]) continue;
    vof[k] = nvtx;
    node_of[nvtx++] = k;
  }
  double bpl = c->param_bytes / c->num_layers;
  double* kv_cap = (double*)calloc(nvtx, sizeof(double));
  double* kv_est = (double*)calloc(nvtx, sizeof(double));
  for (int x = 1; x < nvtx; ++x) {
    int k = node_of[x];
    int held = pl[2 * k + 1] - pl[2 * k];
    kv_cap[x] = dmax(0.0, c->vram_bytes[k] - held * bpl);
  }
  /* out-edges per vertex in plan order */
  int* ob = (int*)calloc(nvtx + 1, sizeof(int));
  int* ofill = (int*)calloc(nvtx, sizeof(int));
  int* e_src = (int*)malloc(sizeof(int) * ne);
  for (int i = 0; i < ne; ++i) {
    e_src[i] = src[i] < 0 ? 0 : vof[src[i]];
    ob[e_src[i] + 1]++;
  }
  for (int x = 0; x < nvtx; ++x) ob[x + 1] += ob[x];
  int* oe = (int*)malloc(sizeof(int) * ne); /* plan edge index per slot */
  for (int i = 0; i < ne; ++i) oe[ob[e_src[i]] + ofill[e_src[i]]++] = i;
  picker_t* pk = (picker_t*)calloc(nvtx, sizeof(picker_t));
  int64_t* wall = (int64_t*)malloc(sizeof(int64_t) * ne);
  double* ftmp = (double*)malloc(sizeof(double) * ne);
  for (int x = 0; x < nvtx; ++x) {
    int d = ob[x + 1] - ob[x];
    for (int j = 0; j < d; ++j) ftmp[j] = fl[oe[ob[x] + j]];
    ora_iwrr_weights(ftmp, d, wall + ob[x]);
    pk[x].w = wall + ob[x];
    pk[x].n = d;
    pk[x].wmax = 1;
    for (int j = 0; j < d; ++j) if (pk[x].w[j] > pk[x].wmax) pk[x].wmax = pk[x].w[j];
    pk[x].round = 1;
    pk[x].idx = 0;
  }
  double kvb = c->kv_bytes_per_token_layer > 0 ? c->kv_bytes_per_token_layer : 2.0 * c->activation_bytes;
  double avg_output = 232.0;
  long samples = 1;
  int64_t denied = 0;
  int* ch_v = (int*)malloc(sizeof(int) * (L + 1));
  double* ch_b = (double*)malloc(sizeof(double) * (L + 1));
  for (int64_t r = 0; r < R; ++r) {
    int v = 0, covered = 0, nh = 0, ok = 1;
    while (covered < L) {
      picker_t* p = &pk[v];
      int pick = -1;
      if (p->n > 0) {
        int64_t positions = p->wmax * (int64_t)p->n;
        for (int64_t it = 0; it < positions; ++it) {
          if (p->idx == p->n) {
            p->idx = 0;
            p->round = p->round == p->wmax ? 1 : p->round + 1;
          }
          int i = p->idx++;
          if (p->w[i] >= p->round) {
            int pe = oe[ob[v] + i];
            int d = dst[pe] < 0 ? 0 : vof[dst[pe]];
            int elig = 1;
            if (d != 0) {
              double charge = (in_len[r] + avg_output) * kvb * (ee[pe] - es[pe]);
              elig = kv_est[d] + charge <= 0.9 * kv_cap[d];
            }
            if (elig) { pick = i; break; }
          }
        }
      }
      if (pick < 0) {
        for (int q = 0; q < nh; ++q) kv_est[ch_v[q]] -= ch_b[q];
        ok = 0;
        break;
      }
      int pe = oe[ob[v] + pick];
      int d = dst[pe] < 0 ? 0 : vof[dst[pe]];
      if (d == 0 || es[pe] != covered) { ok = -1; break; } /* InternalError */
      double bytes = (in_len[r] + avg_output) * kvb * (ee[pe] - es[pe]);
      kv_est[d] += bytes;
      ch_v[nh] = d;
      ch_b[nh] = bytes;
      if (nh < max_hops) {
        hop_node[r * max_hops + nh] = node_of[d];
        hop_s[r * max_hops + nh] = es[pe];
        hop_e[r * max_hops + nh] = ee[pe];
      }
      ++nh;
      covered = ee[pe];
      v = d;
    }
    if (ok < 0) { denied = -2; break; }
    if (!ok) { nhops[r] = -1; ++denied; continue; }
    nhops[r] = nh;
    for (int q = 0; q < nh; ++q) kv_est[ch_v[q]] -= ch_b[q];
    ++samples;
    avg_output += (out_len[r] - avg_output) / (double)samples;
  }
  free(src); free(dst); free(es); free(ee); free(fl); free(order); free(vof); free(node_of);
  free(kv_cap); free(kv_est); free(ob); free(ofill); free(e_src); free(oe); free(pk); free(wall);
  free(ftmp); free(ch_v); free(ch_b);
  return denied;
}
