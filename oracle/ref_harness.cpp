// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" harness around the UNMODIFIED reference library (compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the Python test-suite, the golden-vector generator (tests/golden/make_golden.py)
// and bench.py's reference arm call the reference's own public API:
//
//   build_flow_graph + max_flow      proj/src/flow_graph.cpp:45-229
//   plan_from_placement              proj/src/placement.cpp:459-469
//   iwrr_weights / IwrrPicker        proj/src/scheduler.cpp:28-56
//   Scheduler::admit / complete      proj/src/scheduler.cpp:58-190
//   generate_trace                   proj/src/workload.cpp:37-57
//   swarm / petals / sp heuristics   proj/src/heuristics.cpp:12-131
//   AC1 random raw graphs            proj/tests/acceptance/acceptance_main.cpp:266-295
//   test_flow random graphs          proj/tests/test_flow.cpp:141-188
//
// Placements cross this boundary as int16 [N][2] (start, end) rows in the
// cluster's declared node order; rows with end <= start are idle, exactly like
// an empty Interval in the reference's Placement map (flow_graph.cpp:53).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "helio/cluster.hpp"
#include "helio/errors.hpp"
#include "helio/flow_graph.hpp"
#include "helio/heuristics.hpp"
#include "helio/placement.hpp"
#include "helio/rng.hpp"
#include "helio/scheduler.hpp"
#include "helio/sim.hpp"
#include "helio/workload.hpp"
#include "json.hpp"
#include "oracles/enumerate.hpp"
#include "oracles/random_cluster.hpp"

using namespace helio;

namespace {

void set_err(char* err, int errlen, const std::string& msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

Placement to_placement(const ClusterSpec& c, const int16_t* pl) {
  Placement p;
  for (size_t k = 0; k < c.nodes.size(); ++k) {
    int s = pl[2 * k], e = pl[2 * k + 1];
    if (e > s) p[c.nodes[k].id] = {s, e};
  }
  return p;
}

// Map the reference's three ValidationError texts (flow_graph.cpp:55-59) to codes.
int status_of(const std::string& what) {
  if (what.find("unknown node") != std::string::npos) return 1;
  if (what.find("outside [0,") != std::string::npos) return 2;
  if (what.find("VRAM layer capacity") != std::string::npos) return 3;
  return 9;
}

int node_idx(const ClusterSpec& c, const std::string& id) {
  if (id == c.coordinator_id) return -1;
  return c.node_index(id);
}

}  // namespace

extern "C" {

void* refh_cluster_from_json(const char* text, char* err, int errlen) {
  try {
    return new ClusterSpec(parse_cluster(text, "<refh>"));
  } catch (const std::exception& ex) {
    set_err(err, errlen, ex.what());
    return nullptr;
  }
}

void refh_cluster_free(void* c) { delete static_cast<ClusterSpec*>(c); }

int refh_cluster_num_nodes(void* c) { return static_cast<int>(static_cast<ClusterSpec*>(c)->nodes.size()); }

int refh_max_layers(void* cp, int k) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  return c.max_layers(c.nodes[k]);
}

double refh_compute_edge_capacity(void* cp, int k, int j) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  return compute_edge_capacity(c, c.nodes[k], j);
}

// Full FlowGraph + max_flow for one candidate.  Returns 0 ok, 1/2/3 for the
// three ValidationErrors, -2 when max_e is too small (ne holds the need).
int refh_graph(void* cp, const int16_t* pl, int allow_partial, int max_e, int32_t* nv, int32_t* ne,
               int32_t* u, int32_t* v, int32_t* kind, int32_t* es, int32_t* ee, double* cap,
               double* flow, double* value, char* err, int errlen) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  FlowGraph g;
  try {
    g = build_flow_graph(c, to_placement(c, pl), allow_partial != 0);
  } catch (const ValidationError& ex) {
    set_err(err, errlen, ex.what());
    return status_of(ex.what());
  }
  *value = max_flow(g);
  *nv = g.num_vertices;
  *ne = static_cast<int32_t>(g.edges.size());
  if (static_cast<int>(g.edges.size()) > max_e) return -2;
  for (size_t i = 0; i < g.edges.size(); ++i) {
    const FlowEdge& e = g.edges[i];
    u[i] = e.u;
    v[i] = e.v;
    kind[i] = static_cast<int32_t>(e.kind);
    es[i] = e.exec_start;
    ee[i] = e.exec_end;
    cap[i] = e.cap;
    flow[i] = e.flow;
  }
  return 0;
}

// Bulk scoring: exactly the enumerate.hpp:56-57 pair per candidate, on a
// std::thread pool with static chunks (flow_graph.cpp holds no shared state).
int refh_score(void* cp, const int16_t* pl, int64_t B, int allow_partial, int nthreads,
               double* values, int32_t* status) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  const int64_t N = static_cast<int64_t>(c.nodes.size());
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t b = lo; b < hi; ++b) {
      try {
        FlowGraph g = build_flow_graph(c, to_placement(c, pl + b * N * 2), allow_partial != 0);
        values[b] = max_flow(g);
        status[b] = 0;
      } catch (const ValidationError& ex) {
        values[b] = 0;
        status[b] = status_of(ex.what());
      }
    }
  };
  std::vector<std::thread> pool;
  int64_t chunk = (B + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = t * chunk, hi = std::min(B, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  return 0;
}

// Solve-only rate on pre-built graphs (SURVEY.md §8(d) "CPU reference
// timing" item 4): build every candidate's FlowGraph first (untimed), then
// time max_flow alone on the same std::thread pool.  Invalid rows are skipped.
// Returns the number of graphs solved; *solve_s = wall seconds of the solves.
int64_t refh_solve_only(void* cp, const int16_t* pl, int64_t B, int allow_partial, int nthreads,
                        double* solve_s, double* checksum) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  const int64_t N = static_cast<int64_t>(c.nodes.size());
  if (nthreads < 1) nthreads = 1;
  std::vector<FlowGraph> gs;
  gs.reserve(B);
  for (int64_t b = 0; b < B; ++b) {
    try {
      gs.push_back(build_flow_graph(c, to_placement(c, pl + b * N * 2), allow_partial != 0));
    } catch (const ValidationError&) {
    }
  }
  const int64_t G = static_cast<int64_t>(gs.size());
  std::vector<double> part(nthreads, 0.0);
  auto work = [&](int t, int64_t lo, int64_t hi) {
    double acc = 0;
    for (int64_t b = lo; b < hi; ++b) acc += max_flow(gs[b]);
    part[t] = acc;
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  const int64_t chunk = (G + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = t * chunk, hi = std::min(G, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back(work, t, lo, hi);
  }
  for (auto& th : pool) th.join();
  *solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double acc = 0;
  for (double x : part) acc += x;
  *checksum = acc;
  return G;
}

// The benchmark workload generator G(seed, i) of SURVEY.md §8(d), restated
// here over the reference's own ClusterSpec so the reference arm of bench.py
// needs nothing but this library: k_i from ClusterSpec::max_layers
// (cluster.cpp:62-68), walk adjacency from c.links.  The specification (and
// the product's copy, used by the GPU arm) is paper_2406_01566_b200/csrc/gen.h;
// tests/test_oracle_golden.py checks the two produce identical rows.
namespace gen {
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
uint64_t fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t key_of(uint64_t seed, uint64_t i) { return fmix(fmix(seed + kGolden) + (i + 1) * kGolden); }
uint64_t draw(uint64_t key, uint32_t k) { return fmix(key + (uint64_t)(k + 1) * kGolden); }
uint32_t uniform(uint64_t x, uint32_t m) { return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32); }

// covering chains: a random node order; each node takes U[1,k_i] layers from
// the running layer (wrapping at L); with probability ppm/1e6 a uniform interval
void chain(const std::vector<int>& kmax, int L, uint64_t seed, uint64_t i, uint32_t ppm, int16_t* out) {
  const int N = static_cast<int>(kmax.size());
  const uint64_t key = key_of(seed, i);
  std::vector<int> order(N);
  for (int k = 0; k < N; ++k) order[k] = k;
  for (int k = N - 1; k >= 1; --k) std::swap(order[k], order[uniform(draw(key, k), k + 1)]);
  int layer = 0;
  for (int pos = 0; pos < N; ++pos) {
    const int node = order[pos], k = kmax[node];
    const uint32_t d = (uint32_t)N + 3u * (uint32_t)pos;
    int s = 0, e = 0;
    if (k >= 1) {
      if (ppm > 0 && uniform(draw(key, d), 1000000u) < ppm) {
        const int len = (int)uniform(draw(key, d + 1), (uint32_t)k + 1u);
        s = (int)uniform(draw(key, d + 2), (uint32_t)(L - len) + 1u);
        e = s + len;
      } else {
        const int len = 1 + (int)uniform(draw(key, d + 1), (uint32_t)k);
        s = layer;
        e = std::min(layer + len, L);
        layer = e == L ? 0 : e;
      }
    }
    out[2 * node] = (int16_t)s;
    out[2 * node + 1] = (int16_t)e;
  }
}

// link walks (sparse topologies): from the coordinator, step to a uniformly
// chosen unused node over a declared link; restart at layer 0 on reaching L
// or a dead end.  succ[0] = coordinator's targets, succ[1+k] = node k's.
void walk(const std::vector<int>& kmax, int L, uint64_t seed, uint64_t i,
          const std::vector<std::vector<int>>& succ, int16_t* out) {
  const int N = static_cast<int>(kmax.size());
  const uint64_t key = key_of(seed, i);
  std::vector<char> used(N, 0);
  std::fill(out, out + 2 * N, int16_t(0));
  int prev = -1, layer = 0;
  uint32_t nd = 0;
  for (int step = 0; step < 2 * N; ++step) {
    std::vector<int> open;
    for (int j : succ[prev + 1])
      if (!used[j] && kmax[j] >= 1) open.push_back(j);
    if (open.empty()) {
      if (prev == -1) break;
      prev = -1;
      layer = 0;
      continue;
    }
    const int j = open[uniform(draw(key, nd++), (uint32_t)open.size())];
    used[j] = 1;
    const int len = 1 + (int)uniform(draw(key, nd++), (uint32_t)kmax[j]);
    const int e = std::min(layer + len, L);
    out[2 * j] = (int16_t)layer;
    out[2 * j + 1] = (int16_t)e;
    if (e == L) {
      prev = -1;
      layer = 0;
    } else {
      prev = j;
      layer = e;
    }
  }
}
}  // namespace gen

// rows [first, first + n) of the workload into out[n][N][2]; walk != 0 draws
// link walks.  Returns 0.
int refh_generate(void* cp, uint64_t seed, int64_t first, int64_t n, uint32_t ppm, int walk, int nthreads,
                  int16_t* out) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  const int N = static_cast<int>(c.nodes.size());
  const int L = c.model.num_layers;
  std::vector<int> kmax(N);
  for (int k = 0; k < N; ++k) kmax[k] = c.max_layers(c.nodes[k]);
  // declared links, first occurrence of each (src, dst) pair; undeclared
  // endpoints, coordinator loops and self-links never carry flow
  std::vector<std::vector<int>> succ(N + 1);
  std::vector<std::vector<char>> seen(N + 1, std::vector<char>(N, 0));
  for (const LinkSpec& l : c.links) {
    const int a = l.src == c.coordinator_id ? -1 : c.node_index(l.src);
    const int b = l.dst == c.coordinator_id ? -1 : c.node_index(l.dst);
    if ((a < 0 && l.src != c.coordinator_id) || b < 0 || a == b) continue;
    if (!seen[a + 1][b]) {
      seen[a + 1][b] = 1;
      succ[a + 1].push_back(b);
    }
  }
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      int16_t* o = out + r * 2 * N;
      if (walk)
        gen::walk(kmax, L, seed, (uint64_t)(first + r), succ, o);
      else
        gen::chain(kmax, L, seed, (uint64_t)(first + r), ppm, o);
    }
  };
  std::vector<std::thread> pool;
  const int64_t chunk = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  return 0;
}

double refh_maxflow_raw(int n, int s, int t, int m, const int32_t* u, const int32_t* v,
                        const double* cap, double* flow_out) {
  FlowGraph g;
  g.num_vertices = n;
  g.source = s;
  g.sink = t;
  for (int i = 0; i < m; ++i) {
    FlowEdge e;
    e.u = u[i];
    e.v = v[i];
    e.cap = cap[i];
    g.edges.push_back(e);
  }
  double val = max_flow(g);
  for (int i = 0; i < m; ++i) flow_out[i] = g.edges[i].flow;
  return val;
}

// AC1's random raw graphs, drawn with the reference's own Rng exactly as
// acceptance_main.cpp:270-284 does.  sink = n-1, self-loops allowed.
int64_t refh_ac1_graphs(uint64_t seed, int count, int32_t* n, int32_t* t, int32_t* m, int32_t* eu,
                        int32_t* ev, double* ecap, int64_t cap_edges) {
  Rng rng(seed);
  int64_t off = 0;
  for (int it = 0; it < count; ++it) {
    int nv = 2 + static_cast<int>(rng.uniform_int(19));
    int mm = 1 + static_cast<int>(rng.uniform_int(3 * nv));
    n[it] = nv;
    t[it] = nv - 1;
    m[it] = mm;
    for (int i = 0; i < mm; ++i) {
      int a = static_cast<int>(rng.uniform_int(nv));
      int b = static_cast<int>(rng.uniform_int(nv));
      double cc = static_cast<double>(rng.uniform_int(51));
      if (off < cap_edges) {
        eu[off] = a;
        ev[off] = b;
        ecap[off] = cc;
      }
      ++off;
    }
  }
  return off;
}

// test_flow.cpp:143-159 random_graph(rng, 19) x 400 with seed 20240811:
// sink = 1, self-loops dropped.
int64_t refh_testflow_graphs(uint64_t seed, int count, int max_vertices, int32_t* n, int32_t* m,
                             int32_t* eu, int32_t* ev, double* ecap, int64_t cap_edges) {
  Rng rng(seed);
  int64_t off = 0;
  for (int it = 0; it < count; ++it) {
    int nv = 2 + static_cast<int>(rng.uniform_int(max_vertices - 1));
    int mm = 1 + static_cast<int>(rng.uniform_int(3 * nv));
    int kept = 0;
    for (int i = 0; i < mm; ++i) {
      int a = static_cast<int>(rng.uniform_int(nv));
      int b = static_cast<int>(rng.uniform_int(nv));
      if (a == b) continue;
      double cc = static_cast<double>(rng.uniform_int(51));
      if (off < cap_edges) {
        eu[off] = a;
        ev[off] = b;
        ecap[off] = cc;
      }
      ++off;
      ++kept;
    }
    n[it] = nv;
    m[it] = kept;
  }
  return off;
}

void refh_iwrr_weights(const double* flows, int n, int64_t* out) {
  std::vector<long> w = iwrr_weights(std::vector<double>(flows, flows + n));
  for (int i = 0; i < n; ++i) out[i] = w[i];
}

// IwrrPicker sequence with an eligibility mask per call (mask bit i = eligible).
void refh_picker_seq(const int64_t* weights, int n, int calls, const uint64_t* masks, int32_t* out) {
  IwrrPicker p(std::vector<long>(weights, weights + n));
  for (int k = 0; k < calls; ++k) {
    uint64_t mk = masks[k];
    out[k] = p.next([&](int i) { return ((mk >> i) & 1u) != 0; });
  }
}

// plan_from_placement → PlanEdge list (src/dst as node index, -1 = coordinator).
int refh_plan(void* cp, const int16_t* pl, int allow_partial, int max_edges, int32_t* src,
              int32_t* dst, double* flow, int32_t* es, int32_t* ee, double* objective) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  PlacementPlan plan;
  try {
    plan = plan_from_placement(c, to_placement(c, pl), allow_partial != 0, "custom");
  } catch (const ValidationError& ex) {
    return -status_of(ex.what());
  }
  *objective = plan.objective;
  int ne = static_cast<int>(plan.edges.size());
  for (int i = 0; i < ne && i < max_edges; ++i) {
    src[i] = node_idx(c, plan.edges[i].src);
    dst[i] = node_idx(c, plan.edges[i].dst);
    flow[i] = plan.edges[i].flow;
    es[i] = plan.edges[i].exec_start;
    ee[i] = plan.edges[i].exec_end;
  }
  return ne;
}

// The AC8 loop (acceptance_main.cpp:526-537): admit(i, in[i]) then, if
// admitted, complete(i, out[i]).  Hop lists are written at stride max_hops.
// Returns the number of deferred (nullopt) admissions, or -1 on a plan error.
int64_t refh_route(void* cp, const int16_t* pl, int allow_partial, uint64_t seed, int64_t R,
                   const int32_t* in_len, const int32_t* out_len, int max_hops, int32_t* nhops,
                   int32_t* hop_node, int32_t* hop_s, int32_t* hop_e) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  PlacementPlan plan;
  try {
    plan = plan_from_placement(c, to_placement(c, pl), allow_partial != 0, "custom");
  } catch (const std::exception&) {
    return -1;
  }
  // the reference's ValidationErrors (a plan without a coordinator edge, a
  // route that does not tile the layers) come back as -2 / -3 instead of
  // unwinding through the C ABI
  int64_t denied = 0;
  try {
  Scheduler sched(c, plan, SchedPolicy::kIwrr, seed);
  for (int64_t r = 0; r < R; ++r) {
    std::optional<std::vector<RouteHop>> route;
    try {
      route = sched.admit(static_cast<long>(r), in_len[r]);
    } catch (const std::exception&) {
      return -3;
    }
    if (!route) {
      ++denied;
      nhops[r] = -1;
      continue;
    }
    int h = static_cast<int>(route->size());
    nhops[r] = h;
    for (int k = 0; k < h && k < max_hops; ++k) {
      hop_node[r * max_hops + k] = c.node_index((*route)[k].node);
      hop_s[r * max_hops + k] = (*route)[k].exec_start;
      hop_e[r * max_hops + k] = (*route)[k].exec_end;
    }
    sched.complete(static_cast<long>(r), out_len[r]);
  }
  } catch (const std::exception&) {
    return -2;
  }
  return denied;
}

int refh_trace(int count, double rate, int online, uint64_t seed, double mean_in, double mean_out,
               int max_in, int max_out, double* arrival, int32_t* in_len, int32_t* out_len) {
  LengthParams lp;
  lp.mean_input = mean_in;
  lp.mean_output = mean_out;
  lp.max_input = max_in;
  lp.max_output = max_out;
  std::vector<Request> reqs =
      generate_trace(count, rate, online ? TraceMode::kOnline : TraceMode::kOffline, lp, seed);
  for (int i = 0; i < count; ++i) {
    arrival[i] = reqs[i].arrival_s;
    in_len[i] = reqs[i].input_len;
    out_len[i] = reqs[i].output_len;
  }
  return count;
}

// --- placement search oracles (proj/tests/oracles) ---------------------------

// random_cluster (random_cluster.hpp:22-86) with AC2's parameters
// (acceptance_main.cpp:306-310): returns the reference's serialize_cluster
// JSON into buf; -needed size if buf is too small.
int refh_random_cluster_json(uint64_t seed, int max_nodes, int min_layers, int max_layers, char* buf,
                             int buflen) {
  testutil::RandomClusterParams params;
  params.max_nodes = max_nodes;
  params.min_layers = min_layers;
  params.max_layers = max_layers;
  Rng rng(seed);
  ClusterSpec c = testutil::random_cluster(rng, params);
  std::string s = serialize_cluster(c);
  if (static_cast<int>(s.size()) + 1 > buflen) return -static_cast<int>(s.size() + 1);
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

// best_placement_exhaustive (enumerate.hpp:14-77): best value, the winning
// placement as an int16 [N][2] row, and the number of leaves scored.
double refh_best_exhaustive(void* cp, int allow_partial, int16_t* best_row, int64_t* scored) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  Placement best;
  long n = 0;
  double v = testutil::best_placement_exhaustive(c, allow_partial != 0, &best, &n);
  for (size_t k = 0; k < c.nodes.size(); ++k) {
    auto it = best.find(c.nodes[k].id);
    best_row[2 * k] = it == best.end() ? 0 : static_cast<int16_t>(it->second.start);
    best_row[2 * k + 1] = it == best.end() ? 0 : static_cast<int16_t>(it->second.end);
  }
  *scored = n;
  return v;
}

// swarm_placement / petals_placement / separate_pipelines_placement
// (heuristics.cpp:12-131), method 0 / 1 / 2: the placement as an int16 [N][2]
// row and the warnings joined by newlines.  Returns the number of warnings,
// or -1 with the exception text in `warn` when the heuristic throws.
int refh_heuristic(void* cp, int method, int16_t* row, char* warn, int warnlen) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  try {
    HeuristicResult h = method == 0 ? swarm_placement(c) : method == 1 ? petals_placement(c)
                                                                       : separate_pipelines_placement(c);
    for (size_t k = 0; k < c.nodes.size(); ++k) {
      auto it = h.placement.find(c.nodes[k].id);
      row[2 * k] = it == h.placement.end() ? 0 : static_cast<int16_t>(it->second.start);
      row[2 * k + 1] = it == h.placement.end() ? 0 : static_cast<int16_t>(it->second.end);
    }
    std::string all;
    for (size_t i = 0; i < h.warnings.size(); ++i) all += (i ? "\n" : "") + h.warnings[i];
    set_err(warn, warnlen, all);
    return static_cast<int>(h.warnings.size());
  } catch (const std::exception& e) {
    set_err(warn, warnlen, e.what());
    return -1;
  }
}

// --- plan / report formats, stateful scheduler, simulator, pruning ------------

namespace {
int put_text(const std::string& s, char* buf, int buflen) {
  if (static_cast<int>(s.size()) + 1 > buflen) return -static_cast<int>(s.size() + 1);
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}
}  // namespace

// serialize_plan(plan_from_placement(c, row)) (placement.cpp:459-469, :603-625).
int refh_plan_json(void* cp, const int16_t* pl, int allow_partial, const char* method, char* buf, int buflen) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  try {
    return put_text(serialize_plan(plan_from_placement(c, to_placement(c, pl), allow_partial != 0, method)), buf,
                    buflen);
  } catch (const std::exception& e) {
    set_err(buf, buflen, e.what());
    return -1000000000;
  }
}

// serialize_plan(parse_plan(text)) (placement.cpp:603-658): the reference
// reading a plan written elsewhere and writing it back.
int refh_plan_roundtrip(const char* text, char* buf, int buflen) {
  try {
    return put_text(serialize_plan(parse_plan(text, "<refh>")), buf, buflen);
  } catch (const std::exception& e) {
    set_err(buf, buflen, e.what());
    return -1000000000;
  }
}

// to_dot after max_flow (flow_graph.cpp:257-271), and the min-cut source side
// (:231-255) as vertex ids.
int refh_to_dot(void* cp, const int16_t* pl, int allow_partial, char* buf, int buflen, int32_t* cut, int* ncut) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  try {
    FlowGraph g = build_flow_graph(c, to_placement(c, pl), allow_partial != 0);
    max_flow(g);
    std::vector<int> side = min_cut_source_side(g);
    *ncut = static_cast<int>(side.size());
    for (size_t i = 0; i < side.size(); ++i) cut[i] = side[i];
    return put_text(to_dot(g), buf, buflen);
  } catch (const std::exception& e) {
    set_err(buf, buflen, e.what());
    return -1000000000;
  }
}

// A stateful Scheduler driven by an op list: op k = (kind[k], id[k], len[k]),
// kind 0 = admit(id, len), 1 = complete(id, len) — skipped (nh[k] = -2) when
// that id's admit was deferred, as the simulator only completes admitted
// requests.  For every admit the hop
// count (-1 = deferred) goes to nh[k] and the hops to hop_node/s/e at stride
// max_hops; kv[k] = kv_estimate of node `probe` after the op, avg[k] =
// avg_output().  Returns 0, or -1 with the exception text in err.
int refh_sched_ops(void* cp, const int16_t* pl, int allow_partial, uint64_t seed, int64_t K, const int32_t* kind,
                   const int64_t* id, const int32_t* len, int max_hops, int32_t* nh, int32_t* hop_node,
                   int32_t* hop_s, int32_t* hop_e, const char* probe, double* kv, double* avg, char* err,
                   int errlen) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  try {
    PlacementPlan plan = plan_from_placement(c, to_placement(c, pl), allow_partial != 0, "custom");
    Scheduler sched(c, plan, SchedPolicy::kIwrr, seed);
    std::vector<char> admitted;
    for (int64_t k = 0; k < K; ++k) {
      nh[k] = 0;
      if (id[k] >= static_cast<int64_t>(admitted.size())) admitted.resize(id[k] + 1, 0);
      if (kind[k] == 0) {
        auto r = sched.admit(static_cast<long>(id[k]), len[k]);
        if (!r) {
          nh[k] = -1;
        } else {
          admitted[id[k]] = 1;
          nh[k] = static_cast<int32_t>(r->size());
          for (int h = 0; h < nh[k] && h < max_hops; ++h) {
            hop_node[k * max_hops + h] = c.node_index((*r)[h].node);
            hop_s[k * max_hops + h] = (*r)[h].exec_start;
            hop_e[k * max_hops + h] = (*r)[h].exec_end;
          }
        }
      } else if (admitted[id[k]]) {
        sched.complete(static_cast<long>(id[k]), len[k]);
      } else {
        nh[k] = -2;
      }
      kv[k] = sched.kv_estimate(probe);
      avg[k] = sched.avg_output();
    }
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return -1;
  }
}

// simulate(c, plan_from_placement(c, row), trace, cfg) (sim.cpp:382-388); the
// metrics go out as the reference binding's dict keys (pymodule.cpp:34-74),
// JSON, doubles at full precision.
int refh_simulate(void* cp, const int16_t* pl, int allow_partial, int64_t n, const double* arrival,
                  const int32_t* in_len, const int32_t* out_len, int online, int policy, uint64_t seed,
                  double horizon_s, double warmup_s, char* buf, int buflen) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  try {
    PlacementPlan plan = plan_from_placement(c, to_placement(c, pl), allow_partial != 0, "custom");
    std::vector<Request> reqs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) reqs[i] = {arrival[i], in_len[i], out_len[i]};
    SimConfig cfg;
    cfg.mode = online ? TraceMode::kOnline : TraceMode::kOffline;
    cfg.policy = policy == 0 ? SchedPolicy::kIwrr : policy == 1 ? SchedPolicy::kRandom
                 : policy == 2 ? SchedPolicy::kSqf : SchedPolicy::kSwarm;
    cfg.seed = seed;
    cfg.horizon_s = horizon_s;
    cfg.warmup_s = online ? warmup_s : 0;
    SimMetrics m = simulate(c, plan, reqs, cfg);
    nlohmann::ordered_json d;
    d["window_s"] = m.window_s;
    d["requests_arrived"] = m.requests_arrived;
    d["requests_completed"] = m.requests_completed;
    d["requests_completed_total"] = m.requests_completed_total;
    d["throughput_tps"] = m.throughput_tps;
    d["output_tps"] = m.output_tps;
    d["latency_mean_s"] = m.latency_mean_s;
    d["latency_p50_s"] = m.latency_p50_s;
    d["latency_p95_s"] = m.latency_p95_s;
    d["latency_max_s"] = m.latency_max_s;
    d["ttft_mean_s"] = m.ttft_mean_s;
    d["ttft_p95_s"] = m.ttft_p95_s;
    d["deferrals"] = m.deferrals;
    d["nodes"] = nlohmann::ordered_json::array();
    for (const NodeStats& x : m.nodes)
      d["nodes"].push_back({{"id", x.id}, {"utilization", x.utilization}, {"batches", x.batches},
                            {"layer_tokens", x.layer_tokens}, {"kv_pages", x.kv_pages}});
    d["links"] = nlohmann::ordered_json::array();
    for (const LinkStats& l : m.links)
      d["links"].push_back({{"src", l.src}, {"dst", l.dst}, {"bytes", l.bytes}, {"transfers", l.transfers},
                            {"queue_delay_mean_s", l.queue_delay_mean_s},
                            {"queue_delay_max_s", l.queue_delay_max_s}});
    d["warnings"] = m.warnings;
    return put_text(d.dump(), buf, buflen);
  } catch (const std::exception& e) {
    set_err(buf, buflen, e.what());
    return -1000000000;
  }
}

// serialize_cluster(prune_links(c, degree)) (placement.cpp:230-332,
// cluster.cpp:191-228).
int refh_prune_json(void* cp, double degree, char* buf, int buflen, int* removed) {
  const ClusterSpec& c = *static_cast<ClusterSpec*>(cp);
  try {
    PruneReport rep;
    ClusterSpec p = prune_links(c, degree, &rep);
    *removed = rep.links_removed;
    return put_text(serialize_cluster(p), buf, buflen);
  } catch (const std::exception& e) {
    set_err(buf, buflen, e.what());
    return -1000000000;
  }
}

}  // extern "C"

#define HARNESS_FN(x) refh_##x
#include "milp_harness.inc"
