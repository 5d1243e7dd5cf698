// shim_flow.cpp — engine cache, placement validation and the flow-graph API
// (flow_graph.hpp:43-55) over the C ABI.  No host implementation of
// build_flow_graph or max_flow exists: every graph is built and solved by the
// B200 engine, and without one every call throws InternalError.
#include "shim_engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <list>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>

#include "helio/errors.hpp"

namespace helio {

// --- engine cache -----------------------------------------------------------

namespace gpu {

namespace {

int default_device() {
  const char* d = std::getenv("HELIO_DEVICE");
  return d ? std::atoi(d) : 0;
}

[[noreturn]] void engine_fail(helio_gpu_ctx* ctx, int rc, const std::string& what) {
  std::string msg = what + " failed (" + std::to_string(rc) + ")";
  if (ctx) msg += ": " + std::string(helio_gpu_last_error(ctx));
  if (rc == HELIO_ERR_INVALID) throw ValidationError(msg);
  throw InternalError(msg);
}

// Content fingerprint of a cluster: two independent 64-bit FNV-1a-style
// streams over every field the engine compiles (model, nodes, links), hashed
// in place — no per-call string building (the reference's per-call cost is
// exactly this kind of O(links) string work, cluster.cpp:82-96).
struct Fingerprint {
  uint64_t a = 1469598103934665603ull, b = 0x9E3779B97F4A7C15ull;
  // eight bytes per step (a byte-wise loop cost ~100 us per call on het42's
  // 1,806 links — most of the per-call host time)
  void word(uint64_t w) {
    a = (a ^ w) * 0x100000001B3ull;
    a ^= a >> 31;
    b = (b + w) * 0xBF58476D1CE4E5B9ull;
    b ^= b >> 29;
  }
  void bytes(const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w;
      std::memcpy(&w, c + i, 8);
      word(w);
    }
    if (i < n) {
      uint64_t w = 0;
      std::memcpy(&w, c + i, n - i);
      word(w ^ (uint64_t)(n - i) << 56);
    }
  }
  void d(double v) { bytes(&v, sizeof v); }
  void i(int64_t v) { bytes(&v, sizeof v); }
  void s(const std::string& x) {
    i(static_cast<int64_t>(x.size()));
    bytes(x.data(), x.size());
  }
  bool operator==(const Fingerprint& o) const { return a == o.a && b == o.b; }
};

Fingerprint cluster_fingerprint(const ClusterSpec& c) {
  Fingerprint f;
  f.s(c.coordinator_id);
  f.i(c.model.num_layers);
  f.d(c.model.param_bytes);
  f.d(c.model.token_bytes);
  f.d(c.model.activation_bytes);
  f.d(c.model.kv_bytes_per_token_layer);
  f.i(static_cast<int64_t>(c.nodes.size()));
  for (const auto& n : c.nodes) {
    f.s(n.id);
    f.d(n.vram_bytes);
    f.d(n.kv_reserve);
    f.d(n.peak_layer_tokens);
    f.d(n.nic_in_bps);
    f.d(n.nic_out_bps);
    f.i(static_cast<int64_t>(n.throughput_table.size()));
    for (const auto& [j, v] : n.throughput_table) {
      f.i(j);
      f.d(v);
    }
  }
  f.i(static_cast<int64_t>(c.links.size()));
  for (const auto& l : c.links) {
    f.s(l.src);
    f.s(l.dst);
    f.d(l.bandwidth_bps);
  }
  return f;
}

}  // namespace

Engine::Engine(int device) : device_(device) {
  int rc = helio_gpu_create(device, &ctx_);
  if (rc != HELIO_OK)
    throw InternalError("helio: cannot create the B200 engine on device " + std::to_string(device) +
                        " (helio_gpu_create returned " + std::to_string(rc) +
                        "); this build has no CPU fallback");
}

Engine::~Engine() { helio_gpu_destroy(ctx_); }

void make_cluster_desc(const ClusterSpec& c, ClusterDesc& out) {
  const int N = static_cast<int>(c.nodes.size());
  std::set<std::string> seen;
  for (const auto& n : c.nodes)
    if (!seen.insert(n.id).second) throw ValidationError("duplicate node id '" + n.id + "'");
  out = ClusterDesc{};
  out.vram.resize(N);
  out.kvr.resize(N);
  out.peak.resize(N);
  out.nin.resize(N);
  out.nout.resize(N);
  out.toff.assign(N + 1, 0);
  out.rank.resize(N);
  bool any_table = false;
  for (int i = 0; i < N; ++i) {
    const NodeSpec& n = c.nodes[i];
    out.vram[i] = n.vram_bytes;
    out.kvr[i] = n.kv_reserve;
    out.peak[i] = n.peak_layer_tokens;
    out.nin[i] = n.nic_in_bps;
    out.nout[i] = n.nic_out_bps;
    out.toff[i] = static_cast<int32_t>(out.tval.size());
    if (!n.throughput_table.empty()) {
      any_table = true;
      int expect = 1;
      for (const auto& [j, v] : n.throughput_table) {
        if (j != expect) throw ValidationError("node '" + n.id + "': throughput_table keys must be contiguous from 1");
        out.tval.push_back(v);
        ++expect;
      }
    }
  }
  out.toff[N] = static_cast<int32_t>(out.tval.size());
  std::vector<int> order(N);
  for (int i = 0; i < N; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return c.nodes[a].id < c.nodes[b].id; });
  for (int r = 0; r < N; ++r) out.rank[order[r]] = r;
  std::map<std::string, int> idx;
  for (int i = 0; i < N; ++i) idx[c.nodes[i].id] = i;
  auto endpoint = [&](const std::string& id) {
    if (id == c.coordinator_id) return -1;
    auto it = idx.find(id);
    return it == idx.end() ? -2 : it->second;
  };
  for (const auto& l : c.links) {
    out.lsrc.push_back(endpoint(l.src));
    out.ldst.push_back(endpoint(l.dst));
    out.lbw.push_back(l.bandwidth_bps);
  }
  helio_cluster_desc& d = out.d;
  d.num_nodes = N;
  d.num_links = static_cast<int32_t>(c.links.size());
  d.num_layers = c.model.num_layers;
  d.param_bytes = c.model.param_bytes;
  d.token_bytes = c.model.token_bytes;
  d.activation_bytes = c.model.activation_bytes;
  d.kv_bytes_per_token_layer = c.model.kv_bytes_per_token_layer;
  d.vram_bytes = out.vram.data();
  d.kv_reserve = out.kvr.data();
  d.peak_layer_tokens = out.peak.data();
  d.nic_in_bps = out.nin.data();
  d.nic_out_bps = out.nout.data();
  d.table_off = any_table ? out.toff.data() : nullptr;
  d.table_val = any_table ? out.tval.data() : nullptr;
  d.lex_rank = out.rank.data();
  d.link_src = out.lsrc.data();
  d.link_dst = out.ldst.data();
  d.link_bandwidth_bps = out.lbw.data();
}

void Engine::set_cluster(const ClusterSpec& c) {
  const int N = static_cast<int>(c.nodes.size());
  ClusterDesc desc;
  make_cluster_desc(c, desc);
  kmax_.assign(N, 0);
  int rc = helio_gpu_set_cluster(ctx_, &desc.d, kmax_.data());
  if (rc != HELIO_OK) engine_fail(ctx_, rc, "helio_gpu_set_cluster");
  N_ = N;
  ids_.clear();
  for (const auto& n : c.nodes) ids_.push_back(n.id);
  coordinator_ = c.coordinator_id;
  num_layers_ = c.model.num_layers;
  num_links_ = static_cast<int>(c.links.size());
}

void Engine::check(int rc, const char* what) const {
  if (rc != HELIO_OK) engine_fail(ctx_, rc, what);
}

std::shared_ptr<Engine> engine_for(const ClusterSpec& c) {
  static std::mutex mu;
  static std::list<std::pair<Fingerprint, std::shared_ptr<Engine>>> cache;  // MRU first
  const Fingerprint key = cluster_fingerprint(c);
  std::lock_guard<std::mutex> lock(mu);
  for (auto it = cache.begin(); it != cache.end(); ++it)
    if (it->first == key) {
      cache.splice(cache.begin(), cache, it);
      return cache.front().second;
    }
  auto eng = std::make_shared<Engine>(default_device());
  eng->set_cluster(c);
  cache.emplace_front(key, eng);
  while (cache.size() > 8) cache.pop_back();
  return eng;
}

std::shared_ptr<Engine> raw_engine() {
  static std::mutex mu;
  static std::shared_ptr<Engine> eng;
  std::lock_guard<std::mutex> lock(mu);
  if (!eng) eng = std::make_shared<Engine>(default_device());
  return eng;
}

}  // namespace gpu

// --- placement validation (flow_graph.cpp:52-61) and row conversion ----------

std::vector<int16_t> placement_row(const ClusterSpec& c, const Placement& p) {
  const int L = c.model.num_layers;
  std::vector<int16_t> row(2 * c.nodes.size(), 0);
  for (const auto& [id, iv] : p) {
    if (iv.empty()) continue;
    const int idx = c.node_index(id);
    if (idx < 0) throw ValidationError("placement references unknown node '" + id + "'");
    if (iv.start < 0 || iv.end > L)
      throw ValidationError("placement for '" + id + "' outside [0, " + std::to_string(L) + ")");
    if (iv.len() > c.max_layers(c.nodes[idx]))
      throw ValidationError("placement for '" + id + "' exceeds its VRAM layer capacity");
    row[2 * idx] = static_cast<int16_t>(iv.start);
    row[2 * idx + 1] = static_cast<int16_t>(iv.end);
  }
  return row;
}

namespace detail {

Solved solve_one(const ClusterSpec& c, const Placement& p, bool allow_partial) {
  std::vector<int16_t> row = placement_row(c, p);
  auto eng = gpu::engine_for(c);
  int32_t max_e = static_cast<int32_t>(c.nodes.size() + c.links.size() + 1);
  Solved s;
  s.edges.resize(max_e);
  int32_t nv = 0, ne = 0, st = 0;
  double val = 0;
  eng->check(helio_gpu_flows_host(eng->ctx(), row.data(), 1, allow_partial ? 1 : 0, max_e, &nv, &ne,
                                  s.edges.data(), &val, &st),
             "helio_gpu_flows_host");
  if (st != HELIO_CAND_OK) throw InternalError("engine rejected a validated placement (status " + std::to_string(st) + ")");
  s.edges.resize(ne);
  s.nv = nv;
  s.value = val;
  return s;
}

const std::string& node_name(const ClusterSpec& c, int idx) {
  return idx < 0 ? c.coordinator_id : c.nodes[idx].id;
}

}  // namespace detail

using detail::node_name;
using detail::solve_one;
using detail::Solved;

// --- flow graph API ---------------------------------------------------------

namespace {

// build_flow_graph runs the PARITY build + solve on the device in one call
// (helio_gpu_flows_host), which already yields the reference's per-edge
// flows.  The reference's API hands the graph back with zero flows and solves
// it in max_flow; instead of solving twice, the last few solved graphs of this
// thread are remembered by the fingerprint of exactly what max_flow reads
// (vertex count, source, sink, every edge's u, v, cap).  A graph the caller
// changed in between misses and is solved on the device as a raw graph —
// bit-identical either way, since both paths replay the reference's FIFO
// discharge (flow_graph.cpp:138-229).
struct SolvedGraph {
  uint64_t a = 0, b = 0;
  double value = 0;
  std::vector<double> flows;
};

void graph_fingerprint(const FlowGraph& g, uint64_t& a, uint64_t& b) {
  gpu::Fingerprint f;
  f.i(g.num_vertices);
  f.i(g.source);
  f.i(g.sink);
  f.i(static_cast<int64_t>(g.edges.size()));
  for (const FlowEdge& e : g.edges) {
    f.i(e.u);
    f.i(e.v);
    f.d(e.cap);
  }
  a = f.a;
  b = f.b;
}

thread_local std::deque<SolvedGraph> t_solved;  // most recent first, at most 4

}  // namespace

FlowGraph build_flow_graph(const ClusterSpec& c, const Placement& p, bool allow_partial) {
  Solved s = solve_one(c, p, allow_partial);
  FlowGraph g;
  g.num_vertices = s.nv;
  g.vertex_names = {"source", "sink"};
  g.vertex_names.resize(s.nv);
  for (const helio_edge& e : s.edges) {
    FlowEdge fe;
    fe.u = e.u;
    fe.v = e.v;
    fe.cap = e.cap;
    fe.flow = 0;  // flows are filled by max_flow
    fe.kind = static_cast<EdgeKind>(e.kind);
    fe.src_id = node_name(c, e.src_node);
    fe.dst_id = node_name(c, e.dst_node);
    fe.exec_start = e.exec_start;
    fe.exec_end = e.exec_end;
    if (fe.kind == EdgeKind::kCompute) {
      g.vertex_names[e.u] = "in:" + fe.src_id;
      g.vertex_names[e.v] = "out:" + fe.src_id;
      g.node_vertices[fe.src_id] = {e.u, e.v};
    }
    g.edges.push_back(std::move(fe));
  }
  SolvedGraph sg;
  graph_fingerprint(g, sg.a, sg.b);
  sg.value = s.value;
  sg.flows.reserve(s.edges.size());
  for (const helio_edge& e : s.edges) sg.flows.push_back(e.flow);
  t_solved.push_front(std::move(sg));
  if (t_solved.size() > 4) t_solved.pop_back();
  return g;
}

double max_flow(FlowGraph& g) {
  uint64_t fa = 0, fb = 0;
  graph_fingerprint(g, fa, fb);
  for (const SolvedGraph& sg : t_solved)
    if (sg.a == fa && sg.b == fb && sg.flows.size() == g.edges.size()) {
      for (size_t i = 0; i < g.edges.size(); ++i) g.edges[i].flow = sg.flows[i];
      return sg.value;
    }
  auto eng = gpu::raw_engine();
  const int64_t m = static_cast<int64_t>(g.edges.size());
  std::vector<int32_t> u(m), v(m);
  std::vector<double> cap(m), flow(m);
  for (int64_t i = 0; i < m; ++i) {
    u[i] = g.edges[i].u;
    v[i] = g.edges[i].v;
    cap[i] = g.edges[i].cap;
  }
  int32_t n = g.num_vertices, s = g.source, t = g.sink;
  int64_t off[2] = {0, m};
  double value = 0;
  eng->check(helio_gpu_maxflow_raw_host(eng->ctx(), 1, &n, &s, &t, off, u.data(), v.data(), cap.data(),
                                        &value, flow.data()),
             "helio_gpu_maxflow_raw_host");
  for (int64_t i = 0; i < m; ++i) g.edges[i].flow = flow[i];
  return value;
}

// min_cut_source_side / to_dot: post-solve reports over the flows the device
// computed (flow_graph.cpp:231-271).
std::vector<int> min_cut_source_side(const FlowGraph& g) {
  const int n = g.num_vertices;
  std::vector<std::vector<std::pair<int, double>>> res(n);
  for (const FlowEdge& e : g.edges) {
    res[e.u].push_back({e.v, e.cap - e.flow});
    res[e.v].push_back({e.u, e.flow});
  }
  std::vector<char> seen(n, 0);
  std::deque<int> q{g.source};
  seen[g.source] = 1;
  while (!q.empty()) {
    int x = q.front();
    q.pop_front();
    for (auto [y, r] : res[x])
      if (r > 1e-12 && !seen[y]) {
        seen[y] = 1;
        q.push_back(y);
      }
  }
  std::vector<int> side;
  for (int x = 0; x < n; ++x)
    if (seen[x]) side.push_back(x);
  return side;
}

std::string to_dot(const FlowGraph& g) {
  std::ostringstream os;
  os << "digraph flow {\n  rankdir=LR;\n";
  for (int x = 0; x < g.num_vertices; ++x) os << "  v" << x << " [label=\"" << g.vertex_names[x] << "\"];\n";
  os.setf(std::ios::fixed);
  os.precision(3);
  for (const FlowEdge& e : g.edges) {
    os << "  v" << e.u << " -> v" << e.v << " [label=\"" << e.flow << "/" << e.cap;
    if (e.kind == EdgeKind::kCompute) os << " [" << e.exec_start << "," << e.exec_end << ")";
    os << "\"];\n";
  }
  os << "}\n";
  return os.str();
}

double compute_edge_capacity(const ClusterSpec& c, const NodeSpec& n, int j) {
  if (j < 1 || j > c.max_layers(n))
    throw ValidationError("throughput request for node '" + n.id + "' outside profile range: j=" +
                          std::to_string(j));
  // Locate n in c; a NodeSpec that is not c's own is compiled into a copy.
  int idx = -1;
  for (size_t i = 0; i < c.nodes.size(); ++i)
    if (&c.nodes[i] == &n) idx = static_cast<int>(i);
  const ClusterSpec* cc = &c;
  ClusterSpec tmp;
  if (idx < 0) {
    tmp = c;
    idx = tmp.node_index(n.id);
    if (idx < 0) {
      tmp.nodes.push_back(n);
      idx = static_cast<int>(tmp.nodes.size()) - 1;
    } else {
      tmp.nodes[idx] = n;
    }
    cc = &tmp;
  }
  auto eng = gpu::engine_for(*cc);
  double out = 0;
  eng->check(helio_gpu_compute_edge_capacity(eng->ctx(), idx, j, &out), "helio_gpu_compute_edge_capacity");
  return out;
}

}  // namespace helio
