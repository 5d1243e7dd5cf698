// shim.cpp — the reference's C++ API (namespace helio) over the C ABI.
//
// Same names, argument meaning and error behaviour as the reference
// (proj/include/helio/*.hpp); every graph is built and solved by the B200
// engine (include/helio_gpu.h).  There is no host implementation of
// build_flow_graph, max_flow, plan_from_placement or routing here: if the
// engine cannot be created (no B200) every call throws InternalError.
#include "shim.hpp"

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

// --- cluster model (cluster.cpp:56-100, 237-300) ----------------------------

int ClusterSpec::node_index(const std::string& id) const {
  for (size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].id == id) return static_cast<int>(i);
  return -1;
}

int ClusterSpec::max_layers(const NodeSpec& n) const {
  const double usable = n.vram_bytes * (1.0 - n.kv_reserve);
  int k = static_cast<int>(std::floor(usable / model.bytes_per_layer()));
  if (!n.throughput_table.empty()) k = std::min(k, n.throughput_table.rbegin()->first);
  return std::min(k, model.num_layers);
}

double ClusterSpec::throughput(const NodeSpec& n, int j) const {
  if (j < 1 || j > max_layers(n))
    throw ValidationError("throughput request for node '" + n.id + "' outside profile range: j=" +
                          std::to_string(j));
  if (!n.throughput_table.empty()) return n.throughput_table.at(j);
  return n.peak_layer_tokens / j;
}

double ClusterSpec::layer_token_rate(const NodeSpec& n, int j) const { return j * throughput(n, j); }

static double incident_bw(const ClusterSpec& c, const NodeSpec& n) {
  double best = 0;
  for (const auto& l : c.links)
    if (l.src == n.id || l.dst == n.id) best = std::max(best, l.bandwidth_bps);
  return best;
}

double ClusterSpec::nic_in(const NodeSpec& n) const {
  return n.nic_in_bps > 0 ? n.nic_in_bps : incident_bw(*this, n);
}

double ClusterSpec::nic_out(const NodeSpec& n) const {
  return n.nic_out_bps > 0 ? n.nic_out_bps : incident_bw(*this, n);
}

double link_token_capacity(const LinkSpec& link, double payload_bytes) {
  return link.bandwidth_bps / (8.0 * payload_bytes);
}

void validate_cluster(const ClusterSpec& c) {
  auto fail = [](const std::string& msg) { throw ValidationError(msg); };
  if (c.model.num_layers < 1) fail("model.num_layers must be >= 1");
  if (c.model.param_bytes <= 0) fail("model.param_gb must be > 0");
  if (c.model.token_bytes <= 0) fail("model.token_bytes must be > 0");
  if (c.model.activation_bytes <= 0) fail("model.activation_bytes must be > 0");
  if (c.model.kv_bytes_per_token_layer < 0) fail("model.kv_bytes_per_token_layer must be >= 0");
  if (c.coordinator_id.empty()) fail("coordinator.id must be non-empty");
  if (c.nodes.empty()) fail("cluster needs at least one compute node");
  std::set<std::string> ids;
  for (const auto& n : c.nodes) {
    if (n.id.empty()) fail("node id must be non-empty");
    if (n.id == c.coordinator_id) fail("node id '" + n.id + "' collides with the coordinator");
    if (!ids.insert(n.id).second) fail("duplicate node id '" + n.id + "'");
    if (n.vram_bytes <= 0) fail("node '" + n.id + "': vram_gb must be > 0");
    if (n.kv_reserve < 0 || n.kv_reserve >= 1) fail("node '" + n.id + "': kv_reserve must be in [0, 1)");
    const bool has_peak = n.peak_layer_tokens > 0;
    const bool has_table = !n.throughput_table.empty();
    if (has_peak == has_table)
      fail("node '" + n.id + "': exactly one of peak_layer_tokens_per_s or throughput_table required");
    if (has_table) {
      int expect = 1;
      double prev = 0;
      for (const auto& [j, v] : n.throughput_table) {
        if (j != expect) fail("node '" + n.id + "': throughput_table keys must be contiguous from 1");
        if (v <= 0) fail("node '" + n.id + "': throughput_table values must be > 0");
        if (expect > 1 && v >= prev) fail("node '" + n.id + "': throughput_table must be strictly decreasing");
        prev = v;
        ++expect;
      }
    }
    if (n.nic_in_bps < 0 || n.nic_out_bps < 0) fail("node '" + n.id + "': NIC rates must be >= 0");
  }
  std::set<std::pair<std::string, std::string>> pairs;
  bool coord_out = false, coord_in = false;
  for (const auto& l : c.links) {
    auto known = [&](const std::string& e) { return e == c.coordinator_id || c.node_index(e) >= 0; };
    if (!known(l.src)) fail("link endpoint '" + l.src + "' is not a declared node");
    if (!known(l.dst)) fail("link endpoint '" + l.dst + "' is not a declared node");
    if (l.src == l.dst) fail("self-link on '" + l.src + "'");
    if (!pairs.insert({l.src, l.dst}).second) fail("duplicate link " + l.src + " -> " + l.dst);
    if (l.bandwidth_bps <= 0) fail("link " + l.src + " -> " + l.dst + ": bandwidth must be > 0");
    if (l.latency_s < 0) fail("link " + l.src + " -> " + l.dst + ": latency must be >= 0");
    if (l.src == c.coordinator_id) coord_out = true;
    if (l.dst == c.coordinator_id) coord_in = true;
  }
  if (!coord_out) fail("coordinator has no outgoing link");
  if (!coord_in) fail("coordinator has no incoming link");
  long total = 0;
  for (const auto& n : c.nodes) total += c.max_layers(n);
  if (total < c.model.num_layers)
    fail("insufficient VRAM: total layer capacity " + std::to_string(total) + " < model layers " +
         std::to_string(c.model.num_layers));
}

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

void put(std::string& k, const void* p, size_t n) { k.append(static_cast<const char*>(p), n); }
void put_d(std::string& k, double v) { put(k, &v, sizeof v); }
void put_s(std::string& k, const std::string& s) {
  size_t n = s.size();
  put(k, &n, sizeof n);
  k += s;
}

std::string cluster_key(const ClusterSpec& c) {
  std::string k;
  put_s(k, c.coordinator_id);
  int L = c.model.num_layers;
  put(k, &L, sizeof L);
  put_d(k, c.model.param_bytes);
  put_d(k, c.model.token_bytes);
  put_d(k, c.model.activation_bytes);
  put_d(k, c.model.kv_bytes_per_token_layer);
  for (const auto& n : c.nodes) {
    put_s(k, n.id);
    put_d(k, n.vram_bytes);
    put_d(k, n.kv_reserve);
    put_d(k, n.peak_layer_tokens);
    put_d(k, n.nic_in_bps);
    put_d(k, n.nic_out_bps);
    size_t t = n.throughput_table.size();
    put(k, &t, sizeof t);
    for (const auto& [j, v] : n.throughput_table) {
      put(k, &j, sizeof j);
      put_d(k, v);
    }
  }
  for (const auto& l : c.links) {
    put_s(k, l.src);
    put_s(k, l.dst);
    put_d(k, l.bandwidth_bps);
  }
  return k;
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

void Engine::set_cluster(const ClusterSpec& c) {
  const int N = static_cast<int>(c.nodes.size());
  std::set<std::string> seen;
  for (const auto& n : c.nodes)
    if (!seen.insert(n.id).second) throw ValidationError("duplicate node id '" + n.id + "'");
  std::vector<double> vram(N), kvr(N), peak(N), nin(N), nout(N), tval;
  std::vector<int32_t> toff(N + 1, 0), rank(N), lsrc, ldst;
  std::vector<double> lbw;
  bool any_table = false;
  for (int i = 0; i < N; ++i) {
    const NodeSpec& n = c.nodes[i];
    vram[i] = n.vram_bytes;
    kvr[i] = n.kv_reserve;
    peak[i] = n.peak_layer_tokens;
    nin[i] = n.nic_in_bps;
    nout[i] = n.nic_out_bps;
    toff[i] = static_cast<int32_t>(tval.size());
    if (!n.throughput_table.empty()) {
      any_table = true;
      int expect = 1;
      for (const auto& [j, v] : n.throughput_table) {
        if (j != expect) throw ValidationError("node '" + n.id + "': throughput_table keys must be contiguous from 1");
        tval.push_back(v);
        ++expect;
      }
    }
  }
  toff[N] = static_cast<int32_t>(tval.size());
  std::vector<int> order(N);
  for (int i = 0; i < N; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return c.nodes[a].id < c.nodes[b].id; });
  for (int r = 0; r < N; ++r) rank[order[r]] = r;
  std::map<std::string, int> idx;
  for (int i = 0; i < N; ++i) idx[c.nodes[i].id] = i;
  auto endpoint = [&](const std::string& id) {
    if (id == c.coordinator_id) return -1;
    auto it = idx.find(id);
    return it == idx.end() ? -2 : it->second;
  };
  for (const auto& l : c.links) {
    lsrc.push_back(endpoint(l.src));
    ldst.push_back(endpoint(l.dst));
    lbw.push_back(l.bandwidth_bps);
  }
  helio_cluster_desc d{};
  d.num_nodes = N;
  d.num_links = static_cast<int32_t>(c.links.size());
  d.num_layers = c.model.num_layers;
  d.param_bytes = c.model.param_bytes;
  d.token_bytes = c.model.token_bytes;
  d.activation_bytes = c.model.activation_bytes;
  d.kv_bytes_per_token_layer = c.model.kv_bytes_per_token_layer;
  d.vram_bytes = vram.data();
  d.kv_reserve = kvr.data();
  d.peak_layer_tokens = peak.data();
  d.nic_in_bps = nin.data();
  d.nic_out_bps = nout.data();
  d.table_off = any_table ? toff.data() : nullptr;
  d.table_val = any_table ? tval.data() : nullptr;
  d.lex_rank = rank.data();
  d.link_src = lsrc.data();
  d.link_dst = ldst.data();
  d.link_bandwidth_bps = lbw.data();
  kmax_.assign(N, 0);
  int rc = helio_gpu_set_cluster(ctx_, &d, kmax_.data());
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
  static std::list<std::pair<std::string, std::shared_ptr<Engine>>> cache;  // MRU first
  std::string key = cluster_key(c);
  std::lock_guard<std::mutex> lock(mu);
  for (auto it = cache.begin(); it != cache.end(); ++it)
    if (it->first == key) {
      cache.splice(cache.begin(), cache, it);
      return cache.front().second;
    }
  auto eng = std::make_shared<Engine>(default_device());
  eng->set_cluster(c);
  cache.emplace_front(std::move(key), eng);
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

namespace {

struct Solved {
  int nv = 0;
  double value = 0;
  std::vector<helio_edge> edges;
};

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

}  // namespace

// --- flow graph API ---------------------------------------------------------

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
  return g;
}

double max_flow(FlowGraph& g) {
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

// --- plans (placement.cpp:440-469) -------------------------------------------

PlacementPlan plan_from_placement(const ClusterSpec& c, const Placement& p, bool allow_partial,
                                  const std::string& method) {
  PlacementPlan plan;
  plan.method = method;
  plan.placement = p;
  plan.allow_partial = allow_partial;
  plan.status = MilpStatus::kFeasible;
  Solved s = solve_one(c, p, allow_partial);
  for (const helio_edge& e : s.edges) {
    if (e.kind == HELIO_EDGE_COMPUTE || e.flow <= 1e-9) continue;
    PlanEdge pe;
    pe.src = node_name(c, e.kind == HELIO_EDGE_COORD_OUT ? -1 : e.src_node);
    pe.dst = node_name(c, e.kind == HELIO_EDGE_COORD_IN ? -1 : e.dst_node);
    pe.flow = e.flow;
    pe.exec_start = e.exec_start;
    pe.exec_end = e.exec_end;
    plan.edges.push_back(pe);
  }
  plan.objective = s.value;
  plan.best_bound = plan.objective;
  return plan;
}

// --- IWRR (scheduler.cpp:28-190) ----------------------------------------------

std::vector<long> iwrr_weights(const std::vector<double>& flows) {
  std::vector<int64_t> w(flows.size());
  if (!flows.empty()) {
    auto eng = gpu::raw_engine();
    eng->check(helio_gpu_iwrr_weights(eng->ctx(), flows.data(), static_cast<int32_t>(flows.size()), w.data()),
               "helio_gpu_iwrr_weights");
  }
  return std::vector<long>(w.begin(), w.end());
}

IwrrPicker::IwrrPicker(std::vector<long> weights) : weights_(std::move(weights)) {}

std::vector<int> IwrrPicker::next_batch(const std::vector<uint64_t>& masks) {
  const int n = static_cast<int>(weights_.size());
  const int words = (n + 63) / 64;
  const int calls = words ? static_cast<int>(masks.size()) / words : static_cast<int>(masks.size());
  std::vector<int32_t> out(calls, -1);
  if (calls == 0) return {};
  std::vector<int64_t> w(weights_.begin(), weights_.end());
  int64_t round = round_, idx = idx_;
  auto eng = gpu::raw_engine();
  eng->check(helio_gpu_iwrr_picks(eng->ctx(), w.data(), n, &round, &idx, calls, masks.data(), out.data()),
             "helio_gpu_iwrr_picks");
  round_ = static_cast<long>(round);
  idx_ = static_cast<long>(idx);
  return std::vector<int>(out.begin(), out.end());
}

int IwrrPicker::next(const std::function<bool(int)>& eligible) {
  const int n = static_cast<int>(weights_.size());
  if (n == 0) return -1;
  std::vector<uint64_t> mask((n + 63) / 64, 0);
  for (int i = 0; i < n; ++i)
    if (eligible(i)) mask[i >> 6] |= 1ull << (i & 63);
  return next_batch(mask)[0];
}

Scheduler::Scheduler(const ClusterSpec& c, const PlacementPlan& plan) : cluster_(c), plan_(plan) {
  if (plan.edges.empty()) throw ValidationError("plan has no flow edges to schedule on");
  for (const auto& [id, iv] : plan.placement)
    if (!iv.empty() && c.node_index(id) < 0) throw ValidationError("plan references unknown node '" + id + "'");
  bool coord_out = false;
  for (const PlanEdge& e : plan.edges) {
    auto placed = [&](const std::string& id) {
      if (id == c.coordinator_id) return true;
      auto it = plan.placement.find(id);
      return it != plan.placement.end() && !it->second.empty();
    };
    if (!placed(e.src) || !placed(e.dst))
      throw ValidationError("plan edge " + e.src + "->" + e.dst + " references an unplaced node");
    if (e.src == c.coordinator_id) coord_out = true;
  }
  if (!coord_out) throw ValidationError("plan has no edge leaving the coordinator");
}

std::vector<std::optional<std::vector<RouteHop>>> Scheduler::route(const std::vector<int>& in,
                                                                    const std::vector<int>& out) {
  if (in.size() != out.size()) throw ValidationError("input/output length arrays differ in size");
  const ClusterSpec& c = cluster_;
  auto eng = gpu::engine_for(c);
  std::vector<int16_t> row(2 * c.nodes.size(), 0);
  for (const auto& [id, iv] : plan_.placement) {
    if (iv.empty()) continue;
    int idx = c.node_index(id);
    row[2 * idx] = static_cast<int16_t>(iv.start);
    row[2 * idx + 1] = static_cast<int16_t>(iv.end);
  }
  std::vector<helio_plan_edge> pe;
  for (const PlanEdge& e : plan_.edges) {
    helio_plan_edge x{};
    x.src_node = e.src == c.coordinator_id ? -1 : c.node_index(e.src);
    x.dst_node = e.dst == c.coordinator_id ? -1 : c.node_index(e.dst);
    x.exec_start = e.exec_start;
    x.exec_end = e.exec_end;
    x.flow = e.flow;
    pe.push_back(x);
  }
  const int64_t R = static_cast<int64_t>(in.size());
  const int max_hops = c.model.num_layers;
  std::vector<int32_t> nh(R), hn((size_t)R * max_hops), hs((size_t)R * max_hops), he((size_t)R * max_hops);
  int64_t deferred = 0;
  int rc = helio_gpu_route_host(eng->ctx(), row.data(), pe.data(), static_cast<int32_t>(pe.size()), R, in.data(),
                                out.data(), max_hops, nh.data(), hn.data(), hs.data(), he.data(), &deferred);
  if (rc == HELIO_ERR_INVALID) throw InternalError(helio_gpu_last_error(eng->ctx()));
  eng->check(rc, "helio_gpu_route_host");
  std::vector<std::optional<std::vector<RouteHop>>> routes(R);
  for (int64_t r = 0; r < R; ++r) {
    if (nh[r] < 0) continue;
    std::vector<RouteHop> hops;
    for (int k = 0; k < nh[r]; ++k) {
      size_t at = (size_t)r * max_hops + k;
      hops.push_back({c.nodes[hn[at]].id, hs[at], he[at]});
    }
    routes[r] = std::move(hops);
  }
  return routes;
}

}  // namespace helio
