// shim_sched.cpp — iwrr_weights / IwrrPicker / Scheduler / route_requests
// (proj/src/scheduler.cpp:10-190) over the engine.
//
// * iwrr_weights and the IWRR cycles run on the device
//   (helio_gpu_iwrr_weights / helio_gpu_iwrr_cycles).  A picker walks its
//   cycle: the k-th unmasked pick is cycle[k mod W], a masked pick scans at
//   most one full cycle and leaves the position unchanged on failure — the
//   reference's (round, idx) walk (scheduler.cpp:28-44) without its empty
//   slots.
// * Scheduler::admit/complete keep the reference's KV arithmetic, charge
//   order, rollback and running output mean (scheduler.cpp:100-190).  The
//   scheduler is the reference's single serialised actor: each
//   admit depends on the previous completes, so it stays a host walk over the
//   device-built cycles — a device round trip per admit would cost ~10 us
//   against ~0.2 us.  Bulk routing of a request stream goes through
//   route_requests, which routes every request on the device (route.cu).
#include "shim.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "helio/errors.hpp"

namespace helio {

SchedPolicy sched_policy_from_str(const std::string& s) {
  if (s == "iwrr") return SchedPolicy::kIwrr;
  if (s == "random") return SchedPolicy::kRandom;
  if (s == "sqf") return SchedPolicy::kSqf;
  if (s == "swarm") return SchedPolicy::kSwarm;
  throw ValidationError("unknown scheduler policy '" + s + "' (expected iwrr, random, sqf, or swarm)");
}

std::string sched_policy_name(SchedPolicy p) {
  switch (p) {
    case SchedPolicy::kIwrr: return "iwrr";
    case SchedPolicy::kRandom: return "random";
    case SchedPolicy::kSqf: return "sqf";
    default: return "swarm";
  }
}

namespace {

// Cycles of several candidate lists in one device call.  flows != nullptr:
// weights = iwrr_weights(flows) (cycle <= 32 slots per candidate); otherwise
// the caller's weights.
std::vector<std::vector<long>> device_cycles(const std::vector<std::vector<double>>* flows,
                                             const std::vector<std::vector<long>>* weights) {
  const size_t L = flows ? flows->size() : weights->size();
  std::vector<int32_t> off(L + 1, 0);
  std::vector<int64_t> coff(L + 1, 0);
  std::vector<double> f;
  std::vector<int64_t> w;
  for (size_t l = 0; l < L; ++l) {
    const size_t n = flows ? (*flows)[l].size() : (*weights)[l].size();
    off[l + 1] = off[l] + static_cast<int32_t>(n);
    int64_t slots = 0;
    if (flows) {
      f.insert(f.end(), (*flows)[l].begin(), (*flows)[l].end());
      slots = 32 * static_cast<int64_t>(n);
    } else {
      for (long x : (*weights)[l]) {
        w.push_back(x);
        slots += x > 0 ? x : 0;
      }
    }
    coff[l + 1] = coff[l] + slots;
  }
  if (coff[L] > (int64_t(1) << 28)) throw ValidationError("IWRR weights too large (cycle over 2^28 slots)");
  if (flows) w.assign(off[L], 0);
  std::vector<int32_t> cyc(std::max<int64_t>(coff[L], 1));
  std::vector<int64_t> clen(L, 0);
  if (L > 0) {
    auto eng = gpu::raw_engine();
    eng->check(helio_gpu_iwrr_cycles(eng->ctx(), static_cast<int32_t>(L), off.data(), flows ? f.data() : nullptr,
                                     w.data(), coff.data(), cyc.data(), clen.data()),
               "helio_gpu_iwrr_cycles");
  }
  std::vector<std::vector<long>> out(L);
  for (size_t l = 0; l < L; ++l) out[l].assign(cyc.begin() + coff[l], cyc.begin() + coff[l] + clen[l]);
  return out;
}

}  // namespace

// --- IWRR (scheduler.cpp:22-56) ---------------------------------------------

std::vector<long> iwrr_weights(const std::vector<double>& flows) {
  std::vector<int64_t> w(flows.size());
  if (!flows.empty()) {
    auto eng = gpu::raw_engine();
    eng->check(helio_gpu_iwrr_weights(eng->ctx(), flows.data(), static_cast<int32_t>(flows.size()), w.data()),
               "helio_gpu_iwrr_weights");
  }
  return std::vector<long>(w.begin(), w.end());
}

IwrrPicker::IwrrPicker(std::vector<long> weights) {
  const std::vector<std::vector<long>> one{std::move(weights)};
  weights_ = std::move(device_cycles(nullptr, &one)[0]);
  wmax_ = static_cast<long>(weights_.size());
}

IwrrPicker::IwrrPicker(Cycle cycle) : weights_(std::move(cycle.slots)) { wmax_ = static_cast<long>(weights_.size()); }

int IwrrPicker::next(const std::function<bool(int)>& eligible) {
  const size_t W = weights_.size();
  for (size_t it = 0; it < W; ++it) {
    const size_t p = idx_;
    idx_ = idx_ + 1 == W ? 0 : idx_ + 1;
    if (eligible(static_cast<int>(weights_[p]))) return static_cast<int>(weights_[p]);
  }
  return -1;  // a full cycle: the position is back where it started
}

// --- Scheduler (scheduler.cpp:58-190) ----------------------------------------

Scheduler::Scheduler(const ClusterSpec& c, const PlacementPlan& plan, SchedPolicy policy, uint64_t seed)
    : cluster_(c), policy_(policy), rng_(seed), avg_output_(232.0) {
  if (policy != SchedPolicy::kIwrr)
    throw ValidationError("scheduler policy '" + sched_policy_name(policy) +
                          "' is not supported by the B200 engine (iwrr only: random/sqf/swarm read live "
                          "simulator probes on every pick)");
  if (plan.edges.empty()) throw ValidationError("plan has no flow edges to schedule on");
  vertex_id_.push_back(c.coordinator_id);
  vertex_of_[c.coordinator_id] = 0;
  for (const auto& [id, iv] : plan.placement) {
    if (iv.empty()) continue;
    vertex_of_[id] = static_cast<int>(vertex_id_.size());
    vertex_id_.push_back(id);
  }
  const size_t V = vertex_id_.size();
  out_.resize(V);
  kv_cap_.assign(V, 0.0);
  kv_est_.assign(V, 0.0);
  swarm_rate_.assign(V, 1.0);
  for (size_t v = 1; v < V; ++v) {
    const int ni = c.node_index(vertex_id_[v]);
    if (ni < 0) throw ValidationError("plan references unknown node '" + vertex_id_[v] + "'");
    const NodeSpec& n = c.nodes[ni];
    const int held = plan.placement.at(vertex_id_[v]).len();
    kv_cap_[v] = std::max(0.0, n.vram_bytes - held * c.model.bytes_per_layer());
    swarm_rate_[v] = c.layer_token_rate(n, held);
  }
  for (const PlanEdge& e : plan.edges) {
    auto si = vertex_of_.find(e.src);
    auto di = vertex_of_.find(e.dst);
    if (si == vertex_of_.end() || di == vertex_of_.end())
      throw ValidationError("plan edge " + e.src + "->" + e.dst + " references an unplaced node");
    out_[si->second].push_back({di->second, e.flow, e.exec_start, e.exec_end});
  }
  if (out_[0].empty()) throw ValidationError("plan has no edge leaving the coordinator");
  // every vertex's weights and cycle in one device call
  std::vector<std::vector<double>> flows(V);
  for (size_t v = 0; v < V; ++v)
    for (const OutEdge& e : out_[v]) flows[v].push_back(e.flow);
  std::vector<std::vector<long>> cycles = device_cycles(&flows, nullptr);
  picker_.reserve(V);
  for (size_t v = 0; v < V; ++v) picker_.emplace_back(IwrrPicker::Cycle{std::move(cycles[v])});
}

double Scheduler::hop_charge(const OutEdge& e, int input_len) const {
  const double tokens = input_len + avg_output_;
  return tokens * cluster_.model.kv_token_layer_bytes() * (e.exec_end - e.exec_start);
}

bool Scheduler::hop_eligible(const OutEdge& e, int input_len) const {
  if (e.dst == 0) return true;  // the coordinator never masks
  return kv_est_[e.dst] + hop_charge(e, input_len) <= kWatermark * kv_cap_[e.dst];
}

int Scheduler::pick(int vertex, int input_len) {
  const std::vector<OutEdge>& edges = out_[vertex];
  return picker_[vertex].next([&](int i) { return hop_eligible(edges[i], input_len); });
}

std::optional<std::vector<RouteHop>> Scheduler::admit(long request_id, int input_len) {
  std::vector<RouteHop> hops;
  std::vector<std::pair<int, double>> charged;
  const int L = cluster_.model.num_layers;
  int v = 0, covered = 0;
  while (covered < L) {
    const int p = pick(v, input_len);
    if (p < 0) {  // roll back this request's charges (scheduler.cpp:165-168)
      for (const auto& [vi, bytes] : charged) kv_est_[vi] -= bytes;
      return std::nullopt;
    }
    const OutEdge& e = out_[v][p];
    if (e.dst == 0 || e.exec_start != covered)
      throw InternalError("plan edges do not tile the layer range at '" + vertex_id_[v] + "'");
    const double bytes = hop_charge(e, input_len);
    kv_est_[e.dst] += bytes;
    charged.push_back({e.dst, bytes});
    hops.push_back({vertex_id_[e.dst], e.exec_start, e.exec_end});
    covered = e.exec_end;
    v = e.dst;
  }
  charges_[request_id] = std::move(charged);
  return hops;
}

void Scheduler::complete(long request_id, int output_len) {
  auto it = charges_.find(request_id);
  if (it == charges_.end()) throw InternalError("completing a request that was never admitted");
  for (const auto& [vi, bytes] : it->second) kv_est_[vi] -= bytes;
  charges_.erase(it);
  ++output_samples_;
  avg_output_ += (output_len - avg_output_) / static_cast<double>(output_samples_);
}

double Scheduler::kv_estimate(const std::string& node) const {
  auto it = vertex_of_.find(node);
  return it == vertex_of_.end() ? 0.0 : kv_est_[it->second];
}

double Scheduler::kv_capacity(const std::string& node) const {
  auto it = vertex_of_.find(node);
  return it == vertex_of_.end() ? 0.0 : kv_cap_[it->second];
}

// --- batch routing on the device (route.cu) ------------------------------------

std::vector<std::optional<std::vector<RouteHop>>> route_requests(const ClusterSpec& c, const PlacementPlan& plan,
                                                                 const std::vector<int>& in,
                                                                 const std::vector<int>& out) {
  if (in.size() != out.size()) throw ValidationError("input/output length arrays differ in size");
  if (plan.edges.empty()) throw ValidationError("plan has no flow edges to schedule on");
  auto placed = [&](const std::string& id) {
    if (id == c.coordinator_id) return true;
    auto it = plan.placement.find(id);
    return it != plan.placement.end() && !it->second.empty();
  };
  for (const auto& [id, iv] : plan.placement)
    if (!iv.empty() && c.node_index(id) < 0) throw ValidationError("plan references unknown node '" + id + "'");
  bool coord_out = false;
  for (const PlanEdge& e : plan.edges) {
    if (!placed(e.src) || !placed(e.dst))
      throw ValidationError("plan edge " + e.src + "->" + e.dst + " references an unplaced node");
    if (e.src == c.coordinator_id) coord_out = true;
  }
  if (!coord_out) throw ValidationError("plan has no edge leaving the coordinator");
  auto eng = gpu::engine_for(c);
  std::vector<int16_t> row(2 * c.nodes.size(), 0);
  for (const auto& [id, iv] : plan.placement) {
    if (iv.empty()) continue;
    const int idx = c.node_index(id);
    row[2 * idx] = static_cast<int16_t>(iv.start);
    row[2 * idx + 1] = static_cast<int16_t>(iv.end);
  }
  std::vector<helio_plan_edge> pe;
  for (const PlanEdge& e : plan.edges) {
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
  const int rc = helio_gpu_route_host(eng->ctx(), row.data(), pe.data(), static_cast<int32_t>(pe.size()), R,
                                      in.data(), out.data(), max_hops, nh.data(), hn.data(), hs.data(), he.data(),
                                      &deferred);
  if (rc == HELIO_ERR_INVALID) throw InternalError(helio_gpu_last_error(eng->ctx()));
  eng->check(rc, "helio_gpu_route_host");
  std::vector<std::optional<std::vector<RouteHop>>> routes(R);
  for (int64_t r = 0; r < R; ++r) {
    if (nh[r] < 0) continue;
    std::vector<RouteHop> hops;
    for (int k = 0; k < nh[r]; ++k) {
      const size_t at = (size_t)r * max_hops + k;
      hops.push_back({c.nodes[hn[at]].id, hs[at], he[at]});
    }
    routes[r] = std::move(hops);
  }
  return routes;
}

}  // namespace helio
