// shim_sched.cpp — iwrr_weights / IwrrPicker / Scheduler::route over the
// device route kernels (scheduler.cpp:28-190).
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
