// planner_api.cpp — extern "C" entry points of libhelio_planner.so
// (include/helio_planner.h).  Compiled against the REFERENCE's headers
// (proj/include/helio), like the reference sources it is linked with; the
// drop-in translation units in the same library (shim_flow.cpp,
// shim_sched.cpp) are compiled against this repo's layout-identical headers.
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/helio_planner.h"
#include "helio/errors.hpp"
#include "helio/placement.hpp"
#include "helio/scheduler.hpp"
#include "helio/sim.hpp"
#include "json.hpp"

using namespace helio;

namespace {

void put(char* err, int32_t errlen, const std::string& m) {
  if (err && errlen > 0) {
    std::strncpy(err, m.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

// One exception -> code mapping for every entry (header: 1 Parse,
// 2 Validation, 3 Internal, 4 other).
template <class F>
int guarded(char* err, int32_t errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    put(err, errlen, e.what());
    return 1;
  } catch (const ValidationError& e) {
    put(err, errlen, e.what());
    return 2;
  } catch (const InternalError& e) {
    put(err, errlen, e.what());
    return 3;
  } catch (const std::exception& e) {
    put(err, errlen, e.what());
    return 4;
  }
}

char* dup(const std::string& s) {
  char* p = new char[s.size() + 1];
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// The keys and order of the reference binding's metrics_to_dict
// (proj/bindings/pymodule.cpp:34-74).
std::string metrics_json(const SimMetrics& m) {
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
  for (const NodeStats& n : m.nodes)
    d["nodes"].push_back({{"id", n.id},
                          {"utilization", n.utilization},
                          {"batches", n.batches},
                          {"layer_tokens", n.layer_tokens},
                          {"kv_pages", n.kv_pages}});
  d["links"] = nlohmann::ordered_json::array();
  for (const LinkStats& l : m.links)
    d["links"].push_back({{"src", l.src},
                          {"dst", l.dst},
                          {"bytes", l.bytes},
                          {"transfers", l.transfers},
                          {"queue_delay_mean_s", l.queue_delay_mean_s},
                          {"queue_delay_max_s", l.queue_delay_max_s}});
  d["warnings"] = m.warnings;
  return d.dump();
}

}  // namespace

extern "C" {

int helio_planner_plan_milp(const void* cluster, const helio_plan_options* o, void* plan_out, char* err,
                            int32_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cluster || !o || !plan_out) throw ValidationError("null argument");
    PlanOptions opts;
    opts.allow_partial = o->allow_partial != 0;
    opts.prune_degree = o->prune_degree;
    opts.gap = o->gap;
    opts.time_budget_s = o->time_budget_s;
    opts.node_budget = static_cast<long>(o->node_budget);
    opts.use_warm_starts = o->use_warm_starts != 0;
    opts.lex_tiebreak = o->lex_tiebreak != 0;
    *static_cast<PlacementPlan*>(plan_out) = plan_placement(*static_cast<const ClusterSpec*>(cluster), opts);
  });
}

int helio_planner_simulate(const void* cluster, const void* plan, int64_t n, const double* arrival_s,
                           const int32_t* input_len, const int32_t* output_len, const helio_sim_config* cfg,
                           char** metrics_out, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cluster || !plan || !cfg || !metrics_out || n < 0 || (n > 0 && (!arrival_s || !input_len || !output_len)))
      throw ValidationError("null argument");
    std::vector<Request> reqs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) reqs[i] = {arrival_s[i], input_len[i], output_len[i]};
    SimConfig sc;
    sc.mode = cfg->online ? TraceMode::kOnline : TraceMode::kOffline;
    sc.horizon_s = cfg->horizon_s;
    sc.warmup_s = cfg->warmup_s;
    static const SchedPolicy kPolicy[] = {SchedPolicy::kIwrr, SchedPolicy::kRandom, SchedPolicy::kSqf,
                                          SchedPolicy::kSwarm};
    if (cfg->policy < 0 || cfg->policy > 3) throw ValidationError("unknown scheduler policy index");
    sc.policy = kPolicy[cfg->policy];
    sc.seed = cfg->seed;
    sc.max_batch_requests = cfg->max_batch_requests;
    sc.max_batch_tokens = cfg->max_batch_tokens;
    sc.retry_interval_s = cfg->retry_interval_s;
    sc.batch_overhead_s = cfg->batch_overhead_s;
    const SimMetrics m = simulate(*static_cast<const ClusterSpec*>(cluster),
                                  *static_cast<const PlacementPlan*>(plan), reqs, sc);
    *metrics_out = dup(metrics_json(m));
  });
}

int helio_planner_prune_links(const void* cluster, double degree, void* cluster_out, int32_t* removed,
                              double* before, double* after, char** warnings_json, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cluster || !cluster_out) throw ValidationError("null argument");
    PruneReport rep;
    *static_cast<ClusterSpec*>(cluster_out) = prune_links(*static_cast<const ClusterSpec*>(cluster), degree, &rep);
    if (removed) *removed = rep.links_removed;
    if (before) *before = rep.avg_degree_before;
    if (after) *after = rep.avg_degree_after;
    if (warnings_json) *warnings_json = dup(nlohmann::json(rep.warnings).dump());
  });
}

int helio_planner_upper_bound(const void* cluster, double* out, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cluster || !out) throw ValidationError("null argument");
    *out = throughput_upper_bound(*static_cast<const ClusterSpec*>(cluster));
  });
}

void helio_planner_free(char* p) { delete[] p; }

int helio_planner_layout(int64_t* sizes, int32_t n) {
  const int64_t v[] = {(int64_t)sizeof(ClusterSpec), (int64_t)sizeof(PlacementPlan), (int64_t)sizeof(FlowGraph),
                       (int64_t)sizeof(Scheduler), (int64_t)sizeof(IwrrPicker), (int64_t)sizeof(Rng),
                       (int64_t)alignof(Scheduler)};
  const int32_t m = (int32_t)(sizeof(v) / sizeof(v[0]));
  for (int32_t i = 0; i < n && i < m; ++i) sizes[i] = v[i];
  return m;
}

}  // extern "C"
