/* helio_planner.h — the reference's host planner and simulator linked over
 * this engine (paper_2406_01566_b200/lib/libhelio_planner.so).
 *
 * The library is the reference's own, unmodified host code — MILP planner,
 * branch and bound, simplex, LP export, heuristics, link pruning, trace
 * workload and discrete-event simulator (proj/src/{placement,bnb,lp,lp_format,
 * heuristics,workload,sim,cluster,log}.cpp), compiled where it lies under
 * /root/reference by build.py — with its flow-graph and scheduler translation
 * units replaced by this drop-in (csrc/shim_flow.cpp, csrc/shim_sched.cpp).
 * Every build_flow_graph / max_flow / compute_edge_capacity the planner makes
 * (placement.cpp:89, :223, :358-359, :441-442) runs on the B200, and the
 * simulator's Scheduler (sim.cpp:81-97, :179-192, :225) walks device-built
 * IWRR cycles: north_star's "the MILP driver stays host-side but consumes GPU
 * scores with no CPU fallback".  Only the entry points below are exported.
 *
 * The planner is C++ on both sides of this boundary: `cluster` and `plan`
 * arguments are helio::ClusterSpec* / helio::PlacementPlan* laid out as in
 * proj/include/helio/{cluster,placement}.hpp (this repo's csrc/helio/*.hpp
 * declare the same layouts).  Return codes: 0 ok, 1 ParseError,
 * 2 ValidationError, 3 InternalError, 4 any other exception; the message is
 * written to err[errlen]. */
#ifndef HELIO_PLANNER_H
#define HELIO_PLANNER_H

#include <stdint.h>

#if defined(__GNUC__)
#define HELIO_PLANNER_API __attribute__((visibility("default")))
#else
#define HELIO_PLANNER_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* PlanOptions (proj/include/helio/placement.hpp:66-75). */
typedef struct helio_plan_options {
  int32_t allow_partial;
  double prune_degree; /* <= 0 disables pruning */
  double gap;
  double time_budget_s;
  int64_t node_budget; /* -1 = unlimited */
  int32_t use_warm_starts;
  int32_t lex_tiebreak;
} helio_plan_options;

/* SimConfig (proj/include/helio/sim.hpp:13-23); policy: 0 iwrr, 1 random,
 * 2 sqf, 3 swarm (this engine's Scheduler accepts iwrr only). */
typedef struct helio_sim_config {
  int32_t online;
  double horizon_s;
  double warmup_s;
  int32_t policy;
  uint64_t seed;
  int32_t max_batch_requests;
  int32_t max_batch_tokens;
  double retry_interval_s;
  double batch_overhead_s;
} helio_sim_config;

/* plan_placement(c, opts) (placement.cpp:471-601) into *plan_out. */
HELIO_PLANNER_API int helio_planner_plan_milp(const void* cluster, const helio_plan_options* opts, void* plan_out, char* err,
                            int32_t errlen);

/* simulate(c, plan, trace, cfg) (sim.cpp:382-388) on requests (arrival_s,
 * input_len, output_len)[n]; *metrics_json receives the reference Python
 * binding's metrics dict (pymodule.cpp:34-74) as JSON (free with
 * helio_planner_free). */
HELIO_PLANNER_API int helio_planner_simulate(const void* cluster, const void* plan, int64_t n, const double* arrival_s,
                           const int32_t* input_len, const int32_t* output_len, const helio_sim_config* cfg,
                           char** metrics_json, char* err, int32_t errlen);

/* prune_links(c, target_avg_degree, &report) (placement.cpp:230-332) into
 * *cluster_out; report fields optional (NULL). */
HELIO_PLANNER_API int helio_planner_prune_links(const void* cluster, double target_avg_degree, void* cluster_out,
                              int32_t* links_removed, double* avg_degree_before, double* avg_degree_after,
                              char** warnings_json, char* err, int32_t errlen);

/* throughput_upper_bound(c) (placement.cpp:30-40). */
HELIO_PLANNER_API int helio_planner_upper_bound(const void* cluster, double* out, char* err, int32_t errlen);

HELIO_PLANNER_API void helio_planner_free(char* p);

/* sizeof (ClusterSpec, PlacementPlan, FlowGraph, Scheduler, IwrrPicker, Rng)
 * and alignof(Scheduler) as the reference's headers lay them out, into
 * sizes[0..n); returns how many there are.  The bindings compare them with
 * this repo's declarations before passing objects across. */
HELIO_PLANNER_API int helio_planner_layout(int64_t* sizes, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* HELIO_PLANNER_H */
