// Baseline placement heuristics — same names and result type as
// proj/include/helio/heuristics.hpp:10-26.  They seed the device local search
// (helio_gpu_local_search).
#pragma once

#include <string>
#include <vector>

#include "helio/flow_graph.hpp"

namespace helio {

struct HeuristicResult {
  Placement placement;
  std::vector<std::string> warnings;
};

// Swarm: uniform stages, as many as the smallest node needs to hold one;
// nodes (largest single-layer throughput first) join the lightest stage.
HeuristicResult swarm_placement(const ClusterSpec& c);

// Petals: in declared order, each node takes the k_i-layer window with the
// least throughput served so far (lowest start on ties).
HeuristicResult petals_placement(const ClusterSpec& c);

// Separate pipelines: one evenly split pipeline per device type; types that
// cannot hold the model are left idle.
HeuristicResult separate_pipelines_placement(const ClusterSpec& c);

// Not in the reference: best-improvement single-node-move local search on the
// device (helio_gpu_local_search) from `seed`, scored in PARITY mode so every
// decision is the reference's own max-flow value.  The seed must validate
// (ValidationError otherwise).  max_moves < 0: run to a local optimum.
struct LocalSearchResult {
  Placement placement;
  double value = 0;
  int moves = 0;
  long long scored = 0;
};
// swaps: also exchange two nodes' intervals (HELIO_LS_SWAPS).
LocalSearchResult local_search_placement(const ClusterSpec& c, const Placement& seed, bool allow_partial,
                                         int max_moves = -1, bool swaps = true);
// local search -> sampled multi-node search (helio_gpu_sampled_search, SCORE
// mode) -> local search again (PARITY: the value is reference-exact);
// `scored` counts every placement scored.
LocalSearchResult sampled_search_placement(const ClusterSpec& c, const Placement& seed, bool allow_partial,
                                           int rounds = 30, long long batch = 1 << 20, int max_changes = 3,
                                           unsigned long long rng_seed = 7);

}  // namespace helio
