// shim_heuristics.cpp — host restatement of the reference's baseline placement
// heuristics (src/heuristics.cpp:12-131), the seeds of the device local search.
// They are O(N·L) host loops run once per search, not part of the scored path.
#include <algorithm>
#include <limits>
#include <map>

#include "helio/errors.hpp"
#include "helio/heuristics.hpp"
#include "shim_engine.hpp"

namespace helio {

namespace {

// The stage a node joins: the first stage with the smallest running total.
int lightest(const std::vector<double>& total) {
  return static_cast<int>(std::min_element(total.begin(), total.end()) - total.begin());
}

}  // namespace

// heuristics.cpp:12-54
HeuristicResult swarm_placement(const ClusterSpec& c) {
  HeuristicResult r;
  const int L = c.model.num_layers;
  std::vector<int> usable;
  int smallest = L + 1;
  for (int i = 0; i < static_cast<int>(c.nodes.size()); ++i) {
    const int k = c.max_layers(c.nodes[i]);
    if (k >= 1) {
      usable.push_back(i);
      smallest = std::min(smallest, k);
    } else {
      r.warnings.push_back("swarm: node '" + c.nodes[i].id + "' cannot hold a layer; dropped");
    }
  }
  if (usable.empty()) {
    r.warnings.push_back("swarm: no usable nodes");
    return r;
  }
  const int n_stages = (L + smallest - 1) / smallest;
  const int stage_len = (L + n_stages - 1) / n_stages;
  if (n_stages > static_cast<int>(usable.size()))
    r.warnings.push_back("swarm: fewer nodes than stages; pipeline has gaps");
  std::vector<double> one_layer(c.nodes.size(), 0.0);
  for (int i : usable) one_layer[i] = c.throughput(c.nodes[i], 1);
  std::stable_sort(usable.begin(), usable.end(), [&](int a, int b) { return one_layer[a] > one_layer[b]; });
  std::vector<double> load(n_stages, 0.0);
  for (int i : usable) {
    const int g = lightest(load);
    const int s = g * stage_len;
    r.placement[c.nodes[i].id] = Interval{s, std::min(s + stage_len, L)};
    load[g] += one_layer[i];
  }
  return r;
}

// heuristics.cpp:56-79
HeuristicResult petals_placement(const ClusterSpec& c) {
  HeuristicResult r;
  const int L = c.model.num_layers;
  std::vector<double> served(L, 0.0);
  for (const NodeSpec& n : c.nodes) {
    const int w = std::min(c.max_layers(n), L);
    if (w < 1) {
      r.warnings.push_back("petals: node '" + n.id + "' cannot hold a layer; skipped");
      continue;
    }
    // window sums, left to right; a later window wins only when lighter by
    // more than 1e-12 (ties keep the lowest start)
    int at = 0;
    double least = std::numeric_limits<double>::infinity();
    for (int s = 0; s + w <= L; ++s) {
      double sum = 0.0;
      for (int l = s; l < s + w; ++l) sum += served[l];
      if (sum < least - 1e-12) {
        least = sum;
        at = s;
      }
    }
    r.placement[n.id] = Interval{at, at + w};
    const double rate = c.throughput(n, w);
    for (int l = at; l < at + w; ++l) served[l] += rate;
  }
  return r;
}

// heuristics.cpp:81-129
HeuristicResult separate_pipelines_placement(const ClusterSpec& c) {
  HeuristicResult r;
  const int L = c.model.num_layers;
  std::vector<std::string> types;  // first-appearance order
  std::map<std::string, std::vector<int>> members;
  for (int i = 0; i < static_cast<int>(c.nodes.size()); ++i) {
    const std::string& t = c.nodes[i].type;
    if (t.empty())
      throw ValidationError("separate-pipelines requires a type label on node '" + c.nodes[i].id + "'");
    auto it = members.find(t);
    if (it == members.end()) {
      types.push_back(t);
      members[t] = {i};
    } else {
      it->second.push_back(i);
    }
  }
  bool served = false;
  for (const std::string& t : types) {
    const std::vector<int>& m = members[t];
    long layers = 0;
    for (int i : m) layers += c.max_layers(c.nodes[i]);
    if (layers < L) {
      r.warnings.push_back("separate-pipelines: type '" + t + "' cannot hold the model; unused");
      continue;
    }
    const int used = std::min<int>(static_cast<int>(m.size()), L);
    const int q = L / used, rem = L % used;
    std::vector<Interval> stage(used);
    bool ok = true;
    for (int idx = 0, at = 0; idx < used && ok; ++idx) {
      const int len = q + (idx < rem ? 1 : 0);
      ok = len <= c.max_layers(c.nodes[m[idx]]);
      stage[idx] = Interval{at, at + len};
      at += len;
    }
    if (!ok) {
      r.warnings.push_back("separate-pipelines: type '" + t + "' cannot hold an even pipeline; unused");
      continue;
    }
    if (used < static_cast<int>(m.size())) r.warnings.push_back("separate-pipelines: type '" + t + "' has idle nodes");
    for (int idx = 0; idx < used; ++idx) r.placement[c.nodes[m[idx]].id] = stage[idx];
    served = true;
  }
  if (!served) r.warnings.push_back("separate-pipelines: no type can serve the model");
  return r;
}

LocalSearchResult local_search_placement(const ClusterSpec& c, const Placement& seed, bool allow_partial,
                                         int max_moves, bool swaps) {
  const std::vector<int16_t> row = placement_row(c, seed);  // validates, reference messages
  // N <= 64: the cached PARITY engine.  Larger (sparse) clusters: PARITY's
  // exact FIFO replay costs ~40x SCORE per graph there (syn256: minutes per
  // search), so the moves are scored in SCORE mode on a private context and
  // the final placement's value is re-solved in PARITY below.
  const bool score_moves = c.nodes.size() > 64;
  std::shared_ptr<gpu::Engine> eng = gpu::engine_for(c);
  if (score_moves) {
    eng = std::make_shared<gpu::Engine>(eng->device());
    eng->set_cluster(c);
    eng->check(helio_gpu_set_mode(eng->ctx(), HELIO_MODE_SCORE), "helio_gpu_set_mode");
  }
  std::vector<int16_t> out(row.size(), 0);
  LocalSearchResult r;
  int32_t moves = 0;
  int64_t scored = 0;
  const int32_t hood = HELIO_LS_MOVES | (swaps ? HELIO_LS_SWAPS : 0);
  eng->check(helio_gpu_local_search(eng->ctx(), row.data(), allow_partial ? 1 : 0, max_moves, hood, &r.value,
                                    out.data(), &moves, &scored),
             "helio_gpu_local_search");
  for (size_t i = 0; i < c.nodes.size(); ++i)
    if (out[2 * i + 1] > out[2 * i]) r.placement[c.nodes[i].id] = Interval{out[2 * i], out[2 * i + 1]};
  if (score_moves) r.value = detail::solve_one(c, r.placement, allow_partial).value;
  r.moves = moves;
  r.scored = scored;
  return r;
}

LocalSearchResult sampled_search_placement(const ClusterSpec& c, const Placement& seed, bool allow_partial,
                                           int rounds, long long batch, int max_changes,
                                           unsigned long long rng_seed) {
  LocalSearchResult a = local_search_placement(c, seed, allow_partial);
  const std::vector<int16_t> row = placement_row(c, a.placement);
  // a private SCORE-mode context (the cached engine stays PARITY for its
  // other callers); the closing local search re-scores in PARITY
  auto eng = std::make_unique<gpu::Engine>(gpu::engine_for(c)->device());
  eng->set_cluster(c);
  eng->check(helio_gpu_set_mode(eng->ctx(), HELIO_MODE_SCORE), "helio_gpu_set_mode");
  std::vector<int16_t> out(row.size(), 0);
  double value = 0;
  int32_t improvements = 0;
  int64_t scored = 0;
  eng->check(helio_gpu_sampled_search(eng->ctx(), row.data(), allow_partial ? 1 : 0, rounds, batch, max_changes,
                                      rng_seed, &value, out.data(), &improvements, &scored),
             "helio_gpu_sampled_search");
  Placement mid;
  for (size_t i = 0; i < c.nodes.size(); ++i)
    if (out[2 * i + 1] > out[2 * i]) mid[c.nodes[i].id] = Interval{out[2 * i], out[2 * i + 1]};
  LocalSearchResult r = local_search_placement(c, mid, allow_partial);
  r.moves += a.moves + improvements;
  r.scored += a.scored + scored;
  // the middle phase accepts SCORE-mode moves, which on float capacities can
  // be rounding noise: never return less than the first PARITY local optimum
  if (r.value < a.value) {
    r.placement = a.placement;
    r.value = a.value;
  }
  return r;
}

}  // namespace helio

