// shim_plan.cpp — plan_from_placement (placement.cpp:440-469) over the device's
// PARITY flows.
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

using detail::node_name;
using detail::solve_one;
using detail::Solved;

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

}  // namespace helio
