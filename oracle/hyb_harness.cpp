// TEST INFRASTRUCTURE ONLY — the reference's UNMODIFIED host-side planner
// (MILP, B&B, simplex, heuristics: proj/src/*.cpp except flow_graph.cpp)
// linked against the B200 drop-in's flow-graph translation unit
// (paper_2406_01566_b200/csrc/shim_flow.cpp) and libhelio_gpu.so.  Every
// build_flow_graph / max_flow / compute_edge_capacity the planner makes
// (placement.cpp:89, :223, :358-359, :441-442) runs on the B200 — north_star:
// "the MILP driver stays host-side but consumes GPU scores with no CPU
// fallback".  Built by `make -C oracle hybrid` into oracle/_ref/.
#include <cstdint>
#include <cstring>
#include <string>

#include "helio/cluster.hpp"
#include "helio/errors.hpp"
#include "helio/flow_graph.hpp"
#include "helio/placement.hpp"

extern "C" void* hyb_cluster_from_json(const char* text, char* err, int errlen) {
  try {
    return new helio::ClusterSpec(helio::parse_cluster(text, "<hyb>"));
  } catch (const std::exception& ex) {
    if (err && errlen > 0) {
      std::strncpy(err, ex.what(), errlen - 1);
      err[errlen - 1] = 0;
    }
    return nullptr;
  }
}

extern "C" void hyb_cluster_free(void* c) { delete static_cast<helio::ClusterSpec*>(c); }

#define HARNESS_FN(x) hyb_##x
#include "milp_harness.inc"
