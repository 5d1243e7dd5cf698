// shim_engine.hpp — engine handle and flow-graph helpers of the drop-in.
// Depends only on the cluster and flow-graph types (flow_graph.hpp), so the
// flow-graph translation unit can be linked under the reference's own
// placement/scheduler code (oracle/Makefile's hybrid target).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../../include/helio_gpu.h"
#include "helio/cluster.hpp"
#include "helio/errors.hpp"
#include "helio/flow_graph.hpp"

namespace helio {

// Validates a Placement exactly as build_flow_graph does (flow_graph.cpp:52-61,
// same ValidationError texts) and returns its int16 [N][2] row.
std::vector<int16_t> placement_row(const ClusterSpec& c, const Placement& p);

namespace detail {
// One placement through the engine in PARITY mode: vertices, value and the
// full edge list (reference g.edges order, per-edge flows).
struct Solved {
  int nv = 0;
  double value = 0;
  std::vector<helio_edge> edges;
};
Solved solve_one(const ClusterSpec& c, const Placement& p, bool allow_partial);
const std::string& node_name(const ClusterSpec& c, int idx);
}  // namespace detail

namespace gpu {

// The C-ABI cluster descriptor of a ClusterSpec (arrays owned here).
// Throws ValidationError on duplicate ids or a non-contiguous throughput table.
struct ClusterDesc {
  helio_cluster_desc d{};
  std::vector<double> vram, kvr, peak, nin, nout, tval, lbw;
  std::vector<int32_t> toff, rank, lsrc, ldst;
  ClusterDesc() = default;
  ClusterDesc(const ClusterDesc&) = delete;
  ClusterDesc& operator=(const ClusterDesc&) = delete;
  ClusterDesc& operator=(ClusterDesc&&) = default;
};
void make_cluster_desc(const ClusterSpec& c, ClusterDesc& out);

// One engine context bound to a device with one compiled cluster.
class Engine {
 public:
  explicit Engine(int device);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void set_cluster(const ClusterSpec& c);
  helio_gpu_ctx* ctx() const { return ctx_; }
  int device() const { return device_; }
  int num_nodes() const { return N_; }
  int num_layers() const { return num_layers_; }
  int num_links() const { return num_links_; }
  const std::vector<int32_t>& kmax() const { return kmax_; }
  const std::vector<std::string>& ids() const { return ids_; }
  const std::string& coordinator() const { return coordinator_; }
  void check(int rc, const char* what) const;

 private:
  int device_ = 0;
  helio_gpu_ctx* ctx_ = nullptr;
  int N_ = 0, num_layers_ = 0, num_links_ = 0;
  std::vector<int32_t> kmax_;
  std::vector<std::string> ids_;
  std::string coordinator_;
};

// Engine compiled for this cluster's current contents (small MRU cache).
std::shared_ptr<Engine> engine_for(const ClusterSpec& c);
// Engine without a cluster, for raw graphs and the IWRR helpers.
std::shared_ptr<Engine> raw_engine();

}  // namespace gpu
}  // namespace helio
