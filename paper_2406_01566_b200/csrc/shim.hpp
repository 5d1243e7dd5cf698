// shim.hpp — the reference's C++ surface (helio::) plus the batched engine
// handle the drop-in exposes beside it.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../../include/helio_gpu.h"
#include "helio/cluster.hpp"
#include "helio/errors.hpp"
#include "helio/flow_graph.hpp"
#include "helio/placement.hpp"
#include "helio/scheduler.hpp"

namespace helio {

// Validates a Placement exactly as build_flow_graph does (flow_graph.cpp:52-61,
// same ValidationError texts) and returns its int16 [N][2] row.
std::vector<int16_t> placement_row(const ClusterSpec& c, const Placement& p);

namespace gpu {

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
