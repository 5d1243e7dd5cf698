// shim_cluster.cpp — the cluster model of the drop-in (cluster.cpp:56-100, 237-300).
// Kept in its own translation unit so a build can take these from the
// reference instead (oracle/Makefile's hybrid target).
#include "helio/cluster.hpp"

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

// --- cluster model (cluster.cpp:56-100, 237-300) ----------------------------

int ClusterSpec::node_index(const std::string& id) const {
  for (size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].id == id) return static_cast<int>(i);
  return -1;
}

int ClusterSpec::max_layers(const NodeSpec& n) const {
  const double usable = n.vram_bytes * (1.0 - n.kv_reserve);
  int k = static_cast<int>(std::floor(usable / model.bytes_per_layer()));
  if (!n.throughput_table.empty()) k = std::min(k, n.throughput_table.rbegin()->first);
  return std::min(k, model.num_layers);
}

double ClusterSpec::throughput(const NodeSpec& n, int j) const {
  if (j < 1 || j > max_layers(n))
    throw ValidationError("throughput request for node '" + n.id + "' outside profile range: j=" +
                          std::to_string(j));
  if (!n.throughput_table.empty()) return n.throughput_table.at(j);
  return n.peak_layer_tokens / j;
}

double ClusterSpec::layer_token_rate(const NodeSpec& n, int j) const { return j * throughput(n, j); }

static double incident_bw(const ClusterSpec& c, const NodeSpec& n) {
  double best = 0;
  for (const auto& l : c.links)
    if (l.src == n.id || l.dst == n.id) best = std::max(best, l.bandwidth_bps);
  return best;
}

double ClusterSpec::nic_in(const NodeSpec& n) const {
  return n.nic_in_bps > 0 ? n.nic_in_bps : incident_bw(*this, n);
}

double ClusterSpec::nic_out(const NodeSpec& n) const {
  return n.nic_out_bps > 0 ? n.nic_out_bps : incident_bw(*this, n);
}

double link_token_capacity(const LinkSpec& link, double payload_bytes) {
  return link.bandwidth_bps / (8.0 * payload_bytes);
}

void validate_cluster(const ClusterSpec& c) {
  auto fail = [](const std::string& msg) { throw ValidationError(msg); };
  if (c.model.num_layers < 1) fail("model.num_layers must be >= 1");
  if (c.model.param_bytes <= 0) fail("model.param_gb must be > 0");
  if (c.model.token_bytes <= 0) fail("model.token_bytes must be > 0");
  if (c.model.activation_bytes <= 0) fail("model.activation_bytes must be > 0");
  if (c.model.kv_bytes_per_token_layer < 0) fail("model.kv_bytes_per_token_layer must be >= 0");
  if (c.coordinator_id.empty()) fail("coordinator.id must be non-empty");
  if (c.nodes.empty()) fail("cluster needs at least one compute node");
  std::set<std::string> ids;
  for (const auto& n : c.nodes) {
    if (n.id.empty()) fail("node id must be non-empty");
    if (n.id == c.coordinator_id) fail("node id '" + n.id + "' collides with the coordinator");
    if (!ids.insert(n.id).second) fail("duplicate node id '" + n.id + "'");
    if (n.vram_bytes <= 0) fail("node '" + n.id + "': vram_gb must be > 0");
    if (n.kv_reserve < 0 || n.kv_reserve >= 1) fail("node '" + n.id + "': kv_reserve must be in [0, 1)");
    const bool has_peak = n.peak_layer_tokens > 0;
    const bool has_table = !n.throughput_table.empty();
    if (has_peak == has_table)
      fail("node '" + n.id + "': exactly one of peak_layer_tokens_per_s or throughput_table required");
    if (has_table) {
      int expect = 1;
      double prev = 0;
      for (const auto& [j, v] : n.throughput_table) {
        if (j != expect) fail("node '" + n.id + "': throughput_table keys must be contiguous from 1");
        if (v <= 0) fail("node '" + n.id + "': throughput_table values must be > 0");
        if (expect > 1 && v >= prev) fail("node '" + n.id + "': throughput_table must be strictly decreasing");
        prev = v;
        ++expect;
      }
    }
    if (n.nic_in_bps < 0 || n.nic_out_bps < 0) fail("node '" + n.id + "': NIC rates must be >= 0");
  }
  std::set<std::pair<std::string, std::string>> pairs;
  bool coord_out = false, coord_in = false;
  for (const auto& l : c.links) {
    auto known = [&](const std::string& e) { return e == c.coordinator_id || c.node_index(e) >= 0; };
    if (!known(l.src)) fail("link endpoint '" + l.src + "' is not a declared node");
    if (!known(l.dst)) fail("link endpoint '" + l.dst + "' is not a declared node");
    if (l.src == l.dst) fail("self-link on '" + l.src + "'");
    if (!pairs.insert({l.src, l.dst}).second) fail("duplicate link " + l.src + " -> " + l.dst);
    if (l.bandwidth_bps <= 0) fail("link " + l.src + " -> " + l.dst + ": bandwidth must be > 0");
    if (l.latency_s < 0) fail("link " + l.src + " -> " + l.dst + ": latency must be >= 0");
    if (l.src == c.coordinator_id) coord_out = true;
    if (l.dst == c.coordinator_id) coord_in = true;
  }
  if (!coord_out) fail("coordinator has no outgoing link");
  if (!coord_in) fail("coordinator has no incoming link");
  long total = 0;
  for (const auto& n : c.nodes) total += c.max_layers(n);
  if (total < c.model.num_layers)
    fail("insufficient VRAM: total layer capacity " + std::to_string(total) + " < model layers " +
         std::to_string(c.model.num_layers));
}

}  // namespace helio
