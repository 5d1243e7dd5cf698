// pymodule.cpp — `_helio`, the Python face of the drop-in.
//
// Same names and argument meaning as the reference's bindings
// (proj/bindings/pymodule.cpp:78-219) for the hot-path surface —
// Cluster, Plan, max_flow_value, plan_for_placement, ParseError and
// ValidationError as ValueError subclasses — plus the batched entry points
// the B200 engine adds (Engine.score / best / flows / route, max_flow_values,
// best_placement, route_requests, max_flow_raw).
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <dlfcn.h>

#include <chrono>
#include <cmath>
#include <random>

#include "shim.hpp"
#include "helio/heuristics.hpp"
#include "../../include/helio_planner.h"

namespace py = pybind11;
using namespace helio;

namespace {

// --- cluster JSON (cluster.cpp:102-181 schema, parsed with Python's json) ----

[[noreturn]] void fail_parse(const std::string& origin, const std::string& msg) {
  throw ParseError(origin + ": " + msg);
}

void check_fields(const py::dict& obj, std::initializer_list<const char*> allowed, const std::string& origin,
                  const std::string& where) {
  for (auto kv : obj) {
    std::string k = py::str(kv.first);
    bool ok = false;
    for (const char* a : allowed) ok = ok || k == a;
    if (!ok) fail_parse(origin, "unknown field '" + k + "' in " + where);
  }
}

bool is_number(const py::handle& h) {
  return (py::isinstance<py::int_>(h) || py::isinstance<py::float_>(h)) && !py::isinstance<py::bool_>(h);
}

double get_num(const py::dict& obj, const char* key, const std::string& origin, const double* def = nullptr) {
  if (!obj.contains(key)) {
    if (def) return *def;
    fail_parse(origin, std::string("missing field '") + key + "'");
  }
  py::handle v = obj[key];
  if (!is_number(v)) fail_parse(origin, std::string("field '") + key + "' must be a number");
  return v.cast<double>();
}

std::string get_str(const py::dict& obj, const char* key, const std::string& origin, const char* def = nullptr) {
  if (!obj.contains(key)) {
    if (def) return def;
    fail_parse(origin, std::string("missing field '") + key + "'");
  }
  py::handle v = obj[key];
  if (!py::isinstance<py::str>(v)) fail_parse(origin, std::string("field '") + key + "' must be a string");
  return v.cast<std::string>();
}

ClusterSpec parse_cluster(const std::string& text, const std::string& origin) {
  py::object json = py::module_::import("json");
  py::object root;
  try {
    root = json.attr("loads")(text);
  } catch (py::error_already_set& e) {
    fail_parse(origin, std::string("invalid JSON: ") + e.what());
  }
  if (!py::isinstance<py::dict>(root)) fail_parse(origin, "top level must be an object");
  py::dict r = root;
  check_fields(r, {"model", "coordinator", "nodes", "links"}, origin, "top level");
  ClusterSpec c;
  if (!r.contains("model") || !py::isinstance<py::dict>(r["model"])) fail_parse(origin, "missing 'model' object");
  py::dict m = r["model"];
  check_fields(m, {"name", "num_layers", "param_gb", "token_bytes", "activation_bytes", "kv_bytes_per_token_layer"},
               origin, "model");
  const double four = 4.0, act = 16384.0, zero = 0.0, half = 0.5;
  c.model.name = get_str(m, "name", origin, "");
  c.model.num_layers = static_cast<int>(get_num(m, "num_layers", origin));
  c.model.param_bytes = get_num(m, "param_gb", origin) * 1e9;
  c.model.token_bytes = get_num(m, "token_bytes", origin, &four);
  c.model.activation_bytes = get_num(m, "activation_bytes", origin, &act);
  c.model.kv_bytes_per_token_layer = get_num(m, "kv_bytes_per_token_layer", origin, &zero);
  if (!r.contains("coordinator") || !py::isinstance<py::dict>(r["coordinator"]))
    fail_parse(origin, "missing 'coordinator' object");
  py::dict co = r["coordinator"];
  check_fields(co, {"id"}, origin, "coordinator");
  c.coordinator_id = get_str(co, "id", origin);
  if (!r.contains("nodes") || !py::isinstance<py::list>(r["nodes"])) fail_parse(origin, "missing 'nodes' array");
  for (auto jn_h : py::list(r["nodes"])) {
    if (!py::isinstance<py::dict>(jn_h)) fail_parse(origin, "node entries must be objects");
    py::dict jn = py::reinterpret_borrow<py::dict>(jn_h);
    check_fields(jn, {"id", "type", "vram_gb", "kv_reserve", "peak_layer_tokens_per_s", "throughput_table",
                      "nic_in_gbps", "nic_out_gbps"},
                 origin, "node");
    NodeSpec n;
    n.id = get_str(jn, "id", origin);
    n.type = get_str(jn, "type", origin, "");
    n.vram_bytes = get_num(jn, "vram_gb", origin) * 1e9;
    n.kv_reserve = get_num(jn, "kv_reserve", origin, &half);
    n.peak_layer_tokens = get_num(jn, "peak_layer_tokens_per_s", origin, &zero);
    if (jn.contains("throughput_table")) {
      if (!py::isinstance<py::dict>(jn["throughput_table"]))
        fail_parse(origin, "throughput_table must map layer count to tokens/s");
      for (auto kv : py::dict(jn["throughput_table"])) {
        std::string key = py::str(kv.first);
        int j = 0;
        try {
          j = std::stoi(key);
        } catch (...) {
          fail_parse(origin, "throughput_table key '" + key + "' is not an integer");
        }
        if (!is_number(kv.second)) fail_parse(origin, "throughput_table values must be numbers");
        n.throughput_table[j] = kv.second.cast<double>();
      }
    }
    n.nic_in_bps = get_num(jn, "nic_in_gbps", origin, &zero) * 1e9;
    n.nic_out_bps = get_num(jn, "nic_out_gbps", origin, &zero) * 1e9;
    c.nodes.push_back(std::move(n));
  }
  if (!r.contains("links") || !py::isinstance<py::list>(r["links"])) fail_parse(origin, "missing 'links' array");
  for (auto jl_h : py::list(r["links"])) {
    if (!py::isinstance<py::dict>(jl_h)) fail_parse(origin, "link entries must be objects");
    py::dict jl = py::reinterpret_borrow<py::dict>(jl_h);
    check_fields(jl, {"src", "dst", "bandwidth_mbps", "latency_ms"}, origin, "link");
    LinkSpec l;
    l.src = get_str(jl, "src", origin);
    l.dst = get_str(jl, "dst", origin);
    l.bandwidth_bps = get_num(jl, "bandwidth_mbps", origin) * 1e6;
    l.latency_s = get_num(jl, "latency_ms", origin, &zero) * 1e-3;
    c.links.push_back(std::move(l));
  }
  validate_cluster(c);
  return c;
}

std::string serialize_cluster(const ClusterSpec& c) {
  py::dict root, m;
  m["name"] = c.model.name;
  m["num_layers"] = c.model.num_layers;
  m["param_gb"] = c.model.param_bytes / 1e9;
  m["token_bytes"] = c.model.token_bytes;
  m["activation_bytes"] = c.model.activation_bytes;
  m["kv_bytes_per_token_layer"] = c.model.kv_bytes_per_token_layer;
  root["model"] = m;
  py::dict co;
  co["id"] = c.coordinator_id;
  root["coordinator"] = co;
  py::list nodes;
  for (const auto& n : c.nodes) {
    py::dict jn;
    jn["id"] = n.id;
    jn["type"] = n.type;
    jn["vram_gb"] = n.vram_bytes / 1e9;
    jn["kv_reserve"] = n.kv_reserve;
    jn["peak_layer_tokens_per_s"] = n.peak_layer_tokens;
    if (!n.throughput_table.empty()) {
      py::dict t;
      for (const auto& [j, v] : n.throughput_table) t[py::str(std::to_string(j))] = v;
      jn["throughput_table"] = t;
    }
    jn["nic_in_gbps"] = n.nic_in_bps / 1e9;
    jn["nic_out_gbps"] = n.nic_out_bps / 1e9;
    nodes.append(jn);
  }
  root["nodes"] = nodes;
  py::list links;
  for (const auto& l : c.links) {
    py::dict jl;
    jl["src"] = l.src;
    jl["dst"] = l.dst;
    jl["bandwidth_mbps"] = l.bandwidth_bps / 1e6;
    jl["latency_ms"] = l.latency_s * 1e3;
    links.append(jl);
  }
  root["links"] = links;
  return py::module_::import("json").attr("dumps")(root, py::arg("indent") = 2, py::arg("ensure_ascii") = false).cast<std::string>() + "\n";
}

Placement placement_from_dict(const py::dict& d) {
  Placement p;
  for (const auto& kv : d) {
    auto iv = kv.second.cast<std::pair<int, int>>();
    p[kv.first.cast<std::string>()] = {iv.first, iv.second};
  }
  return p;
}

py::dict placement_to_dict(const Placement& p) {
  py::dict d;
  for (const auto& [id, iv] : p)
    if (!iv.empty()) d[py::str(id)] = py::make_tuple(iv.start, iv.end);
  return d;
}

const char* status_name(MilpStatus s) {
  switch (s) {
    case MilpStatus::kOptimal: return "optimal";
    case MilpStatus::kFeasible: return "feasible";
    case MilpStatus::kInfeasible: return "infeasible";
    case MilpStatus::kUnbounded: return "unbounded";
    default: return "no-incumbent";
  }
}

std::string serialize_plan(const PlacementPlan& plan) {
  py::dict root;
  root["method"] = plan.method;
  root["status"] = status_name(plan.status);
  root["objective"] = plan.objective;
  root["best_bound"] = plan.best_bound;
  root["allow_partial"] = plan.allow_partial;
  root["nodes_explored"] = plan.nodes_explored;
  py::list nodes, edges;
  for (const auto& [id, iv] : plan.placement) {
    if (iv.empty()) continue;
    py::dict jn;
    jn["id"] = id;
    jn["start"] = iv.start;
    jn["end"] = iv.end;
    nodes.append(jn);
  }
  for (const PlanEdge& e : plan.edges) {
    py::dict je;
    je["src"] = e.src;
    je["dst"] = e.dst;
    je["flow"] = e.flow;
    je["exec_start"] = e.exec_start;
    je["exec_end"] = e.exec_end;
    edges.append(je);
  }
  root["nodes"] = nodes;
  root["edges"] = edges;
  return py::module_::import("json").attr("dumps")(root, py::arg("indent") = 2, py::arg("ensure_ascii") = false).cast<std::string>() + "\n";
}

PlacementPlan parse_plan(const std::string& text, const std::string& origin) {
  py::object root;
  try {
    root = py::module_::import("json").attr("loads")(text);
  } catch (py::error_already_set& e) {
    throw ParseError(origin + ": invalid JSON: " + e.what());
  }
  PlacementPlan plan;
  try {
    py::dict r = root;
    plan.method = r["method"].cast<std::string>();
    std::string st = r["status"].cast<std::string>();
    plan.status = st == "optimal" ? MilpStatus::kOptimal
                  : st == "feasible" ? MilpStatus::kFeasible
                  : st == "infeasible" ? MilpStatus::kInfeasible
                  : st == "unbounded" ? MilpStatus::kUnbounded
                                      : MilpStatus::kNoIncumbent;
    plan.objective = r["objective"].cast<double>();
    plan.best_bound = r.contains("best_bound") ? r["best_bound"].cast<double>() : plan.objective;
    plan.allow_partial = r["allow_partial"].cast<bool>();
    plan.nodes_explored = r.contains("nodes_explored") ? r["nodes_explored"].cast<long>() : 0;
    for (auto jn : py::list(r["nodes"])) {
      py::dict d = py::reinterpret_borrow<py::dict>(jn);
      plan.placement[d["id"].cast<std::string>()] = {d["start"].cast<int>(), d["end"].cast<int>()};
    }
    for (auto je : py::list(r["edges"])) {
      py::dict d = py::reinterpret_borrow<py::dict>(je);
      PlanEdge e;
      e.src = d["src"].cast<std::string>();
      e.dst = d["dst"].cast<std::string>();
      e.flow = d["flow"].cast<double>();
      e.exec_start = d["exec_start"].cast<int>();
      e.exec_end = d["exec_end"].cast<int>();
      plan.edges.push_back(e);
    }
  } catch (py::error_already_set& e) {
    throw ParseError(origin + ": bad plan structure: " + e.what());
  } catch (py::cast_error& e) {
    throw ParseError(origin + ": bad plan structure: " + e.what());
  }
  return plan;
}

std::string read_file(const std::string& path) {
  py::object f;
  try {
    f = py::module_::import("builtins").attr("open")(path);
  } catch (py::error_already_set&) {
    throw ParseError(path + ": cannot open file");
  }
  std::string s = f.attr("read")().cast<std::string>();
  f.attr("close")();
  return s;
}

void write_file(const std::string& path, const std::string& text) {
  py::object f;
  try {
    f = py::module_::import("builtins").attr("open")(path, "w");
  } catch (py::error_already_set&) {
    throw ParseError(path + ": cannot open for writing");
  }
  f.attr("write")(text);
  f.attr("close")();
}

// --- generate_trace (workload.cpp:37-57 with rng.hpp:11-54) -------------------
// std::mt19937_64 is fully specified by the standard, and the transforms are
// the reference's hand-rolled ones, so the trace is byte-identical.
struct TraceRng {
  std::mt19937_64 eng;
  double spare = 0;
  bool have = false;
  explicit TraceRng(uint64_t s) : eng(s) {}
  double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    double u1 = uniform(), u2 = uniform();
    while (u1 <= 1e-300) u1 = uniform();
    double r = std::sqrt(-2.0 * std::log(u1));
    double th = 2.0 * M_PI * u2;
    spare = r * std::sin(th);
    have = true;
    return r * std::cos(th);
  }
  double exponential(double rate) {
    double u = uniform();
    while (u <= 1e-300) u = uniform();
    return -std::log(u) / rate;
  }
};

py::tuple generate_trace(int count, double rate, const std::string& mode, uint64_t seed, double mean_input,
                         double mean_output, int max_input, int max_output, double sigma) {
  if (count < 0) throw ValidationError("trace count must be non-negative");
  if (mode != "online" && mode != "offline")
    throw ValidationError("unknown trace mode '" + mode + "' (expected online or offline)");
  const bool online = mode == "online";
  if (online && rate <= 0) throw ValidationError("online traces need a positive arrival rate");
  TraceRng rng(seed);
  py::array_t<double> arr(count);
  py::array_t<int32_t> in(count), out(count);
  auto a = arr.mutable_unchecked<1>();
  auto ii = in.mutable_unchecked<1>();
  auto oo = out.mutable_unchecked<1>();
  auto sample = [&](double mean, int cap) {
    double mu = std::log(mean) - 0.5 * sigma * sigma;
    for (int t = 0; t < 10000; ++t) {
      int len = static_cast<int>(std::llround(std::exp(mu + sigma * rng.normal())));
      if (len >= 1 && len <= cap) return len;
    }
    throw InternalError("length sampler rejected 10000 draws; check mean/cap");
  };
  double t = 0;
  for (int i = 0; i < count; ++i) {
    if (online) t += rng.exponential(rate);
    a(i) = online ? t : 0.0;
    ii(i) = sample(mean_input, max_input);
    oo(i) = sample(mean_output, max_output);
  }
  return py::make_tuple(arr, in, out);
}

// --- the reference planner / simulator linked over this engine ---------------
// lib/libhelio_planner.so (include/helio_planner.h), next to libhelio.so;
// loaded on first use so the scoring surface works without it.
struct Planner {
  decltype(&helio_planner_plan_milp) plan_milp = nullptr;
  decltype(&helio_planner_simulate) simulate = nullptr;
  decltype(&helio_planner_prune_links) prune_links = nullptr;
  decltype(&helio_planner_upper_bound) upper_bound = nullptr;
  decltype(&helio_planner_free) free = nullptr;
  decltype(&helio_planner_layout) layout = nullptr;
};

const Planner& planner() {
  static Planner p;
  static std::string error;
  static bool tried = false;
  if (!tried) {
    tried = true;
    Dl_info info{};
    std::string path = "libhelio_planner.so";
    if (dladdr(reinterpret_cast<void*>(&planner), &info) && info.dli_fname) {
      std::string self = info.dli_fname;
      path = self.substr(0, self.rfind('/') + 1) + "lib/libhelio_planner.so";
    }
    void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      error = dlerror();
    } else {
      p.plan_milp = reinterpret_cast<decltype(p.plan_milp)>(dlsym(h, "helio_planner_plan_milp"));
      p.simulate = reinterpret_cast<decltype(p.simulate)>(dlsym(h, "helio_planner_simulate"));
      p.prune_links = reinterpret_cast<decltype(p.prune_links)>(dlsym(h, "helio_planner_prune_links"));
      p.upper_bound = reinterpret_cast<decltype(p.upper_bound)>(dlsym(h, "helio_planner_upper_bound"));
      p.free = reinterpret_cast<decltype(p.free)>(dlsym(h, "helio_planner_free"));
      p.layout = reinterpret_cast<decltype(p.layout)>(dlsym(h, "helio_planner_layout"));
      if (!p.plan_milp || !p.simulate || !p.prune_links || !p.upper_bound || !p.free || !p.layout) {
        error = "missing symbols";
      } else {
        // objects cross this boundary by pointer: the reference's layouts must be ours
        int64_t theirs[8] = {0};
        const int64_t ours[] = {(int64_t)sizeof(ClusterSpec), (int64_t)sizeof(PlacementPlan),
                                (int64_t)sizeof(FlowGraph), (int64_t)sizeof(Scheduler), (int64_t)sizeof(IwrrPicker),
                                (int64_t)sizeof(Rng), (int64_t)alignof(Scheduler)};
        const int n = p.layout(theirs, 8);
        for (int i = 0; i < 7 && error.empty(); ++i)
          if (n < 7 || theirs[i] != ours[i]) error = "type layouts differ from the reference's (field " + std::to_string(i) + ")";
      }
    }
  }
  if (!error.empty())
    throw InternalError("the reference planner/simulator library (lib/libhelio_planner.so, built by build.py from "
                        "/root/reference) is unavailable: " + error);
  return p;
}

void planner_check(int rc, const char* err) {
  switch (rc) {
    case 0: return;
    case 1: throw ParseError(err);
    case 2: throw ValidationError(err);
    default: throw InternalError(err);
  }
}

py::object json_loads(const char* text) { return py::module_::import("json").attr("loads")(py::str(text)); }

// generate_trace as the reference binding returns it: a list of
// (arrival_s, input_len, output_len) tuples (proj/bindings/pymodule.cpp:179-195)
py::list generate_trace_list(int count, double rate, const std::string& mode, uint64_t seed, double mean_input,
                             double mean_output) {
  py::tuple t = generate_trace(count, rate, mode, seed, mean_input, mean_output, 2048, 1024, 0.496);
  auto a = t[0].cast<py::array_t<double>>().unchecked<1>();
  auto i = t[1].cast<py::array_t<int32_t>>().unchecked<1>();
  auto o = t[2].cast<py::array_t<int32_t>>().unchecked<1>();
  py::list out;
  for (py::ssize_t k = 0; k < a.shape(0); ++k) out.append(py::make_tuple(a(k), i(k), o(k)));
  return out;
}

// Python Scheduler: owns a copy of the cluster and the plan, since the
// reference Scheduler keeps `const ClusterSpec&` (scheduler.hpp:83).
struct PyScheduler {
  std::unique_ptr<ClusterSpec> cluster;
  std::unique_ptr<Scheduler> sched;
};

// NCCL communicator and multi-device handles (csrc/multi.cu).
struct PyComm {
  void* comm = nullptr;
  ~PyComm() { helio_gpu_nccl_comm_destroy(comm); }
};

struct PyMulti {
  helio_gpu_multi* m = nullptr;
  int N = 0;
  std::vector<int32_t> kmax;
  std::string mode = "parity";
  ~PyMulti() { helio_gpu_multi_destroy(m); }
};

// --- batched engine handle ---------------------------------------------------

struct PyEngine {
  std::shared_ptr<gpu::Engine> eng;
  ClusterSpec cluster;
};

py::array_t<int16_t> as_rows(const py::array& a, int N) {
  auto arr = py::array_t<int16_t, py::array::c_style | py::array::forcecast>::ensure(a);
  if (!arr) throw ValidationError("placements must be an int16 array of shape (B, N, 2)");
  if (arr.ndim() == 2 && arr.shape(0) == N && arr.shape(1) == 2) arr = arr.reshape({(py::ssize_t)1, (py::ssize_t)N, (py::ssize_t)2});
  if (arr.ndim() != 3 || arr.shape(1) != N || arr.shape(2) != 2)
    throw ValidationError("placements must have shape (B, " + std::to_string(N) + ", 2)");
  return arr;
}

py::tuple engine_score(PyEngine& pe, const py::array& pl, bool allow_partial) {
  auto rows = as_rows(pl, pe.eng->num_nodes());
  const int64_t B = rows.shape(0);
  py::array_t<double> vals(B);
  py::array_t<int32_t> st(B);
  {
    py::gil_scoped_release rel;
    pe.eng->check(helio_gpu_score_host(pe.eng->ctx(), rows.data(), B, allow_partial ? 1 : 0, vals.mutable_data(),
                                       st.mutable_data()),
                  "helio_gpu_score_host");
  }
  return py::make_tuple(vals, st);
}

py::tuple engine_flows(PyEngine& pe, const py::array& pl, bool allow_partial, int max_edges) {
  auto rows = as_rows(pl, pe.eng->num_nodes());
  const int64_t K = rows.shape(0);
  if (max_edges <= 0) max_edges = pe.eng->num_nodes() + pe.eng->num_links() + 1;
  py::array_t<int32_t> nv(K), ne(K), st(K);
  py::array_t<double> vals(K);
  std::vector<helio_edge> ed((size_t)K * max_edges);
  {
    py::gil_scoped_release rel;
    pe.eng->check(helio_gpu_flows_host(pe.eng->ctx(), rows.data(), K, allow_partial ? 1 : 0, max_edges,
                                       nv.mutable_data(), ne.mutable_data(), ed.data(), vals.mutable_data(),
                                       st.mutable_data()),
                  "helio_gpu_flows_host");
  }
  // edges as a structured numpy block: int32 [K, max_edges, 8] + float64 [K, max_edges, 2]
  py::array_t<int32_t> ints({(py::ssize_t)K, (py::ssize_t)max_edges, (py::ssize_t)8});
  py::array_t<double> dbl({(py::ssize_t)K, (py::ssize_t)max_edges, (py::ssize_t)2});
  auto I = ints.mutable_unchecked<3>();
  auto D = dbl.mutable_unchecked<3>();
  for (int64_t k = 0; k < K; ++k)
    for (int e = 0; e < max_edges; ++e) {
      const helio_edge& x = ed[(size_t)k * max_edges + e];
      I(k, e, 0) = x.u; I(k, e, 1) = x.v; I(k, e, 2) = x.kind; I(k, e, 3) = x.exec_start;
      I(k, e, 4) = x.exec_end; I(k, e, 5) = x.src_node; I(k, e, 6) = x.dst_node; I(k, e, 7) = 0;
      D(k, e, 0) = x.cap; D(k, e, 1) = x.flow;
    }
  return py::make_tuple(vals, st, nv, ne, ints, dbl);
}

py::tuple engine_route(PyEngine& pe, const py::array& placement_row, const py::array& plan_edges_i,
                       const py::array& plan_flows, const py::array& in_len, const py::array& out_len,
                       int max_hops, bool exec_ranges) {
  const int N = pe.eng->num_nodes();
  auto row = as_rows(placement_row, N);
  auto ei = py::array_t<int32_t, py::array::c_style | py::array::forcecast>::ensure(plan_edges_i);
  auto ef = py::array_t<double, py::array::c_style | py::array::forcecast>::ensure(plan_flows);
  auto iin = py::array_t<int32_t, py::array::c_style | py::array::forcecast>::ensure(in_len);
  auto iout = py::array_t<int32_t, py::array::c_style | py::array::forcecast>::ensure(out_len);
  if (ei.ndim() != 2 || ei.shape(1) != 4 || ef.ndim() != 1 || ef.shape(0) != ei.shape(0))
    throw ValidationError("plan edges must be int32 (E, 4) [src, dst, exec_start, exec_end] + float64 (E,) flows");
  const int E = (int)ei.shape(0);
  std::vector<helio_plan_edge> pe_(E);
  for (int i = 0; i < E; ++i) {
    pe_[i].src_node = ei.at(i, 0);
    pe_[i].dst_node = ei.at(i, 1);
    pe_[i].exec_start = ei.at(i, 2);
    pe_[i].exec_end = ei.at(i, 3);
    pe_[i].flow = ef.at(i);
  }
  const int64_t R = iin.size();
  if (iout.size() != R) throw ValidationError("input/output length arrays differ in size");
  if (max_hops <= 0) {
    // longest route the plan allows: hops along node -> node edges from the
    // coordinator (every hop covers >= 1 layer, so at most L)
    std::vector<std::vector<int>> succ(N + 1);
    for (const auto& x : pe_)
      if (x.dst_node >= 0 && x.src_node >= -1 && x.src_node < N) succ[x.src_node + 1].push_back(x.dst_node + 1);
    std::vector<int> memo(N + 1, -1);
    std::function<int(int, int)> longest = [&](int v, int depth) -> int {
      if (depth > pe.eng->num_layers()) return 0;
      if (memo[v] >= 0) return memo[v];
      int best = 0;
      for (int w : succ[v]) best = std::max(best, 1 + longest(w, depth + 1));
      return memo[v] = best;
    };
    max_hops = std::max(1, std::min(pe.eng->num_layers(), longest(0, 0)));
  }
  const py::ssize_t HS = exec_ranges ? R : 0;
  py::array_t<int32_t> nh(R), hn({(py::ssize_t)R, (py::ssize_t)max_hops}), hs({HS, (py::ssize_t)max_hops}),
      he({HS, (py::ssize_t)max_hops});
  int64_t deferred = 0;
  int rc;
  {
    py::gil_scoped_release rel;
    rc = helio_gpu_route_host(pe.eng->ctx(), row.data(), pe_.data(), E, R, iin.data(), iout.data(), max_hops,
                              nh.mutable_data(), hn.mutable_data(), exec_ranges ? hs.mutable_data() : nullptr,
                              exec_ranges ? he.mutable_data() : nullptr, &deferred);
  }
  pe.eng->check(rc, "helio_gpu_route_host");
  return py::make_tuple(nh, hn, hs, he, deferred);
}

}  // namespace

PYBIND11_MODULE(_helio, m) {
  m.doc() = "B200 placement scoring: flow-graph max-flow and IWRR routing (helio drop-in)";

  py::register_exception<ParseError>(m, "ParseError", PyExc_ValueError);
  py::register_exception<ValidationError>(m, "ValidationError", PyExc_ValueError);
  py::register_exception<InternalError>(m, "InternalError", PyExc_RuntimeError);

  py::class_<ClusterSpec>(m, "Cluster")
      .def_static("from_json", [](const std::string& text) { return parse_cluster(text, "<string>"); })
      .def_static("load", [](const std::string& path) { return parse_cluster(read_file(path), path); })
      .def("to_json", &serialize_cluster)
      .def("save", [](const ClusterSpec& c, const std::string& path) { write_file(path, serialize_cluster(c)); })
      .def("validate", [](const ClusterSpec& c) { validate_cluster(c); })
      .def_property_readonly("num_layers", [](const ClusterSpec& c) { return c.model.num_layers; })
      .def_property_readonly("coordinator", [](const ClusterSpec& c) { return c.coordinator_id; })
      .def_property_readonly("node_ids", [](const ClusterSpec& c) {
        std::vector<std::string> ids;
        for (const NodeSpec& n : c.nodes) ids.push_back(n.id);
        return ids;
      })
      .def_property_readonly("num_links", [](const ClusterSpec& c) { return (int)c.links.size(); })
      .def("max_layers", [](const ClusterSpec& c, const std::string& id) {
        int i = c.node_index(id);
        if (i < 0) throw ValidationError("unknown node '" + id + "'");
        return c.max_layers(c.nodes[i]);
      })
      .def("compute_edge_capacity", [](const ClusterSpec& c, const std::string& id, int j) {
        int i = c.node_index(id);
        if (i < 0) throw ValidationError("unknown node '" + id + "'");
        return compute_edge_capacity(c, c.nodes[i], j);
      })
      .def("__repr__", [](const ClusterSpec& c) {
        return "<Cluster '" + c.model.name + "': " + std::to_string(c.nodes.size()) + " nodes, " +
               std::to_string(c.model.num_layers) + " layers>";
      });

  py::class_<PlacementPlan>(m, "Plan")
      .def_static("from_json", [](const std::string& text) { return parse_plan(text, "<string>"); })
      .def_static("load", [](const std::string& path) { return parse_plan(read_file(path), path); })
      .def("to_json", &serialize_plan)
      .def("save", [](const PlacementPlan& p, const std::string& path) { write_file(path, serialize_plan(p)); })
      .def_property_readonly("method", [](const PlacementPlan& p) { return p.method; })
      .def_property_readonly("objective", [](const PlacementPlan& p) { return p.objective; })
      .def_property_readonly("best_bound", [](const PlacementPlan& p) { return p.best_bound; })
      .def_property_readonly("optimal", [](const PlacementPlan& p) { return p.status == MilpStatus::kOptimal; })
      .def_property_readonly("allow_partial", [](const PlacementPlan& p) { return p.allow_partial; })
      .def_property_readonly("placement", [](const PlacementPlan& p) { return placement_to_dict(p.placement); })
      .def_property_readonly("edges",
                             [](const PlacementPlan& p) {
                               py::list out;
                               for (const PlanEdge& e : p.edges)
                                 out.append(py::make_tuple(e.src, e.dst, e.flow, e.exec_start, e.exec_end));
                               return out;
                             })
      .def_property_readonly("warnings", [](const PlacementPlan& p) { return p.warnings; })
      .def("__repr__", [](const PlacementPlan& p) {
        return "<Plan " + p.method + ": " + std::to_string(p.objective) + " tokens/s>";
      });

  py::class_<FlowGraph>(m, "FlowGraph")
      .def_readonly("num_vertices", &FlowGraph::num_vertices)
      .def_readonly("source", &FlowGraph::source)
      .def_readonly("sink", &FlowGraph::sink)
      .def_readonly("vertex_names", &FlowGraph::vertex_names)
      .def_readonly("node_vertices", &FlowGraph::node_vertices)
      .def_property_readonly("edges",
                             [](const FlowGraph& g) {
                               py::list out;
                               for (const FlowEdge& e : g.edges)
                                 out.append(py::make_tuple(e.u, e.v, e.cap, e.flow, static_cast<int>(e.kind), e.src_id,
                                                           e.dst_id, e.exec_start, e.exec_end));
                               return out;
                             })
      .def("to_dot", [](const FlowGraph& g) { return to_dot(g); })
      .def("min_cut_source_side", [](const FlowGraph& g) { return min_cut_source_side(g); });

  m.def(
      "plan",
      [](const ClusterSpec& c, const std::string& method, bool allow_partial, double prune_degree, double gap,
         double time_budget_s, long node_budget, bool warm_starts, bool lex_tiebreak, int max_moves) {
        // pymodule.cpp:130-157: "milp" is the reference's planner linked over
        // this engine (every max-flow it takes runs on the B200); the
        // heuristics wrap their placement into a plan; "local" / "sampled"
        // are this engine's device searches
        if (method == "milp") {
          const Planner& pl = planner();
          helio_plan_options o{allow_partial ? 1 : 0, prune_degree, gap, time_budget_s, (int64_t)node_budget,
                               warm_starts ? 1 : 0, lex_tiebreak ? 1 : 0};
          PlacementPlan plan;
          char err[1024] = {0};
          int rc;
          {
            py::gil_scoped_release rel;
            rc = pl.plan_milp(&c, &o, &plan, err, sizeof(err));
          }
          planner_check(rc, err);
          return plan;
        }
        if (method == "swarm" || method == "petals" || method == "sp") {
          HeuristicResult h = method == "swarm"    ? swarm_placement(c)
                              : method == "petals" ? petals_placement(c)
                                                   : separate_pipelines_placement(c);
          PlacementPlan plan = plan_from_placement(c, h.placement, allow_partial, method);
          for (const std::string& w : h.warnings) plan.warnings.push_back(w);
          return plan;
        }
        if (method == "local" || method == "sampled") {
          // seeds as the reference's MILP warm starts (placement.cpp:491-498)
          std::vector<HeuristicResult> seeds{swarm_placement(c), petals_placement(c)};
          if (std::all_of(c.nodes.begin(), c.nodes.end(), [](const NodeSpec& n) { return !n.type.empty(); }))
            seeds.push_back(separate_pipelines_placement(c));
          Placement best;
          double best_value = 0;
          std::vector<std::string> warnings;
          for (const HeuristicResult& h : seeds) {
            for (const std::string& w : h.warnings) warnings.push_back(w);
            LocalSearchResult r;
            {
              py::gil_scoped_release rel;
              r = method == "local" ? local_search_placement(c, h.placement, allow_partial, max_moves)
                                    : c.nodes.size() <= 64
                                        ? sampled_search_placement(c, h.placement, allow_partial)
                                        // large sparse clusters score ~40x slower per graph
                                        // (syn256): more, smaller rounds
                                        : sampled_search_placement(c, h.placement, allow_partial, 60, 1 << 16);
            }
            if (r.value > best_value) {
              best_value = r.value;
              best = r.placement;
            }
          }
          PlacementPlan plan = plan_from_placement(c, best, allow_partial, method);
          for (const std::string& w : warnings) plan.warnings.push_back(w);
          return plan;
        }
        throw ValidationError("unknown method '" + method + "'");
      },
      py::arg("cluster"), py::arg("method") = "milp", py::arg("allow_partial") = true,
      py::arg("prune_degree") = 0.0, py::arg("gap") = 0.02, py::arg("time_budget_s") = 600.0,
      py::arg("node_budget") = -1, py::arg("warm_starts") = true, py::arg("lex_tiebreak") = true,
      py::arg("max_moves") = -1,
      "Compute a placement plan (method: milp, swarm, petals, or sp, as the reference; plus local = device "
      "local search from the heuristic seeds, sampled = local search, sampled multi-node search, local search "
      "again from each seed).");

  m.def(
      "simulate",
      [](const ClusterSpec& c, const PlacementPlan& plan, const py::list& trace, const std::string& mode,
         const std::string& scheduler, uint64_t seed, double horizon_s, double warmup_s) {
        // pymodule.cpp:197-218: the reference's discrete-event simulator
        // (sim.cpp) over this engine's Scheduler
        std::vector<double> arr;
        std::vector<int32_t> in, out;
        for (const auto& row : trace) {
          auto t = row.cast<std::tuple<double, int, int>>();
          arr.push_back(std::get<0>(t));
          in.push_back(std::get<1>(t));
          out.push_back(std::get<2>(t));
        }
        if (mode != "online" && mode != "offline")
          throw ValidationError("unknown trace mode '" + mode + "' (expected online or offline)");
        const SchedPolicy pol = sched_policy_from_str(scheduler);
        helio_sim_config cfg{mode == "online" ? 1 : 0, horizon_s, mode == "online" ? warmup_s : 0.0,
                             static_cast<int32_t>(pol), seed, 32, 2048, 0.01, 0.002};
        const Planner& pl = planner();
        char* js = nullptr;
        char err[1024] = {0};
        int rc;
        {
          py::gil_scoped_release rel;
          rc = pl.simulate(&c, &plan, (int64_t)arr.size(), arr.data(), in.data(), out.data(), &cfg, &js, err,
                           sizeof(err));
        }
        planner_check(rc, err);
        py::object d = json_loads(js);
        pl.free(js);
        return d;
      },
      py::arg("cluster"), py::arg("plan"), py::arg("trace"), py::arg("mode") = "online",
      py::arg("scheduler") = "iwrr", py::arg("seed") = 1, py::arg("horizon_s") = 120.0,
      py::arg("warmup_s") = 20.0,
      "Run a trace through the reference's discrete-event simulator over this engine; returns a metrics dict.");

  m.def(
      "prune_links",
      [](const ClusterSpec& c, double target_avg_degree) {
        const Planner& pl = planner();
        ClusterSpec out;
        int32_t removed = 0;
        double before = 0, after = 0;
        char* warn = nullptr;
        char err[1024] = {0};
        planner_check(pl.prune_links(&c, target_avg_degree, &out, &removed, &before, &after, &warn, err,
                                     sizeof(err)),
                      err);
        py::dict rep;
        rep["links_removed"] = removed;
        rep["avg_degree_before"] = before;
        rep["avg_degree_after"] = after;
        rep["warnings"] = json_loads(warn);
        pl.free(warn);
        return py::make_tuple(out, rep);
      },
      py::arg("cluster"), py::arg("target_avg_degree"),
      "The reference's prune_links (placement.cpp:230-332): (pruned cluster, report dict).");

  m.def(
      "throughput_upper_bound",
      [](const ClusterSpec& c) {
        double v = 0;
        char err[1024] = {0};
        planner_check(planner().upper_bound(&c, &v, err, sizeof(err)), err);
        return v;
      },
      py::arg("cluster"), "Compute-only throughput ceiling for a cluster.");

  py::class_<PyScheduler>(m, "Scheduler")
      .def(py::init([](const ClusterSpec& c, const PlacementPlan& plan, const std::string& policy, uint64_t seed) {
             auto ps = std::make_unique<PyScheduler>();
             ps->cluster = std::make_unique<ClusterSpec>(c);
             ps->sched = std::make_unique<Scheduler>(*ps->cluster, plan, sched_policy_from_str(policy), seed);
             return ps;
           }),
           py::arg("cluster"), py::arg("plan"), py::arg("policy") = "iwrr", py::arg("seed") = 1)
      .def(
          "admit",
          [](PyScheduler& s, long request_id, int input_len) -> py::object {
            auto r = s.sched->admit(request_id, input_len);
            if (!r) return py::none();
            py::list hops;
            for (const RouteHop& h : *r) hops.append(py::make_tuple(h.node, h.exec_start, h.exec_end));
            return std::move(hops);
          },
          py::arg("request_id"), py::arg("input_len"),
          "Scheduler::admit (scheduler.cpp:158-181): [(node, exec_start, exec_end)] or None when deferred.")
      .def("complete", [](PyScheduler& s, long id, int out) { s.sched->complete(id, out); }, py::arg("request_id"),
           py::arg("output_len"))
      .def("kv_estimate", [](const PyScheduler& s, const std::string& n) { return s.sched->kv_estimate(n); })
      .def("kv_capacity", [](const PyScheduler& s, const std::string& n) { return s.sched->kv_capacity(n); })
      .def_property_readonly("avg_output", [](const PyScheduler& s) { return s.sched->avg_output(); })
      .def(
          "run_ac8",
          [](PyScheduler& s, py::array_t<int32_t, py::array::c_style | py::array::forcecast> in,
             py::array_t<int32_t, py::array::c_style | py::array::forcecast> out) {
            // admit(r, in[r]); if admitted complete(r, out[r]) (acceptance_main.cpp:529-537),
            // timed without Python in the loop: (hops per request or -1, seconds)
            const int64_t R = in.size();
            py::array_t<int32_t> nh(R);
            auto n = nh.mutable_unchecked<1>();
            const int32_t* pi = in.data();
            const int32_t* po = out.data();
            double secs = 0;
            {
              py::gil_scoped_release rel;
              const auto t0 = std::chrono::steady_clock::now();
              for (int64_t r = 0; r < R; ++r) {
                auto route = s.sched->admit((long)r, pi[r]);
                if (!route) {
                  n(r) = -1;
                  continue;
                }
                n(r) = (int32_t)route->size();
                s.sched->complete((long)r, po[r]);
              }
              secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            }
            return py::make_tuple(nh, secs);
          },
          py::arg("input_lens"), py::arg("output_lens"));

  m.def(
      "heuristic_placement",
      [](const ClusterSpec& c, const std::string& method) {
        HeuristicResult h;
        if (method == "swarm") h = swarm_placement(c);
        else if (method == "petals") h = petals_placement(c);
        else if (method == "sp") h = separate_pipelines_placement(c);
        else throw ValidationError("unknown method '" + method + "'");
        return py::make_tuple(placement_to_dict(h.placement), h.warnings);
      },
      py::arg("cluster"), py::arg("method"), "(placement, warnings) of a baseline heuristic (heuristics.cpp).");

  m.def(
      "local_search",
      [](const ClusterSpec& c, const py::dict& seed, bool allow_partial, int max_moves, bool swaps) {
        const Placement p = placement_from_dict(seed);
        LocalSearchResult r;
        {
          py::gil_scoped_release rel;
          r = local_search_placement(c, p, allow_partial, max_moves, swaps);
        }
        return py::make_tuple(placement_to_dict(r.placement), r.value, r.moves, r.scored);
      },
      py::arg("cluster"), py::arg("seed"), py::arg("allow_partial") = true, py::arg("max_moves") = -1,
      py::arg("swaps") = true,
      "Device local search from a placement: (placement, value, moves, placements scored).");

  m.def(
      "plan_for_placement",
      [](const ClusterSpec& c, const py::dict& placement, bool allow_partial) {
        return plan_from_placement(c, placement_from_dict(placement), allow_partial, "custom");
      },
      py::arg("cluster"), py::arg("placement"), py::arg("allow_partial") = true,
      "Wrap an explicit {node: (start, end)} placement into a plan (device max-flow).");

  m.def(
      "max_flow_value",
      [](const ClusterSpec& c, const py::dict& placement, bool allow_partial) {
        std::vector<int16_t> row = placement_row(c, placement_from_dict(placement));
        auto eng = gpu::engine_for(c);
        double v = 0;
        int32_t st = 0;
        eng->check(helio_gpu_score_host(eng->ctx(), row.data(), 1, allow_partial ? 1 : 0, &v, &st),
                   "helio_gpu_score_host");
        if (st != HELIO_CAND_OK) throw InternalError("engine rejected a validated placement");
        return v;
      },
      py::arg("cluster"), py::arg("placement"), py::arg("allow_partial") = true,
      "Token throughput of a fixed placement.");

  m.def(
      "build_flow_graph",
      [](const ClusterSpec& c, const py::dict& placement, bool allow_partial) {
        return build_flow_graph(c, placement_from_dict(placement), allow_partial);
      },
      py::arg("cluster"), py::arg("placement"), py::arg("allow_partial") = true);

  m.def("max_flow", [](FlowGraph& g) { return max_flow(g); }, py::arg("graph"),
        "Solve in place (fills edge flows), returns the value.");

  m.def(
      "max_flow_raw",
      [](py::array_t<int32_t, py::array::c_style | py::array::forcecast> n,
         py::array_t<int32_t, py::array::c_style | py::array::forcecast> s,
         py::array_t<int32_t, py::array::c_style | py::array::forcecast> t,
         py::array_t<int64_t, py::array::c_style | py::array::forcecast> off,
         py::array_t<int32_t, py::array::c_style | py::array::forcecast> u,
         py::array_t<int32_t, py::array::c_style | py::array::forcecast> v,
         py::array_t<double, py::array::c_style | py::array::forcecast> cap) {
        const int64_t G = n.size();
        if (s.size() != G || t.size() != G || off.size() != G + 1) throw ValidationError("bad raw graph arrays");
        const int64_t E = off.at(G);
        if (u.size() < E || v.size() < E || cap.size() < E) throw ValidationError("bad raw edge arrays");
        py::array_t<double> vals(G), flows(std::max<int64_t>(E, 0));
        auto eng = gpu::raw_engine();
        int rc;
        {
          py::gil_scoped_release rel;
          rc = helio_gpu_maxflow_raw_host(eng->ctx(), G, n.data(), s.data(), t.data(), off.data(), u.data(), v.data(),
                                          cap.data(), vals.mutable_data(), flows.mutable_data());
        }
        eng->check(rc, "helio_gpu_maxflow_raw_host");
        return py::make_tuple(vals, flows);
      },
      py::arg("n"), py::arg("source"), py::arg("sink"), py::arg("edge_off"), py::arg("u"), py::arg("v"),
      py::arg("cap"), "max_flow on G raw graphs; returns (values[G], flows[E]).");

  m.def("iwrr_weights", [](const std::vector<double>& flows) { return iwrr_weights(flows); });

  py::class_<IwrrPicker>(m, "IwrrPicker")
      .def(py::init<std::vector<long>>())
      .def("next", [](IwrrPicker& p, const std::function<bool(int)>& f) { return p.next(f); })
      .def("next_all", [](IwrrPicker& p, int count) {
        // `count` picks with every candidate eligible
        std::vector<int> out;
        for (int k = 0; k < count; ++k) out.push_back(p.next([](int) { return true; }));
        return out;
      });

  m.def(
      "route_requests",
      [](const ClusterSpec& c, const PlacementPlan& plan, const std::vector<int>& in, const std::vector<int>& out) {
        std::vector<std::optional<std::vector<RouteHop>>> routes;
        {
          py::gil_scoped_release rel;
          routes = route_requests(c, plan, in, out);
        }
        py::list res;
        for (auto& r : routes) {
          if (!r) {
            res.append(py::none());
            continue;
          }
          py::list hops;
          for (auto& h : *r) hops.append(py::make_tuple(h.node, h.exec_start, h.exec_end));
          res.append(hops);
        }
        return res;
      },
      py::arg("cluster"), py::arg("plan"), py::arg("input_lens"), py::arg("output_lens"),
      "IWRR routes in AC8 order (admit then complete); None = deferred.");

  m.def("generate_trace", &generate_trace_list, py::arg("count"), py::arg("rate") = 0.0,
        py::arg("mode") = "offline", py::arg("seed") = 1, py::arg("mean_input") = 763.0,
        py::arg("mean_output") = 232.0, "Sample (arrival_s, input_len, output_len) request tuples.");
  m.def("generate_trace_arrays", &generate_trace, py::arg("count"), py::arg("rate") = 0.0,
        py::arg("mode") = "offline", py::arg("seed") = 1, py::arg("mean_input") = 763.0,
        py::arg("mean_output") = 232.0, py::arg("max_input") = 2048, py::arg("max_output") = 1024,
        py::arg("sigma") = 0.496,
        "generate_trace as three arrays (arrival_s[], input_len[], output_len[]) for large traces.");

  m.def(
      "generate_host",
      [](const std::vector<int32_t>& kmax, int L, uint64_t seed, int64_t first, int64_t B, uint32_t ppm) {
        const int N = (int)kmax.size();
        py::array_t<int16_t> out({(py::ssize_t)B, (py::ssize_t)N, (py::ssize_t)2});
        {
          py::gil_scoped_release rel;
          helio_generate_host(kmax.data(), N, L, seed, first, B, ppm, out.mutable_data());
        }
        return out;
      },
      py::arg("kmax"), py::arg("num_layers"), py::arg("seed"), py::arg("first"), py::arg("count"),
      py::arg("p_uniform_ppm") = 0);

  // torch.distributed, when installed, must own the process's libnccl.so.2
  // (multi.cu binds whichever copy is loaded): import it before NCCL is used
  auto nccl_prepare = [] {
    try {
      py::module_::import("torch");
    } catch (py::error_already_set&) {
    }
  };
  m.def("nccl_unique_id", [nccl_prepare] {
    nccl_prepare();
    std::string id(128, '\0');
    if (helio_gpu_nccl_unique_id(reinterpret_cast<uint8_t*>(&id[0])) != HELIO_OK)
      throw InternalError("ncclGetUniqueId failed");
    return py::bytes(id);
  }, "128-byte NCCL unique id (rank 0 draws it and sends it to every rank).");

  py::class_<PyComm>(m, "NcclComm")
      .def(py::init([nccl_prepare](py::bytes id, int nranks, int rank, int device) {
             nccl_prepare();
             std::string s = id;
             if (s.size() != 128) throw ValidationError("NCCL unique id must be 128 bytes");
             auto c = std::make_unique<PyComm>();
             int rc;
             {
               py::gil_scoped_release rel;
               rc = helio_gpu_nccl_comm_create(reinterpret_cast<const uint8_t*>(s.data()), nranks, rank, device,
                                               &c->comm);
             }
             if (rc != HELIO_OK) throw InternalError("ncclCommInitRank failed");
             return c;
           }),
           py::arg("unique_id"), py::arg("nranks"), py::arg("rank"), py::arg("device"))
      .def_property_readonly("handle", [](const PyComm& c) { return reinterpret_cast<uintptr_t>(c.comm); });

  py::class_<PyMulti>(m, "MultiEngine")
      .def(py::init([](const ClusterSpec& c, const std::vector<int32_t>& devices) {
             auto pm = std::make_unique<PyMulti>();
             int rc = helio_gpu_multi_create(devices.data(), (int32_t)devices.size(), &pm->m);
             if (rc != HELIO_OK)
               throw InternalError("helio: cannot create contexts on the requested devices (helio_gpu_multi_create "
                                   "returned " + std::to_string(rc) + "); this build has no CPU fallback");
             gpu::ClusterDesc desc;
             gpu::make_cluster_desc(c, desc);
             pm->kmax.assign(c.nodes.size(), 0);
             rc = helio_gpu_multi_set_cluster(pm->m, &desc.d, pm->kmax.data());
             if (rc != HELIO_OK) throw ValidationError(helio_gpu_multi_last_error(pm->m));
             pm->N = (int)c.nodes.size();
             return pm;
           }),
           py::arg("cluster"), py::arg("devices"))
      .def_property_readonly("count", [](const PyMulti& p) { return helio_gpu_multi_count(p.m); })
      .def_property_readonly("kmax", [](const PyMulti& p) { return p.kmax; })
      .def_property(
          "mode", [](const PyMulti& p) { return p.mode; },
          [](PyMulti& p, const std::string& mode) {
            if (mode != "parity" && mode != "score") throw ValidationError("mode must be 'parity' or 'score'");
            if (helio_gpu_multi_set_mode(p.m, mode == "score" ? HELIO_MODE_SCORE : HELIO_MODE_PARITY) != HELIO_OK)
              throw InternalError(helio_gpu_multi_last_error(p.m));
            p.mode = mode;
          })
      .def(
          "score_best",
          [](PyMulti& p, const py::array& placements, bool allow_partial) {
            auto rows = as_rows(placements, p.N);
            const int64_t B = rows.shape(0);
            py::array_t<double> vals(B);
            py::array_t<int32_t> st(B);
            double best = 0;
            int64_t idx = -1;
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_multi_score_best_host(p.m, rows.data(), B, allow_partial ? 1 : 0, vals.mutable_data(),
                                                   st.mutable_data(), &best, &idx);
            }
            if (rc != HELIO_OK) throw InternalError(helio_gpu_multi_last_error(p.m));
            return py::make_tuple(vals, st, best, idx);
          },
          py::arg("placements"), py::arg("allow_partial") = true,
          "Score a host batch split over the devices: (values, status, best value, first-max index).")
      .def(
          "score_best_host_ptr",
          [](PyMulti& p, uintptr_t pl, int64_t B, uintptr_t vals, uintptr_t st, bool allow_partial) {
            double best = 0;
            int64_t idx = -1;
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_multi_score_best_host(p.m, reinterpret_cast<const int16_t*>(pl), B, allow_partial ? 1 : 0,
                                                   reinterpret_cast<double*>(vals), reinterpret_cast<int32_t*>(st),
                                                   &best, &idx);
            }
            if (rc != HELIO_OK) throw InternalError(helio_gpu_multi_last_error(p.m));
            return py::make_tuple(best, idx);
          },
          py::arg("placements_ptr"), py::arg("count"), py::arg("values_ptr"), py::arg("status_ptr"),
          py::arg("allow_partial") = true)
      .def(
          "sampled_search",
          [](PyMulti& p, py::array_t<int16_t, py::array::c_style | py::array::forcecast> seed, bool allow_partial,
             int32_t iterations, int64_t batch, int32_t max_changes, uint64_t rng_seed) {
            if (seed.ndim() != 2 || seed.shape(0) != p.N || seed.shape(1) != 2)
              throw py::value_error("seed must be int16 [num_nodes, 2]");
            py::array_t<int16_t> row({(py::ssize_t)p.N, (py::ssize_t)2});
            double value = 0;
            int32_t improvements = 0;
            int64_t scored = 0;
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_multi_sampled_search(p.m, seed.data(), allow_partial ? 1 : 0, iterations, batch,
                                                  max_changes, rng_seed, &value, row.mutable_data(), &improvements,
                                                  &scored);
            }
            if (rc != HELIO_OK) throw InternalError(helio_gpu_multi_last_error(p.m));
            return py::make_tuple(value, row, improvements, scored);
          },
          py::arg("seed"), py::arg("allow_partial") = true, py::arg("iterations") = 20,
          py::arg("batch") = 1 << 20, py::arg("max_changes") = 3, py::arg("rng_seed") = 1,
          "Engine.sampled_search with each round's mutants split over the devices (same result as one device).");

  py::class_<PyEngine>(m, "Engine")
      .def(py::init([](const ClusterSpec& c, int device) {
             auto pe = new PyEngine();
             pe->cluster = c;
             pe->eng = std::make_shared<gpu::Engine>(device);
             pe->eng->set_cluster(pe->cluster);
             return pe;
           }),
           py::arg("cluster"), py::arg("device") = 0)
      .def_property_readonly("num_nodes", [](const PyEngine& e) { return e.eng->num_nodes(); })
      .def_property_readonly("num_layers", [](const PyEngine& e) { return e.eng->num_layers(); })
      .def_property_readonly("kmax", [](const PyEngine& e) { return e.eng->kmax(); })
      .def_property_readonly("device", [](const PyEngine& e) { return e.eng->device(); })
      .def_property_readonly("launch_count", [](const PyEngine& e) { return helio_gpu_launch_count(e.eng->ctx()); })
      .def("last_kernel_ms", [](const PyEngine& e) { return helio_gpu_last_kernel_ms(e.eng->ctx()); })
      .def_property(
          "mode", [](const PyEngine& e) { return helio_gpu_get_mode(e.eng->ctx()) == HELIO_MODE_SCORE ? "score" : "parity"; },
          [](PyEngine& e, const std::string& m) {
            if (m != "parity" && m != "score") throw ValidationError("mode must be 'parity' or 'score'");
            e.eng->check(helio_gpu_set_mode(e.eng->ctx(), m == "score" ? HELIO_MODE_SCORE : HELIO_MODE_PARITY),
                         "helio_gpu_set_mode");
          },
          "'parity' (bit-exact FIFO replay, default) or 'score' (value-only Edmonds-Karp)")
      .def("score", &engine_score, py::arg("placements"), py::arg("allow_partial") = true,
           "Host arrays in, (values, status) out; copies inside.")
      .def(
          "score_device",
          [](PyEngine& e, uintptr_t pl, int64_t B, uintptr_t values, uintptr_t status, bool allow_partial,
             uintptr_t stream) {
            e.eng->check(helio_gpu_score(e.eng->ctx(), reinterpret_cast<const int16_t*>(pl), B, allow_partial ? 1 : 0,
                                         reinterpret_cast<double*>(values), reinterpret_cast<int32_t*>(status),
                                         reinterpret_cast<void*>(stream)),
                         "helio_gpu_score");
          },
          py::arg("placements_ptr"), py::arg("count"), py::arg("values_ptr"), py::arg("status_ptr"),
          py::arg("allow_partial") = true, py::arg("stream") = 0)
      .def(
          "score_host_ptr",
          [](PyEngine& e, uintptr_t pl, int64_t B, uintptr_t values, uintptr_t status, bool allow_partial) {
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_score_host(e.eng->ctx(), reinterpret_cast<const int16_t*>(pl), B, allow_partial ? 1 : 0,
                                        reinterpret_cast<double*>(values), reinterpret_cast<int32_t*>(status));
            }
            e.eng->check(rc, "helio_gpu_score_host");
          },
          py::arg("placements_ptr"), py::arg("count"), py::arg("values_ptr"), py::arg("status_ptr"),
          py::arg("allow_partial") = true)
      .def(
          "score_best_host_ptr",
          [](PyEngine& e, uintptr_t pl, int64_t B, uintptr_t values, uintptr_t status, bool allow_partial) {
            double best = 0;
            int64_t idx = -1;
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_score_best_host(e.eng->ctx(), reinterpret_cast<const int16_t*>(pl), B,
                                             allow_partial ? 1 : 0, reinterpret_cast<double*>(values),
                                             reinterpret_cast<int32_t*>(status), &best, &idx);
            }
            e.eng->check(rc, "helio_gpu_score_best_host");
            return py::make_tuple(best, idx);
          },
          py::arg("placements_ptr"), py::arg("count"), py::arg("values_ptr"), py::arg("status_ptr"),
          py::arg("allow_partial") = true, "Host buffers: every value + status, and the first maximum.")
      .def(
          "generate_device",
          [](PyEngine& e, uint64_t seed, int64_t first, int64_t B, uint32_t ppm, uintptr_t out, uintptr_t stream) {
            e.eng->check(helio_gpu_generate(e.eng->ctx(), seed, first, B, ppm, reinterpret_cast<int16_t*>(out),
                                            reinterpret_cast<void*>(stream)),
                         "helio_gpu_generate");
          },
          py::arg("seed"), py::arg("first"), py::arg("count"), py::arg("p_uniform_ppm"), py::arg("out_ptr"),
          py::arg("stream") = 0)
      .def(
          "generate_walk_device",
          [](PyEngine& e, uint64_t seed, int64_t first, int64_t B, uintptr_t out, uintptr_t stream) {
            e.eng->check(helio_gpu_generate_walk(e.eng->ctx(), seed, first, B, reinterpret_cast<int16_t*>(out),
                                                 reinterpret_cast<void*>(stream)),
                         "helio_gpu_generate_walk");
          },
          py::arg("seed"), py::arg("first"), py::arg("count"), py::arg("out_ptr"), py::arg("stream") = 0)
      .def(
          "generate_walk_host",
          [](PyEngine& e, uint64_t seed, int64_t first, int64_t B) {
            const int N = e.eng->num_nodes();
            py::array_t<int16_t> out({(py::ssize_t)B, (py::ssize_t)N, (py::ssize_t)2});
            e.eng->check(helio_gpu_generate_walk_host(e.eng->ctx(), seed, first, B, out.mutable_data()),
                         "helio_gpu_generate_walk_host");
            return out;
          },
          py::arg("seed"), py::arg("first"), py::arg("count"))
      .def_property_readonly("csr_slab_bytes", [](const PyEngine& e) { return helio_gpu_csr_slab_bytes(e.eng->ctx()); })
      .def(
          "build_csr_device",
          [](PyEngine& e, uintptr_t pl, int64_t B, uintptr_t slabs, uintptr_t status, bool allow_partial,
             uintptr_t stream) {
            e.eng->check(helio_gpu_build_csr(e.eng->ctx(), reinterpret_cast<const int16_t*>(pl), B, allow_partial ? 1 : 0,
                                             reinterpret_cast<void*>(slabs), reinterpret_cast<int32_t*>(status),
                                             reinterpret_cast<void*>(stream)),
                         "helio_gpu_build_csr");
          },
          py::arg("placements_ptr"), py::arg("count"), py::arg("slabs_ptr"), py::arg("status_ptr"),
          py::arg("allow_partial") = true, py::arg("stream") = 0)
      .def(
          "solve_csr_device",
          [](PyEngine& e, uintptr_t slabs, int64_t B, uintptr_t values, uintptr_t status, uintptr_t stream) {
            e.eng->check(helio_gpu_solve_csr(e.eng->ctx(), reinterpret_cast<const void*>(slabs), B,
                                             reinterpret_cast<double*>(values), reinterpret_cast<int32_t*>(status),
                                             reinterpret_cast<void*>(stream)),
                         "helio_gpu_solve_csr");
          },
          py::arg("slabs_ptr"), py::arg("count"), py::arg("values_ptr"), py::arg("status_ptr"), py::arg("stream") = 0)
      .def(
          "argmax_device",
          [](PyEngine& e, uintptr_t values, uintptr_t status, int64_t B, int64_t base, uintptr_t best, uintptr_t index,
             uintptr_t stream) {
            e.eng->check(helio_gpu_argmax(e.eng->ctx(), reinterpret_cast<const double*>(values),
                                          reinterpret_cast<const int32_t*>(status), B, base,
                                          reinterpret_cast<double*>(best), reinterpret_cast<int64_t*>(index),
                                          reinterpret_cast<void*>(stream)),
                         "helio_gpu_argmax");
          },
          py::arg("values_ptr"), py::arg("status_ptr"), py::arg("count"), py::arg("index_base"), py::arg("best_ptr"),
          py::arg("index_ptr"), py::arg("stream") = 0)
      .def(
          "check_division",
          [](PyEngine& e, int64_t count, uint64_t seed) {
            int64_t bad = -1;
            e.eng->check(helio_gpu_check_division(e.eng->ctx(), count, seed, &bad), "helio_gpu_check_division");
            return bad;
          },
          py::arg("count"), py::arg("seed") = 1,
          "Mismatches of the masked routing replay's reciprocal-based division against IEEE division.")
      .def(
          "argmax_ranked",
          [](PyEngine& e, uintptr_t values, uintptr_t status, int64_t B, int64_t base, uintptr_t best, uintptr_t index,
             uintptr_t comm, uintptr_t stream) {
            e.eng->check(helio_gpu_argmax_ranked(e.eng->ctx(), reinterpret_cast<const double*>(values),
                                                 reinterpret_cast<const int32_t*>(status), B, base,
                                                 reinterpret_cast<double*>(best), reinterpret_cast<int64_t*>(index),
                                                 reinterpret_cast<void*>(comm), reinterpret_cast<void*>(stream)),
                         "helio_gpu_argmax_ranked");
          },
          py::arg("values_ptr"), py::arg("status_ptr"), py::arg("count"), py::arg("index_base"), py::arg("best_ptr"),
          py::arg("index_ptr"), py::arg("comm"), py::arg("stream") = 0,
          "This rank's shard argmax, all-gathered over the NCCL communicator `comm` (NcclComm.handle) and reduced "
          "to the global first maximum on every rank (device pointers, stream ordered).")
      .def("flows", &engine_flows, py::arg("placements"), py::arg("allow_partial") = true, py::arg("max_edges") = 0,
           "(values, status, num_vertices, num_edges, int32 [K,E,8] {u,v,kind,exec_start,exec_end,src,dst,0}, "
           "float64 [K,E,2] {cap,flow})")
      .def("route", &engine_route, py::arg("placement_row"), py::arg("plan_edges"), py::arg("plan_flows"),
           py::arg("input_lens"), py::arg("output_lens"), py::arg("max_hops") = 0, py::arg("exec_ranges") = true)
      .def(
          "plan_edges",
          [](PyEngine& e, const py::array& placement_row, bool allow_partial) {
            // plan_from_placement's edge filter (placement.cpp:440-455) over the
            // device's PARITY flows: non-compute edges with flow > 1e-9, the
            // coordinator as -1.  Returns (int32 [E,4] src,dst,exec_start,exec_end;
            // float64 [E] flow; objective).
            const int N = e.eng->num_nodes();
            auto row = as_rows(placement_row, N);
            if (row.shape(0) != 1) throw ValidationError("plan_edges takes one placement row");
            const int max_e = N + e.eng->num_links() + 1;
            std::vector<helio_edge> ed(max_e);
            int32_t nv = 0, ne = 0, st = 0;
            double val = 0;
            e.eng->check(helio_gpu_flows_host(e.eng->ctx(), row.data(), 1, allow_partial ? 1 : 0, max_e, &nv, &ne,
                                              ed.data(), &val, &st),
                         "helio_gpu_flows_host");
            if (st != HELIO_CAND_OK) throw ValidationError("placement rejected (status " + std::to_string(st) + ")");
            std::vector<const helio_edge*> keep;
            for (int i = 0; i < ne; ++i)
              if (ed[i].kind != HELIO_EDGE_COMPUTE && ed[i].flow > 1e-9) keep.push_back(&ed[i]);
            py::array_t<int32_t> ints({(py::ssize_t)keep.size(), (py::ssize_t)4});
            py::array_t<double> fl((py::ssize_t)keep.size());
            for (size_t i = 0; i < keep.size(); ++i) {
              const helio_edge& x = *keep[i];
              ints.mutable_at(i, 0) = x.kind == HELIO_EDGE_COORD_OUT ? -1 : x.src_node;
              ints.mutable_at(i, 1) = x.kind == HELIO_EDGE_COORD_IN ? -1 : x.dst_node;
              ints.mutable_at(i, 2) = x.exec_start;
              ints.mutable_at(i, 3) = x.exec_end;
              fl.mutable_at(i) = x.flow;
            }
            return py::make_tuple(ints, fl, val);
          },
          py::arg("placement_row"), py::arg("allow_partial") = true)
      .def(
          "best_exhaustive",
          [](PyEngine& e, bool allow_partial, int64_t max_leaves) {
            const int N = e.eng->num_nodes();
            py::array_t<int16_t> row({(py::ssize_t)N, (py::ssize_t)2});
            double best = 0;
            int64_t scored = 0, total = 0;
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_best_exhaustive(e.eng->ctx(), allow_partial ? 1 : 0, max_leaves, &best,
                                             row.mutable_data(), &scored, &total);
            }
            e.eng->check(rc, "helio_gpu_best_exhaustive");
            return py::make_tuple(best, row, scored, total);
          },
          py::arg("allow_partial") = true, py::arg("max_leaves") = 2000000000LL,
          "Exhaustive search in the reference's enumeration order: (best value, row, leaves scored, leaf space).")
      .def(
          "local_search",
          [](PyEngine& e, py::array_t<int16_t, py::array::c_style | py::array::forcecast> seed, bool allow_partial,
             int32_t max_moves, bool swaps) {
            const int N = e.eng->num_nodes();
            if (seed.ndim() != 2 || seed.shape(0) != N || seed.shape(1) != 2)
              throw py::value_error("seed must be int16 [num_nodes, 2]");
            py::array_t<int16_t> row({(py::ssize_t)N, (py::ssize_t)2});
            double value = 0;
            int32_t moves = 0;
            int64_t scored = 0;
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_local_search(e.eng->ctx(), seed.data(), allow_partial ? 1 : 0, max_moves,
                                          HELIO_LS_MOVES | (swaps ? HELIO_LS_SWAPS : 0), &value,
                                          row.mutable_data(), &moves, &scored);
            }
            e.eng->check(rc, "helio_gpu_local_search");
            return py::make_tuple(value, row, moves, scored);
          },
          py::arg("seed"), py::arg("allow_partial") = true, py::arg("max_moves") = -1, py::arg("swaps") = true,
          "Best-improvement local search over single-node moves (+ interval swaps): "
          "(value, row, moves, placements scored).")
      .def(
          "sampled_search",
          [](PyEngine& e, py::array_t<int16_t, py::array::c_style | py::array::forcecast> seed, bool allow_partial,
             int32_t iterations, int64_t batch, int32_t max_changes, uint64_t rng_seed) {
            const int N = e.eng->num_nodes();
            if (seed.ndim() != 2 || seed.shape(0) != N || seed.shape(1) != 2)
              throw py::value_error("seed must be int16 [num_nodes, 2]");
            py::array_t<int16_t> row({(py::ssize_t)N, (py::ssize_t)2});
            double value = 0;
            int32_t improvements = 0;
            int64_t scored = 0;
            int rc;
            {
              py::gil_scoped_release rel;
              rc = helio_gpu_sampled_search(e.eng->ctx(), seed.data(), allow_partial ? 1 : 0, iterations, batch,
                                            max_changes, rng_seed, &value, row.mutable_data(), &improvements,
                                            &scored);
            }
            e.eng->check(rc, "helio_gpu_sampled_search");
            return py::make_tuple(value, row, improvements, scored);
          },
          py::arg("seed"), py::arg("allow_partial") = true, py::arg("iterations") = 20,
          py::arg("batch") = 1 << 20, py::arg("max_changes") = 3, py::arg("rng_seed") = 1,
          "Sampled multi-node search: `iterations` rounds of `batch` mutants (1..max_changes nodes "
          "re-assigned) of the incumbent; the round's first maximum is taken when >= the incumbent (plateau "
          "moves), the best seen is returned: (value, row, rounds that raised it, scored).")
      .def("sync", [](PyEngine& e) { e.eng->check(helio_gpu_sync(e.eng->ctx()), "helio_gpu_sync"); });
}
