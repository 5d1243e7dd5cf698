/* helio_gpu.h — C ABI of the B200 placement-scoring engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj, "helio"):
 *
 *   reference interface (file:line)                 replaced by
 *   ------------------------------------------------------------------------
 *   FlowGraph build_flow_graph(c, p, partial)       helio_gpu_flows_host (graph + flows)
 *       include/helio/flow_graph.hpp:43, src/flow_graph.cpp:45-136
 *   double max_flow(FlowGraph&)                     helio_gpu_maxflow_raw_host
 *       include/helio/flow_graph.hpp:46, src/flow_graph.cpp:138-229
 *   build_flow_graph + max_flow per candidate       helio_gpu_score / helio_gpu_score_host
 *       (the pair at tests/oracles/enumerate.hpp:56-57, bindings/pymodule.cpp:170-171,
 *        src/placement.cpp:358-359 and :441-442)
 *   strict-'>' argmax over candidates               helio_gpu_argmax
 *       tests/oracles/enumerate.hpp:59
 *   compute_edge_capacity / ClusterSpec::max_layers helio_gpu_set_cluster (K0, precomputed once)
 *       src/flow_graph.cpp:38-43, src/cluster.cpp:62-100
 *   iwrr_weights + IwrrPicker + Scheduler::admit    helio_gpu_route_host
 *       src/scheduler.cpp:28-56, :157-190 (AC8 admit/complete loop)
 *
 * Conventions: every entry returns an int status (HELIO_OK == 0); nothing
 * throws across the ABI; helio_gpu_last_error() holds the message of the last
 * failure.  Buffers are caller-owned.  "d_" pointers are device memory,
 * "h_" pointers host memory (pinned or pageable).  A context is bound to one
 * device; concurrent calls on one context are serialised by the context
 * (graphs may be solved from many threads); use one context per
 * thread for parallelism.  `stream` is a
 * cudaStream_t (NULL = the context's own stream).
 *
 * Placements are int16 [B][N][2] rows (start, end) in the cluster's declared
 * node order; a row with end <= start is an idle node, exactly like an empty
 * Interval in the reference's Placement map (src/flow_graph.cpp:53).
 */
#ifndef HELIO_GPU_H
#define HELIO_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* call status */
#define HELIO_OK 0
#define HELIO_ERR_INVALID 1     /* bad argument / cluster */
#define HELIO_ERR_CUDA 2        /* CUDA runtime failure */
#define HELIO_ERR_NO_CLUSTER 3  /* helio_gpu_set_cluster not called */
#define HELIO_ERR_TOO_LARGE 4   /* graph exceeds the device limits */

/* per-candidate status (values[i] is 0 when status[i] != 0) */
#define HELIO_CAND_OK 0
#define HELIO_CAND_UNKNOWN_NODE 1 /* "placement references unknown node" (flow_graph.cpp:55) */
#define HELIO_CAND_RANGE 2        /* "placement ... outside [0, L)" (flow_graph.cpp:56-57) */
#define HELIO_CAND_VRAM 3         /* "exceeds its VRAM layer capacity" (flow_graph.cpp:58-59) */
#define HELIO_CAND_TOO_LARGE 4    /* graph does not fit one SM's shared memory */
#define HELIO_CAND_EDGE_BUFFER 5  /* flows: caller's max_edges too small (num_edges holds the need) */

/* scoring modes (helio_gpu_set_mode):
 *   PARITY — replays the reference's FIFO preflow-push discharge sequence
 *            (flow_graph.cpp:138-229): values and per-edge flows are
 *            bit-identical to the reference.  Default; used for every
 *            per-edge-flow entry point.
 *   SCORE  — value only (Edmonds-Karp over a bitset BFS for graphs of at
 *            most 128 vertices; push-relabel with global relabels above).
 *            Exact on integer capacities; within rounding (<= 1e-6 relative, asserted
 *            by the tests) on float capacities.  For bulk placement search. */
#define HELIO_MODE_PARITY 0
#define HELIO_MODE_SCORE 1

/* edge kinds, same numbering as helio::EdgeKind (flow_graph.hpp:21) */
#define HELIO_EDGE_COMPUTE 0
#define HELIO_EDGE_COORD_OUT 1
#define HELIO_EDGE_COORD_IN 2
#define HELIO_EDGE_INTERCONNECT 3

typedef struct helio_gpu_ctx helio_gpu_ctx;

/* A ClusterSpec (cluster.hpp:10-58) with ids replaced by indices.  Derived
 * quantities (k_i, T_j, NIC clamps, token capacities) are computed by the
 * library with the reference's own expressions. */
typedef struct {
  int32_t num_nodes;
  int32_t num_links;
  int32_t num_layers;               /* ModelSpec::num_layers */
  double param_bytes;               /* ModelSpec::param_bytes */
  double token_bytes;               /* ModelSpec::token_bytes */
  double activation_bytes;          /* ModelSpec::activation_bytes */
  double kv_bytes_per_token_layer;  /* ModelSpec::kv_bytes_per_token_layer (0 = 2*act) */
  const double* vram_bytes;         /* [N] NodeSpec::vram_bytes */
  const double* kv_reserve;         /* [N] */
  const double* peak_layer_tokens;  /* [N] */
  const double* nic_in_bps;         /* [N] 0 = max incident link bandwidth */
  const double* nic_out_bps;        /* [N] */
  const int32_t* table_off;         /* [N+1] throughput_table values for keys 1..len, or NULL */
  const double* table_val;
  const int32_t* lex_rank;          /* [N] rank of node id in byte-lexicographic order */
  const int32_t* link_src;          /* [M] node index, -1 = coordinator, -2 = undeclared id */
  const int32_t* link_dst;          /* [M] */
  const double* link_bandwidth_bps; /* [M] */
} helio_cluster_desc;

/* One FlowEdge (flow_graph.hpp:23-31) in g.edges order. */
typedef struct {
  int32_t u, v;
  int32_t kind;
  int32_t exec_start, exec_end;
  int32_t src_node, dst_node; /* node index, -1 = coordinator */
  int32_t pad;
  double cap;
  double flow;
} helio_edge;

/* One PlanEdge (placement.hpp:47-51): src/dst node index, -1 = coordinator. */
typedef struct {
  int32_t src_node, dst_node;
  int32_t exec_start, exec_end;
  double flow;
} helio_plan_edge;

int helio_gpu_create(int device, helio_gpu_ctx** out);
void helio_gpu_destroy(helio_gpu_ctx* ctx);
const char* helio_gpu_last_error(const helio_gpu_ctx* ctx);
int helio_gpu_sync(helio_gpu_ctx* ctx);

/* K0: compile and upload a cluster.  k_out (optional, [N]) receives k_i. */
int helio_gpu_set_cluster(helio_gpu_ctx* ctx, const helio_cluster_desc* desc, int32_t* k_out);

int helio_gpu_set_mode(helio_gpu_ctx* ctx, int mode);
int helio_gpu_get_mode(const helio_gpu_ctx* ctx);

/* compute_edge_capacity(c, node, j) for 1 <= j <= k_i, from the compiled table. */
int helio_gpu_compute_edge_capacity(const helio_gpu_ctx* ctx, int32_t node, int32_t j, double* out);

/* Batched build_flow_graph + max_flow value, device buffers, async on stream. */
int helio_gpu_score(helio_gpu_ctx* ctx, const int16_t* d_placements, int64_t B, int allow_partial,
                    double* d_values, int32_t* d_status, void* stream);

/* Same, host buffers (host<->device copies inside, pipelined); synchronous. */
int helio_gpu_score_host(helio_gpu_ctx* ctx, const int16_t* h_placements, int64_t B,
                         int allow_partial, double* h_values, int32_t* h_status);

/* Same, plus the first maximum over status==0 candidates with value > 0
 * (enumerate.hpp:59), reduced on the device; h_values/h_status may both be
 * NULL when only the winner is wanted.  *h_index = -1 if nothing beats 0. */
int helio_gpu_score_best_host(helio_gpu_ctx* ctx, const int16_t* h_placements, int64_t B,
                              int allow_partial, double* h_values, int32_t* h_status,
                              double* h_best, int64_t* h_index);

/* The split K1 -> HBM -> K2 pipeline (north_star's builder and solver as
 * separate launches; the fused helio_gpu_score is the production path).
 * helio_gpu_build_csr writes each candidate's flow network — the reference's
 * vertex, edge and per-vertex arc order — to a fixed-size slab of
 * helio_gpu_csr_slab_bytes() bytes: int32 {V, E, status, 0}, int32 arc
 * offsets [V+1], int32 arcs (head | reverse-arc << 16) [2E], float64
 * capacities [2E] (each section 16-byte aligned).  helio_gpu_solve_csr runs
 * the PARITY solver on the slabs; values are bit-identical to
 * helio_gpu_score in PARITY mode.  Graphs larger than the slab get
 * HELIO_CAND_TOO_LARGE. */
int64_t helio_gpu_csr_slab_bytes(const helio_gpu_ctx* ctx);
int helio_gpu_build_csr(helio_gpu_ctx* ctx, const int16_t* d_placements, int64_t B, int allow_partial,
                        void* d_slabs, int32_t* d_status, void* stream);
int helio_gpu_solve_csr(helio_gpu_ctx* ctx, const void* d_slabs, int64_t B, double* d_values,
                        int32_t* d_status, void* stream);

/* Full FlowGraph (edges in reference order, with max_flow's per-edge flows)
 * for K candidates; synchronous, host buffers.  h_edges is [K][max_edges]. */
int helio_gpu_flows_host(helio_gpu_ctx* ctx, const int16_t* h_placements, int64_t K,
                         int allow_partial, int32_t max_edges, int32_t* h_num_vertices,
                         int32_t* h_num_edges, helio_edge* h_edges, double* h_values,
                         int32_t* h_status);

/* max_flow on G raw graphs (any source/sink, self-loops, parallel edges, zero
 * capacities — flow_graph.cpp:138-229).  Edges of graph g are
 * [edge_off[g], edge_off[g+1]).  h_flows (optional) receives per-edge flows. */
int helio_gpu_maxflow_raw_host(helio_gpu_ctx* ctx, int64_t G, const int32_t* h_n,
                               const int32_t* h_source, const int32_t* h_sink,
                               const int64_t* h_edge_off, const int32_t* h_u, const int32_t* h_v,
                               const double* h_cap, double* h_values, double* h_flows);

/* First index of the maximum value among status==0 candidates with value > 0
 * (enumerate.hpp:59 strict '>' from best = 0).  Writes (0, -1) if none.
 * index_base is added to the index (global candidate numbering). */
int helio_gpu_argmax(helio_gpu_ctx* ctx, const double* d_values, const int32_t* d_status,
                     int64_t B, int64_t index_base, double* d_best, int64_t* d_index,
                     void* stream);

/* Candidate generator G(seed, i): random covering chains,
 * counter-based (splitmix64), identical on host and device.  p_uniform_ppm
 * mixes in uniform random intervals (parts per million per node). */
int helio_gpu_generate(helio_gpu_ctx* ctx, uint64_t seed, int64_t first, int64_t B,
                       uint32_t p_uniform_ppm, int16_t* d_out, void* stream);
void helio_generate_host(const int32_t* k, int32_t num_nodes, int32_t num_layers, uint64_t seed,
                         int64_t first, int64_t B, uint32_t p_uniform_ppm, int16_t* h_out);

/* Exhaustive placement search (tests/oracles/enumerate.hpp:14-77) on the
 * device: every combination of per-node choices {idle} + {[s, e): e - s <= k_i}
 * that covers all L <= 32 layers is scored in PARITY mode in the reference's
 * DFS order, and the first strict maximum over 0 wins (:59).  h_best_row is
 * int16 [N][2] (all zero if nothing beats 0).  Fails with
 * HELIO_ERR_TOO_LARGE when the leaf space exceeds max_leaves (> 0). */
int helio_gpu_best_exhaustive(helio_gpu_ctx* ctx, int allow_partial, int64_t max_leaves,
                              double* h_best_value, int16_t* h_best_row, int64_t* h_leaves_scored,
                              int64_t* h_leaves_total);

/* Best-improvement local search from a seed placement (
 * seeds typically come from the heuristics of src/heuristics.cpp:12-131).
 * Each iteration scores, in the context's mode, the neighbourhood of the
 * current placement and moves to its first strict maximum when that beats
 * the current value (enumerate.hpp:59).  Neighbourhood bits:
 *   HELIO_LS_MOVES  every placement that differs in exactly one node's
 *                   interval, node-major; per node the choices of
 *                   enumerate.hpp:21-28 (idle, then [s, e) with e - s <= k_i
 *                   in (s, e) order);
 *   HELIO_LS_SWAPS  then every exchange of two nodes' intervals, (i, j) with
 *                   i < j in order (an exchange that breaks k_i scores as
 *                   invalid and is never taken).
 * Stops at a local optimum or after max_moves moves (< 0: no limit).  The
 * seed must pass validation (HELIO_ERR_INVALID otherwise).  Outputs the final
 * value and int16 [N][2] row, the moves taken and the placements scored
 * (seed included). */
#define HELIO_LS_MOVES 1
#define HELIO_LS_SWAPS 2
int helio_gpu_local_search(helio_gpu_ctx* ctx, const int16_t* h_seed, int allow_partial, int32_t max_moves,
                           int32_t neighbourhood, double* h_value, int16_t* h_row, int32_t* h_moves,
                           int64_t* h_scored);

/* Sampled multi-node search from a seed placement (SURVEY.md §8(f) rank 1,
 * past the local optima of helio_gpu_local_search).  Each of `iterations`
 * rounds scores, in the context's mode, `batch` mutants of the incumbent —
 * each re-assigns 1..max_changes random nodes (keep start / keep end / shift
 * the stage boundary shared with a chain successor / start where another node
 * ends / idle / uniform; lengths within k_i, so every mutant validates) — and
 * moves to the round's first maximum (enumerate.hpp:59 order) when it is at
 * least the incumbent's value: equal values are sideways moves along a
 * plateau.  The best placement seen (first strict improvement kept) is
 * returned.  Draws are counter-based over (rng_seed, round, mutant): the
 * result is deterministic.  The seed must validate.  Outputs the best value
 * and int16 [N][2] row, the number of rounds that raised the best value and
 * the placements scored (seed included). */
int helio_gpu_sampled_search(helio_gpu_ctx* ctx, const int16_t* h_seed, int allow_partial, int32_t iterations,
                             int64_t batch, int32_t max_changes, uint64_t rng_seed, double* h_value,
                             int16_t* h_row, int32_t* h_improvements, int64_t* h_scored);

/* Link-walking covering chains (gen.h hg_candidate_walk) for sparse
 * topologies, device and host (identical output). */
int helio_gpu_generate_walk(helio_gpu_ctx* ctx, uint64_t seed, int64_t first, int64_t B,
                            int16_t* d_out, void* stream);
int helio_gpu_generate_walk_host(const helio_gpu_ctx* ctx, uint64_t seed, int64_t first, int64_t B,
                                 int16_t* h_out);

/* IWRR routing of R requests over a plan (scheduler.cpp:58-190) in the AC8
 * admit/complete order: request r is admitted with in_len[r] and completed at
 * once with out_len[r].  Plan edges in plan order; placement is the plan's
 * int16 [N][2] row.  hop arrays are [R][max_hops] (h_hop_start/h_hop_end may
 * both be NULL to return node ids only); h_num_hops[r] = -1 for a deferred
 * request; hop entries past a request's count (all of a deferred request's)
 * are unspecified.  *h_deferred receives the number of deferrals.  When KV
 * masking can bind, the exact replay of the reference's eligibility tests runs
 * (route.cu route_masked_spec / route_masked_warp); otherwise the closed form. */
int helio_gpu_route_host(helio_gpu_ctx* ctx, const int16_t* h_placement,
                         const helio_plan_edge* h_plan_edges, int32_t num_plan_edges, int64_t R,
                         const int32_t* h_in_len, const int32_t* h_out_len, int32_t max_hops,
                         int32_t* h_num_hops, int32_t* h_hop_node, int32_t* h_hop_start,
                         int32_t* h_hop_end, int64_t* h_deferred);

/* iwrr_weights (scheduler.cpp:46-56) of one candidate list, on the device. */
int helio_gpu_iwrr_weights(helio_gpu_ctx* ctx, const double* h_flows, int32_t n, int64_t* h_weights);

/* IWRR cycles of `nlists` candidate lists (list l = entries [h_off[l],
 * h_off[l+1]) of the flattened arrays): with h_flows != NULL the weights are
 * iwrr_weights(flows) (scheduler.cpp:46-56) and written to h_weights; with
 * h_flows == NULL h_weights is read as the caller's weights (the IwrrPicker
 * constructor, scheduler.cpp:24-26).  List l's cycle — the (round, index)
 * slots with w_i >= round in the order IwrrPicker::next visits them
 * (scheduler.cpp:28-44) — is written to h_cycles[h_cyc_off[l] ...] as
 * candidate indices, its length (sum of the weights) to h_cyc_len[l].  Slot
 * ranges must hold the cycle (32 * list size always does for flow weights).
 * The k-th unmasked IwrrPicker::next call of a fresh picker returns
 * cycle[k mod length]. */
int helio_gpu_iwrr_cycles(helio_gpu_ctx* ctx, int32_t nlists, const int32_t* h_off, const double* h_flows,
                          int64_t* h_weights, const int64_t* h_cyc_off, int32_t* h_cycles,
                          int64_t* h_cyc_len);

/* IwrrPicker::next (scheduler.cpp:28-44) `calls` times on the device.  The
 * picker state (round, idx) is read from and written back to *h_round/*h_idx
 * (a fresh picker is round 1, idx 0).  h_masks holds, per call, ceil(n/64)
 * little-endian words of eligibility bits.  h_out[k] = candidate or -1. */
int helio_gpu_iwrr_picks(helio_gpu_ctx* ctx, const int64_t* h_weights, int32_t n, int64_t* h_round,
                         int64_t* h_idx, int32_t calls, const uint64_t* h_masks, int32_t* h_out);

/* --- multi-GPU (csrc/multi.cu) ---------------------
 *
 * Ranked argmax, one process per GPU: this rank's shard [index_base,
 * index_base + B) is reduced on the device to (best value, global index), the
 * 16-byte records of all ranks are all-gathered over `nccl_comm` (an
 * ncclComm_t) and reduced deterministically — max value, then min index, the
 * first-wins strict '>' of tests/oracles/enumerate.hpp:59 over the global
 * order — into d_best / d_index on every rank.  Stream ordered on `stream`
 * (NULL = the context's stream); no host synchronisation. */
int helio_gpu_argmax_ranked(helio_gpu_ctx* ctx, const double* d_values, const int32_t* d_status, int64_t B,
                            int64_t index_base, double* d_best, int64_t* d_index, void* nccl_comm, void* stream);

/* NCCL communicator helpers for callers without one: rank 0 draws the
 * 128-byte unique id and sends it to every rank over the caller's channel. */
int helio_gpu_nccl_unique_id(uint8_t* id128);
int helio_gpu_nccl_comm_create(const uint8_t* id128, int32_t nranks, int32_t rank, int32_t device, void** comm);
int helio_gpu_nccl_comm_destroy(void* comm);

/* One process, several GPUs: one context per device; host batches are split
 * into contiguous shards (one host thread per device) and the first maxima
 * merged in index order. */
typedef struct helio_gpu_multi helio_gpu_multi;
int helio_gpu_multi_create(const int32_t* devices, int32_t n, helio_gpu_multi** out);
void helio_gpu_multi_destroy(helio_gpu_multi* m);
const char* helio_gpu_multi_last_error(const helio_gpu_multi* m);
int32_t helio_gpu_multi_count(const helio_gpu_multi* m);
helio_gpu_ctx* helio_gpu_multi_context(helio_gpu_multi* m, int32_t i);
int helio_gpu_multi_set_cluster(helio_gpu_multi* m, const helio_cluster_desc* desc, int32_t* k_out);
int helio_gpu_multi_set_mode(helio_gpu_multi* m, int mode);
int helio_gpu_multi_score_best_host(helio_gpu_multi* m, const int16_t* h_placements, int64_t B, int allow_partial,
                                    double* h_values, int32_t* h_status, double* h_best, int64_t* h_index);
/* helio_gpu_sampled_search with every round's mutants split over the devices:
 * the same mutants, the same first-maximum tie-break — the same result as one
 * device. */
int helio_gpu_multi_sampled_search(helio_gpu_multi* m, const int16_t* h_seed, int allow_partial, int32_t iterations,
                                   int64_t batch, int32_t max_changes, uint64_t rng_seed, double* h_value,
                                   int16_t* h_row, int32_t* h_improvements, int64_t* h_scored);

/* Self-test of the masked routing replay's division (route.cu div_by_count:
 * reciprocal-based, correctly rounded) against IEEE division on `count`
 * counter-generated operand pairs of the routing domain; *mismatches = 0
 * expected. */
int helio_gpu_check_division(helio_gpu_ctx* ctx, int64_t count, uint64_t seed, int64_t* mismatches);

/* Introspection for benchmarks: kernels launched by this context so far, and
 * the device time (ms) of the last score call's dominant kernel. */
int64_t helio_gpu_launch_count(const helio_gpu_ctx* ctx);
double helio_gpu_last_kernel_ms(const helio_gpu_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HELIO_GPU_H */
