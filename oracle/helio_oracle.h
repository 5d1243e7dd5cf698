/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the reference's
 * hot path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and only as the checker.  It is pinned against the compiled
 * reference (oracle/_ref/libhelio_ref.so) and the committed golden vectors in
 * tests/golden/.  See helio_oracle.c for the file:line each function follows. */
#ifndef HELIO_ORACLE_H
#define HELIO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Cluster in plain arrays (ids replaced by indices + byte-lexicographic ranks). */
typedef struct {
  int32_t num_nodes, num_links, num_layers;
  double param_bytes, token_bytes, activation_bytes, kv_bytes_per_token_layer;
  const double* vram_bytes;        /* [N] */
  const double* kv_reserve;        /* [N] */
  const double* peak_layer_tokens; /* [N] */
  const double* nic_in_bps;        /* [N] */
  const double* nic_out_bps;       /* [N] */
  const int32_t* table_off;        /* [N+1] throughput_table values for keys 1..len */
  const double* table_val;
  const int32_t* lex_rank;         /* [N] rank of node id in byte order */
  const int32_t* link_src;         /* [M] node index, -1 coordinator, -2 undeclared id */
  const int32_t* link_dst;         /* [M] */
  const double* link_bw;           /* [M] bits/s */
} ora_cluster;

int ora_max_layers(const ora_cluster* c, int k);
double ora_compute_edge_capacity(const ora_cluster* c, int k, int j);

/* build_flow_graph for one int16[N][2] placement.  Returns 0, or 1/2/3 for the
 * unknown-node / range / VRAM ValidationErrors, or -2 if max_e is too small. */
int ora_build(const ora_cluster* c, const int16_t* pl, int allow_partial, int max_e,
              int32_t* nv, int32_t* ne, int32_t* u, int32_t* v, int32_t* kind, int32_t* es,
              int32_t* ee, double* cap);

/* max_flow on a raw graph (edges in order); flow[] may be NULL. */
double ora_max_flow(int n, int s, int t, int m, const int32_t* u, const int32_t* v,
                    const double* cap, double* flow);

/* build + max_flow per candidate. */
int ora_score(const ora_cluster* c, const int16_t* pl, int64_t B, int allow_partial,
              double* values, int32_t* status);

void ora_iwrr_weights(const double* flows, int n, int64_t* w);

/* plan_from_placement: positive-flow non-compute edges (src/dst node index,
 * -1 = coordinator).  Returns edge count or -status. */
int ora_plan(const ora_cluster* c, const int16_t* pl, int allow_partial, int max_edges,
             int32_t* src, int32_t* dst, double* flow, int32_t* es, int32_t* ee,
             double* objective);

/* AC8 admit/complete loop over R requests (see ora_route in helio_oracle.c). */
int64_t ora_route(const ora_cluster* c, const int16_t* pl, int allow_partial, int64_t R,
                  const int32_t* in_len, const int32_t* out_len, int max_hops, int32_t* nhops,
                  int32_t* hop_node, int32_t* hop_s, int32_t* hop_e);

#ifdef __cplusplus
}
#endif
#endif
