// search.cu — exhaustive placement search on the device.
//
// Reference: best_placement_exhaustive (tests/oracles/enumerate.hpp:14-77).
// Node i's choices are {idle} followed by every [s, e) with e - s <= k_i in
// (s, e) order (:21-28); the DFS visits nodes in declaration order, so leaf
// order is mixed-radix order with node 0 as the most significant digit.  The
// DFS prunes subtrees that can no longer cover all L layers (:37-51), i.e. it
// scores exactly the covering leaves, in order, and keeps the first strict
// maximum over best = 0 (:59).  Here: leaves are enumerated by index in
// chunks, non-covering ones are dropped with an order-preserving select, the
// survivors are materialised as placement rows and scored by the PARITY
// kernel (bit-identical values), and K4's first-max argmax combines chunks.
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <vector>

#include "engine.h"
#include "gen.h"

using namespace helio_engine;

namespace {

struct Choices {
  int N;
  const int32_t* off;       // [N+1] into s/e/mask
  const int64_t* radix;     // [N] product of choice counts of nodes after i
  const int16_t* cs;        // start
  const int16_t* ce;        // end
  const uint64_t* cmask;    // coverage bits of the choice
};

__global__ void enum_flag(Choices ch, int64_t base, int64_t n, uint64_t full, uint8_t* flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx = base + t;
    uint64_t cov = 0;
    for (int i = 0; i < ch.N; ++i) {
      const int64_t r = ch.radix[i];
      const int64_t d = idx / r;
      idx -= d * r;
      cov |= ch.cmask[ch.off[i] + (int)d];
    }
    flag[t] = cov == full ? 1 : 0;
  }
}

__global__ void enum_rows(Choices ch, int64_t base, const int64_t* sel, int64_t m, int16_t* rows) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx = base + sel[t];
    for (int i = 0; i < ch.N; ++i) {
      const int64_t r = ch.radix[i];
      const int64_t d = idx / r;
      idx -= d * r;
      const int c = ch.off[i] + (int)d;
      rows[(t * ch.N + i) * 2] = ch.cs[c];
      rows[(t * ch.N + i) * 2 + 1] = ch.ce[c];
    }
  }
}

}  // namespace

// defined in helio_gpu.cu
int helio_engine_score_parity(helio_gpu_ctx* ctx, const int16_t* d_pl, int64_t B, int partial, double* d_val,
                              int32_t* d_st, cudaStream_t st);

extern "C" int helio_gpu_best_exhaustive(helio_gpu_ctx* ctx, int allow_partial, int64_t max_leaves,
                                         double* h_best_value, int16_t* h_best_row, int64_t* h_scored,
                                         int64_t* h_total) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (!h_best_value || !h_best_row) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  const int N = ctx->N, L = ctx->L;
  if (L > 32) return fail(ctx, HELIO_ERR_INVALID, "exhaustive search needs num_layers <= 32 (enumerate.hpp:30-35)");
  CK(cudaSetDevice(ctx->device));
  // choices per node, in the reference's order
  std::vector<int32_t> off(N + 1, 0);
  std::vector<int16_t> cs, ce;
  std::vector<uint64_t> cm;
  for (int i = 0; i < N; ++i) {
    off[i] = (int32_t)cs.size();
    cs.push_back(0);
    ce.push_back(0);
    cm.push_back(0);
    const int k = ctx->h_kmax[i];
    for (int s = 0; s < L; ++s)
      for (int e = s + 1; e <= L && e - s <= k; ++e) {
        cs.push_back((int16_t)s);
        ce.push_back((int16_t)e);
        uint64_t m = 0;
        for (int l = s; l < e; ++l) m |= 1ull << l;
        cm.push_back(m);
      }
  }
  off[N] = (int32_t)cs.size();
  std::vector<int64_t> radix(N, 1);
  double total_d = 1.0;
  int64_t total = 1;
  for (int i = N - 1; i >= 0; --i) {
    radix[i] = total;
    const int64_t c = off[i + 1] - off[i];
    total_d *= (double)c;
    if (total_d > 9.0e18) return fail(ctx, HELIO_ERR_TOO_LARGE, "placement space exceeds 2^63 leaves");
    total *= c;
  }
  if (max_leaves > 0 && total > max_leaves)
    return fail(ctx, HELIO_ERR_TOO_LARGE, "placement space (" + std::to_string(total) + " leaves) exceeds max_leaves");
  const uint64_t full = L >= 64 ? ~0ull : ((1ull << L) - 1);
  cudaStream_t st = ctx->stream;
  const int64_t chunk = std::min<int64_t>(total, 1 << 22);
  int rc = HELIO_OK;
  int32_t* d_off = nullptr;
  int64_t *d_radix = nullptr, *d_sel = nullptr, *d_nsel = nullptr, *d_bidx = nullptr;
  int16_t *d_cs = nullptr, *d_ce = nullptr, *d_rows = nullptr;
  uint64_t* d_cm = nullptr;
  uint8_t* d_flag = nullptr;
  double *d_val = nullptr, *d_best = nullptr;
  int32_t* d_st = nullptr;
  void* d_tmp = nullptr;
  size_t tmp = 0;
  auto A = [&](void** p, size_t bytes) {
    if (!rc && cudaMalloc(p, std::max<size_t>(bytes, 8)) != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "search alloc");
  };
  A((void**)&d_off, 4 * (N + 1));
  A((void**)&d_radix, 8 * N);
  A((void**)&d_cs, 2 * cs.size());
  A((void**)&d_ce, 2 * ce.size());
  A((void**)&d_cm, 8 * cm.size());
  A((void**)&d_flag, chunk);
  A((void**)&d_sel, 8 * chunk);
  A((void**)&d_nsel, 8);
  A((void**)&d_rows, 4 * (size_t)N * chunk);
  A((void**)&d_val, 8 * chunk);
  A((void**)&d_st, 4 * chunk);
  A((void**)&d_best, 8);
  A((void**)&d_bidx, 8);
  if (!rc) {
    cub::DeviceSelect::Flagged(nullptr, tmp, cub::CountingInputIterator<int64_t>(0), d_flag, d_sel, d_nsel,
                               (int)chunk, st);
    A(&d_tmp, tmp);
  }
  if (!rc) {
    cudaMemcpyAsync(d_off, off.data(), 4 * (N + 1), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_radix, radix.data(), 8 * N, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_cs, cs.data(), 2 * cs.size(), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_ce, ce.data(), 2 * ce.size(), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_cm, cm.data(), 8 * cm.size(), cudaMemcpyHostToDevice, st);
  }
  Choices ch{N, d_off, d_radix, d_cs, d_ce, d_cm};
  double best = 0.0;
  int64_t best_leaf = -1, scored = 0;
  std::vector<int16_t> best_row(2 * N, 0);
  for (int64_t base = 0; !rc && base < total; base += chunk) {
    const int64_t n = std::min(chunk, total - base);
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 16 * ctx->sm_count);
    enum_flag<<<grid, 256, 0, st>>>(ch, base, n, full, d_flag);
    cub::DeviceSelect::Flagged(d_tmp, tmp, cub::CountingInputIterator<int64_t>(0), d_flag, d_sel, d_nsel, (int)n, st);
    ctx->launches += 2;
    int64_t m = 0;
    if (cudaMemcpyAsync(&m, d_nsel, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = fail(ctx, HELIO_ERR_CUDA, std::string("search select: ") + cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (m == 0) continue;
    const int g2 = (int)std::min<int64_t>((m + 255) / 256, 16 * ctx->sm_count);
    enum_rows<<<g2, 256, 0, st>>>(ch, base, d_sel, m, d_rows);
    ctx->launches++;
    rc = helio_engine_score_parity(ctx, d_rows, m, allow_partial ? 1 : 0, d_val, d_st, st);
    if (rc) break;
    rc = helio_gpu_argmax(ctx, d_val, d_st, m, 0, d_best, d_bidx, st);
    if (rc) break;
    double cb = 0;
    int64_t ci = -1;
    if (cudaMemcpyAsync(&cb, d_best, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&ci, d_bidx, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = fail(ctx, HELIO_ERR_CUDA, "search argmax readback");
      break;
    }
    scored += m;
    if (ci >= 0 && cb > best) {  // strict: earlier chunks win ties (enumerate.hpp:59)
      best = cb;
      if (cudaMemcpyAsync(best_row.data(), d_rows + ci * 2 * N, 4 * N, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess) {
        rc = fail(ctx, HELIO_ERR_CUDA, "search row readback");
        break;
      }
      best_leaf = ci;
    }
  }
  (void)best_leaf;
  cudaFree(d_off); cudaFree(d_radix); cudaFree(d_cs); cudaFree(d_ce); cudaFree(d_cm); cudaFree(d_flag);
  cudaFree(d_sel); cudaFree(d_nsel); cudaFree(d_rows); cudaFree(d_val); cudaFree(d_st); cudaFree(d_best);
  cudaFree(d_bidx); cudaFree(d_tmp);
  if (rc) return rc;
  *h_best_value = best;
  std::copy(best_row.begin(), best_row.end(), h_best_row);
  if (h_scored) *h_scored = scored;
  if (h_total) *h_total = total;
  return HELIO_OK;
}

// ---------------------------------------------------------------------------
// Best-improvement local search over single-node moves (SURVEY.md §8(f) rank
// 1: the enumerate consumer generalised to clusters whose placement space is
// far beyond exhaustive search, seeded from the heuristics of
// src/heuristics.cpp:12-131).  One iteration scores every placement that
// differs from the current one in exactly one node's interval — node i
// takes any choice of enumerate.hpp:21-28 ({idle} then [s, e) with
// e - s <= k_i in (s, e) order), neighbours ordered node-major — with the
// context's scoring mode, and moves to the first strict maximum if it beats
// the current value (enumerate.hpp:59's strict '>' and first-wins rule).
namespace {

// Move t: node_of[t] >= 0 gives that node the packed interval choice[t];
// node_of[t] < 0 exchanges the intervals of nodes ~node_of[t] and choice[t].
__global__ void neighbour_rows(const int32_t* __restrict__ cur, int N, const int16_t* __restrict__ node_of,
                               const int32_t* __restrict__ choice, int64_t C, int32_t* __restrict__ rows) {
  const int64_t words = C * N;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < words;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = q / N;
    const int k = (int)(q - t * N);
    const int a = node_of[t];
    int32_t w = __ldg(cur + k);
    if (a >= 0) {
      if (k == a) w = choice[t];
    } else {
      const int i = ~a, j = choice[t];
      if (k == i) w = __ldg(cur + j);
      else if (k == j) w = __ldg(cur + i);
    }
    rows[q] = w;
  }
}

}  // namespace

extern "C" int helio_gpu_local_search(helio_gpu_ctx* ctx, const int16_t* h_seed, int allow_partial,
                                      int32_t max_moves, int32_t neighbourhood, double* h_value, int16_t* h_row,
                                      int32_t* h_moves, int64_t* h_scored) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (!h_seed || !h_value || !h_row) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if ((neighbourhood & (HELIO_LS_MOVES | HELIO_LS_SWAPS)) == 0 || (neighbourhood & ~(HELIO_LS_MOVES | HELIO_LS_SWAPS)))
    return fail(ctx, HELIO_ERR_INVALID, "neighbourhood must be a non-empty set of HELIO_LS_* bits");
  const int N = ctx->N, L = ctx->L;
  CK(cudaSetDevice(ctx->device));
  // the move list: (node, packed interval) in neighbour order
  std::vector<int16_t> node_of;
  std::vector<int32_t> choice;
  auto pack = [](int s, int e) { return (int32_t)(uint16_t)s | (int32_t)((uint32_t)(uint16_t)e << 16); };
  if (neighbourhood & HELIO_LS_MOVES)
    for (int i = 0; i < N; ++i) {
      node_of.push_back((int16_t)i);
      choice.push_back(0);
      const int k = ctx->h_kmax[i];
      for (int s = 0; s < L; ++s)
        for (int e = s + 1; e <= L && e - s <= k; ++e) {
          node_of.push_back((int16_t)i);
          choice.push_back(pack(s, e));
        }
    }
  if (neighbourhood & HELIO_LS_SWAPS)
    for (int i = 0; i < N; ++i)
      for (int j = i + 1; j < N; ++j) {
        node_of.push_back((int16_t)~i);
        choice.push_back(j);
      }
  const int64_t C = (int64_t)choice.size();
  cudaStream_t st = ctx->stream;
  int rc = HELIO_OK;
  int16_t* d_node = nullptr;
  int32_t *d_choice = nullptr, *d_cur = nullptr, *d_rows = nullptr, *d_st = nullptr;
  double *d_val = nullptr, *d_best = nullptr;
  int64_t* d_bidx = nullptr;
  auto A = [&](void** p, size_t bytes) {
    if (!rc && cudaMalloc(p, std::max<size_t>(bytes, 8)) != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "local search alloc");
  };
  A((void**)&d_node, 2 * C);
  A((void**)&d_choice, 4 * C);
  A((void**)&d_cur, 4 * N);
  A((void**)&d_rows, 4 * (size_t)N * C);
  A((void**)&d_val, 8 * C);
  A((void**)&d_st, 4 * C);
  A((void**)&d_best, 8);
  A((void**)&d_bidx, 8);
  std::vector<int32_t> cur(N);
  for (int i = 0; i < N; ++i) cur[i] = pack(h_seed[2 * i], h_seed[2 * i + 1]);
  double value = 0.0;
  int32_t moves = 0;
  int64_t scored = 0;
  auto sync_read = [&](void* dst, const void* src, size_t bytes) {
    if (!rc && (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess))
      rc = fail(ctx, HELIO_ERR_CUDA, std::string("local search readback: ") + cudaGetErrorString(cudaGetLastError()));
  };
  if (!rc) {
    cudaMemcpyAsync(d_node, node_of.data(), 2 * C, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_choice, choice.data(), 4 * C, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_cur, cur.data(), 4 * N, cudaMemcpyHostToDevice, st);
    // the seed's own value and status
    rc = helio_gpu_score(ctx, reinterpret_cast<const int16_t*>(d_cur), 1, allow_partial, d_val, d_st, st);
    int32_t s0 = 0;
    sync_read(&value, d_val, 8);
    sync_read(&s0, d_st, 4);
    scored = 1;
    if (!rc && s0 != 0) rc = fail(ctx, HELIO_ERR_INVALID, "seed placement fails validation (status " + std::to_string(s0) + ")");
  }
  while (!rc && (max_moves < 0 || moves < max_moves)) {
    const int grid = (int)std::min<int64_t>((C * N + 255) / 256, 16 * ctx->sm_count);
    neighbour_rows<<<grid, 256, 0, st>>>(d_cur, N, d_node, d_choice, C, d_rows);
    ctx->launches++;
    rc = helio_gpu_score(ctx, reinterpret_cast<const int16_t*>(d_rows), C, allow_partial, d_val, d_st, st);
    if (rc) break;
    rc = helio_gpu_argmax(ctx, d_val, d_st, C, 0, d_best, d_bidx, st);
    if (rc) break;
    double best = 0.0;
    int64_t bi = -1;
    sync_read(&best, d_best, 8);
    sync_read(&bi, d_bidx, 8);
    scored += C;
    if (rc || bi < 0 || !(best > value)) break;
    value = best;
    if (node_of[bi] >= 0) {
      cur[node_of[bi]] = choice[bi];
    } else {
      std::swap(cur[~node_of[bi]], cur[choice[bi]]);
    }
    ++moves;
    if (cudaMemcpyAsync(d_cur, cur.data(), 4 * N, cudaMemcpyHostToDevice, st) != cudaSuccess)
      rc = fail(ctx, HELIO_ERR_CUDA, "local search upload");
  }
  if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "local search sync");
  cudaFree(d_node); cudaFree(d_choice); cudaFree(d_cur); cudaFree(d_rows); cudaFree(d_val); cudaFree(d_st);
  cudaFree(d_best); cudaFree(d_bidx);
  if (rc) return rc;
  *h_value = value;
  for (int i = 0; i < N; ++i) {
    h_row[2 * i] = (int16_t)(cur[i] & 0xffff);
    h_row[2 * i + 1] = (int16_t)((uint32_t)cur[i] >> 16);
  }
  if (h_moves) *h_moves = moves;
  if (h_scored) *h_scored = scored;
  return HELIO_OK;
}

// ---------------------------------------------------------------------------
// Sampled multi-node search (beyond the 1-move local
// search): every iteration scores `batch` mutants of the incumbent, each
// changing 1..max_changes random nodes, and moves to the first strict best if
// it beats the incumbent.  Local optima of the single-node neighbourhood are
// usually one 2-3-node change away from something better; the full 2-move
// neighbourhood of het42 has ~3e8 members, so it is sampled — at ~60M
// evals/s a 1M-mutant iteration costs ~17 ms.  A change re-assigns one node
// (any node with k_i >= 1) to an interval built from the incumbent:
//   20% keep its start, new length; 20% keep its end, new length;
//   15% move the stage boundary it shares with a chain successor (a node
//       starting where it ends) by 1-4 layers, both nodes re-assigned;
//   25% start where a random other node ends (wrapping at L) — extend a chain;
//   10% idle; 10% uniform interval.
// Lengths are U[1, k_i] truncated to [0, L], so every mutant validates.
// Counter-based draws (gen.h) over (seed, iteration, mutant): deterministic.
namespace {

__global__ void copy_rows(const int32_t* __restrict__ cur, int N, int64_t B, int32_t* __restrict__ rows) {
  const int64_t words = B * N;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < words; q += (int64_t)gridDim.x * blockDim.x)
    rows[q] = __ldg(cur + (q % N));
}

// Mutant b of a round is drawn from hg_key(seed, first + b): a round's
// 'batch' mutants are one counter range, so devices can split it.
__global__ void mutate_rows(const int32_t* __restrict__ cur, const int32_t* __restrict__ kmax, int N, int L,
                            uint64_t seed, int64_t first, int64_t B, int max_changes, int32_t* __restrict__ rows) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = hg_key(seed, (uint64_t)(first + b));
    const int c = 1 + (int)hg_uniform(hg_draw(key, 0), (uint32_t)max_changes);
    for (int j = 0; j < c; ++j) {
      const uint64_t d0 = hg_draw(key, 1 + 4 * j), d1 = hg_draw(key, 2 + 4 * j), d2 = hg_draw(key, 3 + 4 * j),
                     d3 = hg_draw(key, 4 + 4 * j);
      const int node = (int)hg_uniform(d0, (uint32_t)N);
      const int k = __ldg(kmax + node);
      if (k < 1) continue;
      const int32_t w = __ldg(cur + node);
      int s = (int16_t)(w & 0xffff), e = (int16_t)(w >> 16);
      const bool used = e > s;
      const int len = 1 + (int)hg_uniform(d2, (uint32_t)k);
      const uint32_t op = hg_uniform(d1, 100);
      if (op < 20) {  // keep start
        if (!used) s = (int)hg_uniform(d3, (uint32_t)L);
        e = min(s + len, L);
      } else if (op < 40) {  // keep end
        if (!used) e = 1 + (int)hg_uniform(d3, (uint32_t)L);
        s = max(e - len, 0);
      } else if (op < 55) {  // shift the stage boundary to a chain successor
        if (!used || e >= L) continue;
        int m = -1;
        const int off = (int)hg_uniform(d3, (uint32_t)N);
        for (int q = 0; q < N && m < 0; ++q) {
          const int cand = off + q < N ? off + q : off + q - N;
          const int32_t a = __ldg(cur + cand);
          const int as = (int16_t)(a & 0xffff), ae = (int16_t)(a >> 16);
          if (cand != node && ae > as && as == e) m = cand;
        }
        if (m < 0) continue;
        const int32_t a = __ldg(cur + m);
        const int me = (int16_t)(a >> 16), km = __ldg(kmax + m);
        const int delta = 1 + (int)((d2 >> 1) & 3);
        int ne = (d2 & 1) ? e + delta : e - delta;
        ne = max(max(ne, s), me - km);
        ne = min(min(ne, s + k), me);
        if (ne == e) continue;
        rows[b * N + node] = ne > s ? (int32_t)(uint16_t)s | (int32_t)((uint32_t)(uint16_t)ne << 16) : 0;
        rows[b * N + m] = me > ne ? (int32_t)(uint16_t)ne | (int32_t)((uint32_t)(uint16_t)me << 16) : 0;
        continue;
      } else if (op < 80) {  // attach after another node's end
        const int32_t a = __ldg(cur + hg_uniform(d3, (uint32_t)N));
        const int as = (int16_t)(a & 0xffff), ae = (int16_t)(a >> 16);
        s = (ae > as && ae < L) ? ae : 0;
        e = min(s + len, L);
      } else if (op < 90) {  // idle
        s = e = 0;
      } else {  // uniform
        const int ln = min(len, L);
        s = (int)hg_uniform(d3, (uint32_t)(L - ln + 1));
        e = s + ln;
      }
      rows[b * N + node] = (int32_t)(uint16_t)s | (int32_t)((uint32_t)(uint16_t)e << 16);
    }
  }
}

}  // namespace

extern "C" int helio_gpu_sampled_search(helio_gpu_ctx* ctx, const int16_t* h_seed, int allow_partial,
                                        int32_t iterations, int64_t batch, int32_t max_changes, uint64_t rng_seed,
                                        double* h_value, int16_t* h_row, int32_t* h_improvements,
                                        int64_t* h_scored) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (!h_seed || !h_value || !h_row) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (iterations < 0 || batch < 1 || max_changes < 1)
    return fail(ctx, HELIO_ERR_INVALID, "need iterations >= 0, batch >= 1, max_changes >= 1");
  const int N = ctx->N, L = ctx->L;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  int rc = HELIO_OK;
  int32_t *d_cur = nullptr, *d_keep = nullptr, *d_rows = nullptr, *d_st = nullptr, *d_kmax = nullptr;
  double *d_val = nullptr, *d_best = nullptr;
  int64_t* d_bidx = nullptr;
  auto A = [&](void** p, size_t bytes) {
    if (!rc && cudaMalloc(p, std::max<size_t>(bytes, 8)) != cudaSuccess) rc = fail(ctx, HELIO_ERR_CUDA, "sampled search alloc");
  };
  A((void**)&d_cur, 4 * N);
  A((void**)&d_keep, 4 * N);
  A((void**)&d_kmax, 4 * N);
  A((void**)&d_rows, 4 * (size_t)N * batch);
  A((void**)&d_val, 8 * batch);
  A((void**)&d_st, 4 * batch);
  A((void**)&d_best, 8);
  A((void**)&d_bidx, 8);
  auto sync_read = [&](void* dst, const void* src, size_t bytes) {
    if (!rc && (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess))
      rc = fail(ctx, HELIO_ERR_CUDA, std::string("sampled search readback: ") + cudaGetErrorString(cudaGetLastError()));
  };
  double value = 0.0, best_value = 0.0;
  int32_t improvements = 0;
  int64_t scored = 0;
  if (!rc) {
    std::vector<int32_t> cur(N);
    for (int i = 0; i < N; ++i)
      cur[i] = (int32_t)(uint16_t)h_seed[2 * i] | (int32_t)((uint32_t)(uint16_t)h_seed[2 * i + 1] << 16);
    cudaMemcpyAsync(d_cur, cur.data(), 4 * N, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_keep, cur.data(), 4 * N, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_kmax, ctx->h_kmax.data(), 4 * N, cudaMemcpyHostToDevice, st);
    rc = helio_gpu_score(ctx, reinterpret_cast<const int16_t*>(d_cur), 1, allow_partial, d_val, d_st, st);
    int32_t s0 = 0;
    sync_read(&value, d_val, 8);
    sync_read(&s0, d_st, 4);
    scored = 1;
    best_value = value;
    if (!rc && s0 != 0) rc = fail(ctx, HELIO_ERR_INVALID, "seed placement fails validation (status " + std::to_string(s0) + ")");
  }
  const int grid_w = (int)std::min<int64_t>(((int64_t)N * batch + 255) / 256, 16 * ctx->sm_count);
  const int grid_b = (int)std::min<int64_t>((batch + 255) / 256, 16 * ctx->sm_count);
  for (int32_t it = 0; !rc && it < iterations; ++it) {
    copy_rows<<<grid_w, 256, 0, st>>>(d_cur, N, batch, d_rows);
    mutate_rows<<<grid_b, 256, 0, st>>>(d_cur, d_kmax, N, L, hg_key(rng_seed, (uint64_t)it), 0, batch, max_changes,
                                        d_rows);
    ctx->launches += 2;
    rc = helio_gpu_score(ctx, reinterpret_cast<const int16_t*>(d_rows), batch, allow_partial, d_val, d_st, st);
    if (rc) break;
    rc = helio_gpu_argmax(ctx, d_val, d_st, batch, 0, d_best, d_bidx, st);
    if (rc) break;
    double best = 0.0;
    int64_t bi = -1;
    sync_read(&best, d_best, 8);
    sync_read(&bi, d_bidx, 8);
    scored += batch;
    if (!rc && bi >= 0 && best >= value) {  // equal values: a sideways move along the plateau
      if (best > best_value) {
        best_value = best;
        ++improvements;
        if (cudaMemcpyAsync(d_keep, d_rows + bi * N, 4 * N, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
          rc = fail(ctx, HELIO_ERR_CUDA, "sampled search update");
      }
      value = best;
      if (cudaMemcpyAsync(d_cur, d_rows + bi * N, 4 * N, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        rc = fail(ctx, HELIO_ERR_CUDA, "sampled search update");
    }
  }
  std::vector<int32_t> out(N);
  sync_read(out.data(), d_keep, 4 * N);
  value = best_value;
  cudaFree(d_keep);
  cudaFree(d_cur); cudaFree(d_kmax); cudaFree(d_rows); cudaFree(d_val); cudaFree(d_st); cudaFree(d_best);
  cudaFree(d_bidx);
  if (rc) return rc;
  *h_value = value;
  for (int i = 0; i < N; ++i) {
    h_row[2 * i] = (int16_t)(out[i] & 0xffff);
    h_row[2 * i + 1] = (int16_t)((uint32_t)out[i] >> 16);
  }
  if (h_improvements) *h_improvements = improvements;
  if (h_scored) *h_scored = scored;
  return HELIO_OK;
}

// One sampled-search round on a slice [first, first + n) of the round's
// mutants (csrc/multi.cu's multi-device search): rows = mutants of d_cur,
// scored, and the slice's first maximum (global index) in d_best / d_bidx.
int helio_engine_sampled_round(helio_gpu_ctx* ctx, const int32_t* d_cur, const int32_t* d_kmax, uint64_t round_key,
                               int64_t first, int64_t n, int max_changes, int allow_partial, int32_t* d_rows,
                               double* d_val, int32_t* d_st, double* d_best, int64_t* d_bidx, cudaStream_t st) {
  const int N = ctx->N, L = ctx->L;
  const int grid_w = (int)std::min<int64_t>(((int64_t)N * n + 255) / 256, 16 * ctx->sm_count);
  const int grid_b = (int)std::min<int64_t>((n + 255) / 256, 16 * ctx->sm_count);
  copy_rows<<<grid_w, 256, 0, st>>>(d_cur, N, n, d_rows);
  mutate_rows<<<grid_b, 256, 0, st>>>(d_cur, d_kmax, N, L, round_key, first, n, max_changes, d_rows);
  ctx->launches += 2;
  int rc = helio_gpu_score(ctx, reinterpret_cast<const int16_t*>(d_rows), n, allow_partial, d_val, d_st, st);
  if (rc) return rc;
  return helio_gpu_argmax(ctx, d_val, d_st, n, first, d_best, d_bidx, st);
}
