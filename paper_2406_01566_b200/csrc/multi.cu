// multi.cu — multi-GPU entry points of the C ABI.
//
// The path shards by candidate: every candidate is independent, so a batch is
// split into contiguous global-index ranges and the only exchange is the
// argmax (tests/oracles/enumerate.hpp:56-59: strict '>' over the enumeration
// order = max value, then min index).  Two forms:
//
// * ranked (one process per GPU): helio_gpu_argmax_ranked reduces this rank's
//   shard on the device, all-gathers the 16-byte (value bits, global index)
//   records over an NCCL communicator and reduces them on the device — stream
//   ordered, no host synchronisation.  helio_gpu_nccl_* create the
//   communicator for callers that have none (the unique id travels over the
//   caller's own channel: MPI, torch.distributed, a file).
// * multi-device (one process, several GPUs): helio_gpu_multi_* own one
//   context per device; host batches are split across them with one host
//   thread per device and the per-device first maxima merged on the host.
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is resolved at run time (nccl_api below)

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"
#include "gen.h"

using namespace helio_engine;

int helio_engine_argmax(helio_gpu_ctx* ctx, const double* d_values, const int32_t* d_status, int64_t B,
                        int64_t index_base, double* d_best, int64_t* d_index, cudaStream_t st);
int helio_engine_sampled_round(helio_gpu_ctx* ctx, const int32_t* d_cur, const int32_t* d_kmax, uint64_t round_key,
                               int64_t first, int64_t n, int max_changes, int allow_partial, int32_t* d_rows,
                               double* d_val, int32_t* d_st, double* d_best, int64_t* d_bidx, cudaStream_t st);

namespace {

// NCCL is bound lazily, never as a load-time dependency: a process that also
// uses torch.distributed must share torch's libnccl.so.2 (whose newer symbols
// torch needs), so the library already loaded under that soname is used when
// there is one (RTLD_NOLOAD), else $HELIO_NCCL_LIB, else the system
// libnccl.so.2.  The Python bindings import torch first when it is installed.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  bool ok = false;
};

const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) {
      const char* env = std::getenv("HELIO_NCCL_LIB");
      if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.comm_count = reinterpret_cast<decltype(api.comm_count)>(dlsym(h, "ncclCommCount"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count && api.all_gather;
  });
  return api;
}

__global__ void pack_record(const double* __restrict__ best, const int64_t* __restrict__ index,
                            long long* __restrict__ rec) {
  rec[0] = __double_as_longlong(*best);
  rec[1] = (long long)*index;
}

// rank records in rank order = global index order of the shards: max value,
// then min index among valid (index >= 0) records
__global__ void reduce_records(const long long* __restrict__ recs, int n, double* best, int64_t* index) {
  double bv = 0.0;
  long long bi = -1;
  for (int r = 0; r < n; ++r) {
    const long long i = recs[2 * r + 1];
    const double v = __longlong_as_double(recs[2 * r]);
    if (i >= 0 && (bi < 0 || v > bv || (v == bv && i < bi))) {
      bv = v;
      bi = i;
    }
  }
  *best = bv;
  *index = bi;
}

}  // namespace

struct helio_gpu_multi {
  std::vector<helio_gpu_ctx*> ctx;
  std::vector<int> device;
  int N = 0;
  std::string err;
  std::mutex mu;
};

extern "C" {

int helio_gpu_nccl_unique_id(uint8_t* id128) {
  if (!id128) return HELIO_ERR_INVALID;
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return HELIO_ERR_CUDA;
  ncclUniqueId id;
  if (nc.get_unique_id(&id) != ncclSuccess) return HELIO_ERR_CUDA;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, 128);
  return HELIO_OK;
}

int helio_gpu_nccl_comm_create(const uint8_t* id128, int32_t nranks, int32_t rank, int32_t device, void** comm) {
  if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return HELIO_ERR_INVALID;
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return HELIO_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return HELIO_ERR_CUDA;
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  ncclComm_t c = nullptr;
  if (nc.comm_init_rank(&c, nranks, id, rank) != ncclSuccess) return HELIO_ERR_CUDA;
  *comm = c;
  return HELIO_OK;
}

int helio_gpu_nccl_comm_destroy(void* comm) {
  if (!comm) return HELIO_OK;
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return HELIO_ERR_CUDA;
  return nc.comm_destroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? HELIO_OK : HELIO_ERR_CUDA;
}

int helio_gpu_argmax_ranked(helio_gpu_ctx* ctx, const double* d_values, const int32_t* d_status, int64_t B,
                            int64_t index_base, double* d_best, int64_t* d_index, void* comm, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!comm || !d_best || !d_index || B < 0 || (B > 0 && (!d_values || !d_status)))
    return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return fail(ctx, HELIO_ERR_CUDA, "NCCL (libnccl.so.2) could not be loaded");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int n = 0;
  if (nc.comm_count(c, &n) != ncclSuccess || n < 1) return fail(ctx, HELIO_ERR_CUDA, "ncclCommCount failed");
  // records: [0, 2) this rank's, [2, 2 + 2n) everyone's — in the context's
  // host-entry arena (grow-only; this call is stream ordered on `st`, so the
  // arena's synchronous host users are ordered behind it by api_begin/end)
  char* base = nullptr;
  int rc = host_arena(ctx, sizeof(long long) * (2 + 2 * (size_t)n), &base);
  if (rc) return rc;
  long long* rec = reinterpret_cast<long long*>(base);
  long long* all = rec + 2;
  CK(api_begin(ctx, st));
  rc = helio_engine_argmax(ctx, d_values, d_status, B, index_base, d_best, d_index, st);
  if (rc) return rc;
  pack_record<<<1, 1, 0, st>>>(d_best, d_index, rec);
  if (nc.all_gather(rec, all, 2, ncclInt64, c, st) != ncclSuccess)
    return fail(ctx, HELIO_ERR_CUDA, "ncclAllGather failed");
  reduce_records<<<1, 1, 0, st>>>(all, n, d_best, d_index);
  CK(cudaGetLastError());
  CK(api_end(ctx, st));
  ctx->launches += 2;
  return HELIO_OK;
}

// --- one process, several devices ---------------------------------------------

int helio_gpu_multi_create(const int32_t* devices, int32_t n, helio_gpu_multi** out) {
  if (!devices || n < 1 || !out) return HELIO_ERR_INVALID;
  auto* m = new helio_gpu_multi;
  for (int i = 0; i < n; ++i) {
    helio_gpu_ctx* c = nullptr;
    const int rc = helio_gpu_create(devices[i], &c);
    if (rc != HELIO_OK) {
      for (helio_gpu_ctx* x : m->ctx) helio_gpu_destroy(x);
      delete m;
      return rc;
    }
    m->ctx.push_back(c);
    m->device.push_back(devices[i]);
  }
  *out = m;
  return HELIO_OK;
}

void helio_gpu_multi_destroy(helio_gpu_multi* m) {
  if (!m) return;
  for (helio_gpu_ctx* c : m->ctx) helio_gpu_destroy(c);
  delete m;
}

const char* helio_gpu_multi_last_error(const helio_gpu_multi* m) { return m ? m->err.c_str() : "null handle"; }

int32_t helio_gpu_multi_count(const helio_gpu_multi* m) { return m ? (int32_t)m->ctx.size() : 0; }

helio_gpu_ctx* helio_gpu_multi_context(helio_gpu_multi* m, int32_t i) {
  return m && i >= 0 && i < (int)m->ctx.size() ? m->ctx[i] : nullptr;
}

int helio_gpu_multi_set_cluster(helio_gpu_multi* m, const helio_cluster_desc* desc, int32_t* k_out) {
  if (!m || !desc) return HELIO_ERR_INVALID;
  std::lock_guard<std::mutex> lock(m->mu);
  for (size_t i = 0; i < m->ctx.size(); ++i) {
    const int rc = helio_gpu_set_cluster(m->ctx[i], desc, i == 0 ? k_out : nullptr);
    if (rc != HELIO_OK) {
      m->err = helio_gpu_last_error(m->ctx[i]);
      return rc;
    }
  }
  m->N = desc->num_nodes;
  return HELIO_OK;
}

int helio_gpu_multi_set_mode(helio_gpu_multi* m, int mode) {
  if (!m) return HELIO_ERR_INVALID;
  std::lock_guard<std::mutex> lock(m->mu);
  for (helio_gpu_ctx* c : m->ctx) {
    const int rc = helio_gpu_set_mode(c, mode);
    if (rc != HELIO_OK) {
      m->err = helio_gpu_last_error(c);
      return rc;
    }
  }
  return HELIO_OK;
}

int helio_gpu_multi_score_best_host(helio_gpu_multi* m, const int16_t* h_pl, int64_t B, int allow_partial,
                                    double* h_values, int32_t* h_status, double* h_best, int64_t* h_index) {
  if (!m) return HELIO_ERR_INVALID;
  std::lock_guard<std::mutex> lock(m->mu);
  if (m->N <= 0) {
    m->err = "no cluster set";
    return HELIO_ERR_NO_CLUSTER;
  }
  if (B < 0 || !h_best || !h_index || (B > 0 && !h_pl) || ((!h_values) != (!h_status))) {
    m->err = "bad buffers";
    return HELIO_ERR_INVALID;
  }
  const int n = (int)m->ctx.size();
  std::vector<int> rc(n, HELIO_OK);
  std::vector<double> best(n, 0.0);
  std::vector<int64_t> idx(n, -1);
  std::vector<std::thread> pool;
  for (int i = 0; i < n; ++i) {
    const int64_t lo = B * i / n, hi = B * (i + 1) / n;
    if (hi <= lo) continue;
    pool.emplace_back([&, i, lo, hi] {
      rc[i] = helio_gpu_score_best_host(m->ctx[i], h_pl + lo * 2 * m->N, hi - lo, allow_partial,
                                        h_values ? h_values + lo : nullptr, h_status ? h_status + lo : nullptr,
                                        &best[i], &idx[i]);
      if (idx[i] >= 0) idx[i] += lo;
    });
  }
  for (auto& t : pool) t.join();
  double bv = 0.0;
  int64_t bi = -1;
  for (int i = 0; i < n; ++i) {  // shards in index order
    if (rc[i] != HELIO_OK) {
      m->err = helio_gpu_last_error(m->ctx[i]);
      return rc[i];
    }
    if (idx[i] >= 0 && (bi < 0 || best[i] > bv)) {
      bv = best[i];
      bi = idx[i];
    }
  }
  *h_best = bv;
  *h_index = bi;
  return HELIO_OK;
}

}  // extern "C"

// Sampled multi-node search (helio_gpu_sampled_search) over several devices:
// each round's `batch` counter-drawn mutants are split into contiguous slices,
// one per device, every device scores its slice and reduces its first
// maximum, and the host merges them in index order — the same mutants and the
// same tie-break as one device, so the same search path and result.
extern "C" int helio_gpu_multi_sampled_search(helio_gpu_multi* m, const int16_t* h_seed, int allow_partial,
                                              int32_t iterations, int64_t batch, int32_t max_changes,
                                              uint64_t rng_seed, double* h_value, int16_t* h_row,
                                              int32_t* h_improvements, int64_t* h_scored) {
  if (!m) return HELIO_ERR_INVALID;
  std::lock_guard<std::mutex> lock(m->mu);
  if (m->N <= 0) {
    m->err = "no cluster set";
    return HELIO_ERR_NO_CLUSTER;
  }
  if (!h_seed || !h_value || !h_row || iterations < 0 || batch < 1 || max_changes < 1) {
    m->err = "bad arguments";
    return HELIO_ERR_INVALID;
  }
  const int nd = (int)m->ctx.size(), N = m->N;
  struct Dev {
    int32_t *cur = nullptr, *kmax = nullptr, *rows = nullptr, *st = nullptr;
    double *val = nullptr, *best = nullptr;
    int64_t* bidx = nullptr;
    int64_t lo = 0, n = 0;
    int rc = HELIO_OK;
    double hb = 0;
    int64_t hi = -1;
  };
  std::vector<Dev> dv(nd);
  std::vector<int32_t> cur(N);
  for (int i = 0; i < N; ++i)
    cur[i] = (int32_t)(uint16_t)h_seed[2 * i] | (int32_t)((uint32_t)(uint16_t)h_seed[2 * i + 1] << 16);
  int rc = HELIO_OK;
  auto fail_m = [&](int code, const std::string& msg) {
    m->err = msg;
    return code;
  };
  for (int d = 0; d < nd && !rc; ++d) {
    helio_gpu_ctx* c = m->ctx[d];
    Dev& x = dv[d];
    x.lo = batch * d / nd;
    x.n = batch * (d + 1) / nd - x.lo;
    if (cudaSetDevice(c->device) != cudaSuccess ||
        cudaMalloc(&x.cur, 4 * N) != cudaSuccess || cudaMalloc(&x.kmax, 4 * N) != cudaSuccess ||
        cudaMalloc(&x.rows, 4 * (size_t)N * std::max<int64_t>(x.n, 1)) != cudaSuccess ||
        cudaMalloc(&x.val, 8 * std::max<int64_t>(x.n, 1)) != cudaSuccess ||
        cudaMalloc(&x.st, 4 * std::max<int64_t>(x.n, 1)) != cudaSuccess || cudaMalloc(&x.best, 8) != cudaSuccess ||
        cudaMalloc(&x.bidx, 8) != cudaSuccess ||
        cudaMemcpy(x.cur, cur.data(), 4 * N, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(x.kmax, c->h_kmax.data(), 4 * N, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = fail_m(HELIO_ERR_CUDA, "multi sampled search: allocation failed");
  }
  // the seed's value on device 0
  double value = 0.0;
  if (!rc) {
    helio_gpu_ctx* c = m->ctx[0];
    int32_t s0 = 0;
    rc = helio_gpu_score(c, reinterpret_cast<const int16_t*>(dv[0].cur), 1, allow_partial, dv[0].val, dv[0].st,
                         c->stream);
    // read back on the context's (non-blocking) stream the score ran on
    if (!rc && (cudaMemcpyAsync(&value, dv[0].val, 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                cudaMemcpyAsync(&s0, dv[0].st, 4, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                cudaStreamSynchronize(c->stream) != cudaSuccess))
      rc = HELIO_ERR_CUDA;
    if (rc) m->err = helio_gpu_last_error(c);
    if (!rc && s0 != 0) rc = fail_m(HELIO_ERR_INVALID, "seed placement fails validation");
  }
  double best_value = value;
  std::vector<int32_t> keep = cur;
  int32_t improvements = 0;
  int64_t scored = 1;
  for (int32_t it = 0; !rc && it < iterations; ++it) {
    const uint64_t key = hg_key(rng_seed, (uint64_t)it);
    std::vector<std::thread> pool;
    for (int d = 0; d < nd; ++d) {
      if (dv[d].n == 0) continue;
      pool.emplace_back([&, d] {
        helio_gpu_ctx* c = m->ctx[d];
        Dev& x = dv[d];
        std::lock_guard<std::recursive_mutex> ctx_lock(c->mu);
        cudaSetDevice(c->device);
        x.rc = helio_engine_sampled_round(c, x.cur, x.kmax, key, x.lo, x.n, max_changes, allow_partial, x.rows, x.val,
                                          x.st, x.best, x.bidx, c->stream);
        if (!x.rc && (cudaMemcpyAsync(&x.hb, x.best, 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                      cudaMemcpyAsync(&x.hi, x.bidx, 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                      cudaStreamSynchronize(c->stream) != cudaSuccess))
          x.rc = HELIO_ERR_CUDA;
      });
    }
    for (auto& t : pool) t.join();
    double best = 0.0;
    int64_t bi = -1;
    int owner = -1;
    for (int d = 0; d < nd && !rc; ++d) {  // slices in index order: strict '>' keeps the first maximum
      if (dv[d].n == 0) continue;
      if (dv[d].rc) {
        rc = dv[d].rc;
        m->err = helio_gpu_last_error(m->ctx[d]);
        break;
      }
      if (dv[d].hi >= 0 && (bi < 0 || dv[d].hb > best)) {
        best = dv[d].hb;
        bi = dv[d].hi;
        owner = d;
      }
    }
    if (rc) break;
    scored += batch;
    if (bi >= 0 && best >= value) {  // equal values: a sideways move along the plateau
      Dev& o = dv[owner];
      cudaSetDevice(m->ctx[owner]->device);
      if (cudaMemcpy(cur.data(), o.rows + (bi - o.lo) * N, 4 * N, cudaMemcpyDeviceToHost) != cudaSuccess) {
        rc = fail_m(HELIO_ERR_CUDA, "multi sampled search: row read-back failed");
        break;
      }
      if (best > best_value) {
        best_value = best;
        ++improvements;
        keep = cur;
      }
      value = best;
      for (int d = 0; d < nd && !rc; ++d) {
        cudaSetDevice(m->ctx[d]->device);
        if (cudaMemcpy(dv[d].cur, cur.data(), 4 * N, cudaMemcpyHostToDevice) != cudaSuccess)
          rc = fail_m(HELIO_ERR_CUDA, "multi sampled search: update failed");
      }
    }
  }
  for (int d = 0; d < nd; ++d) {
    cudaSetDevice(m->ctx[d]->device);
    cudaFree(dv[d].cur);
    cudaFree(dv[d].kmax);
    cudaFree(dv[d].rows);
    cudaFree(dv[d].val);
    cudaFree(dv[d].st);
    cudaFree(dv[d].best);
    cudaFree(dv[d].bidx);
  }
  if (rc) return rc;
  *h_value = best_value;
  for (int i = 0; i < N; ++i) {
    h_row[2 * i] = (int16_t)(keep[i] & 0xffff);
    h_row[2 * i + 1] = (int16_t)((uint32_t)keep[i] >> 16);
  }
  if (h_improvements) *h_improvements = improvements;
  if (h_scored) *h_scored = scored;
  return HELIO_OK;
}
