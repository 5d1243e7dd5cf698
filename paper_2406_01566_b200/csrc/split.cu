// split.cu — the split K1 -> HBM -> K2 pipeline of north_star / SURVEY.md §8(d).
//
//   K1 csr_build_kernel  placement row -> the reference's flow network (same
//                        builders as the fused kernel) -> one fixed-size slab
//                        per candidate in HBM, written with coalesced 16-byte
//                        stores: {V, E, status} | int32 arc offsets [V+1] |
//                        int32 arcs (head | rev << 16) [2E] | f64 capacities [2E]
//   K2 csr_solve_kernel  slab -> shared memory (16-byte loads) -> the PARITY
//                        FIFO preflow-push replay -> value
//
// The production path is the fused kernel (score_kernel), which never writes
// the network to HBM; this pipeline exists to expose K1's output and to
// measure the design choice (bench.py `split_pipeline`): the slab is ~4.8 KB
// per het42 candidate, written once and read once.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/helio_gpu.h"
#include "engine.h"

using namespace helio_engine;

#define FLOW_EPS 1e-12  // kFlowEps, flow_graph.cpp:15
#define FULL 0xffffffffu
#define ST_OVERFLOW 100

#include "device_common.cuh"
#include "build.cuh"
#include "solve_parity.cuh"

namespace {

struct Slab {
  int V, A;       // capacities
  int o_abeg, o_arc, o_cap, bytes;
};

Slab make_slab(int V, int A) {
  Slab s;
  s.V = V;
  s.A = A;
  int o = 16;  // meta: V, E, status, pad
  s.o_abeg = o;
  o += (4 * (V + 1) + 15) / 16 * 16;
  s.o_arc = o;
  o += (4 * A + 15) / 16 * 16;
  s.o_cap = o;
  o += 8 * A;
  s.bytes = (o + 127) / 128 * 128;
  return s;
}

// 16-byte vector copy between shared and global memory by a warp
__device__ __forceinline__ void warp_copy16(void* dst, const void* src, int bytes, int lane) {
  const int n16 = bytes >> 4;
  uint4* d = reinterpret_cast<uint4*>(dst);
  const uint4* s = reinterpret_cast<const uint4*>(src);
  for (int i = lane; i < n16; i += 32) d[i] = s[i];
}

__global__ void csr_build_kernel(ClusterDev cd, Layout lay, Slab sl, const int16_t* __restrict__ pl, int64_t B,
                                 int partial, char* __restrict__ slabs, int32_t* __restrict__ status,
                                 unsigned long long* work) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Gs g = slot_view(smem + wib * lay.bytes, lay);
  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(work, 1ull);
    w = __shfl_sync(FULL, w, 0);
    if ((int64_t)w >= B) break;
    const int64_t b = (int64_t)w;
    char* out = slabs + b * (int64_t)sl.bytes;
    int V = 0, E = 0;
    int st = cd.less_cout ? build_graph_small(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E)
                          : build_graph(cd, g, lay, pl + b * 2 * cd.N, partial, lane, V, E);
    if (st == ST_OVERFLOW || (st == 0 && (V > sl.V || 2 * E > sl.A))) st = HELIO_CAND_TOO_LARGE;
    if (st == 0) {
      const int A = 2 * E;
      // arc offsets and packed heads/reverse indices through a shared staging
      // area (the slot's count/queue regions are free before the solve)
      int32_t* sabeg = reinterpret_cast<int32_t*>(g.vs);  // 16V bytes >= 4(V+1)
      for (int x = lane; x <= V; x += 32) sabeg[x] = g.abeg[x];
      __syncwarp();
      warp_copy16(out + sl.o_abeg, sabeg, (4 * (V + 1) + 15) & ~15, lane);
      __syncwarp();
      int32_t* sarc = reinterpret_cast<int32_t*>(g.vs);  // reuse after the copy
      for (int a0 = 0; a0 < A; a0 += 4 * V) {
        const int n = min(4 * V, A - a0);
        for (int a = lane; a < n; a += 32)
          sarc[a] = (int32_t)((uint16_t)g.to[a0 + a]) | ((int32_t)((uint16_t)g.rv[a0 + a]) << 16);
        __syncwarp();
        warp_copy16(out + sl.o_arc + 4 * a0, sarc, (4 * n + 15) & ~15, lane);
        __syncwarp();
      }
      warp_copy16(out + sl.o_cap, g.cap, (8 * A + 15) & ~15, lane);
    }
    if (lane == 0) {
      int32_t* meta = reinterpret_cast<int32_t*>(out);
      meta[0] = V;
      meta[1] = E;
      meta[2] = st;
      status[b] = st;
    }
    __syncwarp();
  }
}

__global__ void csr_solve_kernel(Layout lay, Slab sl, const char* __restrict__ slabs, int64_t B,
                                 double* __restrict__ values, int32_t* __restrict__ status,
                                 unsigned long long* work) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Gs g = slot_view(smem + wib * lay.bytes, lay);
  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(work, 1ull);
    w = __shfl_sync(FULL, w, 0);
    if ((int64_t)w >= B) break;
    const int64_t b = (int64_t)w;
    const char* in = slabs + b * (int64_t)sl.bytes;
    const int32_t* meta = reinterpret_cast<const int32_t*>(in);
    const int V = __ldg(meta), E = __ldg(meta + 1), st = __ldg(meta + 2);
    double value = 0.0;
    if (st == 0) {
      const int A = 2 * E;
      const int32_t* abeg = reinterpret_cast<const int32_t*>(in + sl.o_abeg);
      const int32_t* arc = reinterpret_cast<const int32_t*>(in + sl.o_arc);
      warp_copy16(g.cap, in + sl.o_cap, (8 * A + 15) & ~15, lane);
      for (int x = lane; x <= V; x += 32) g.abeg[x] = (int16_t)__ldg(abeg + x);
      for (int a = lane; a < A; a += 32) {
        const int32_t p = __ldg(arc + a);
        g.to[a] = (int16_t)(p & 0xffff);
        g.rv[a] = (int16_t)(p >> 16);
      }
      __syncwarp();
      solve_fifo2(g, V, 0, 1, lane);
      // net flow into the sink in edge order (:222-227): the sink's arcs are
      // the reverses of the node -> coordinator edges, in edge order
      if (lane == 0) {
        const double* cap0 = reinterpret_cast<const double*>(in + sl.o_cap);
        for (int a = g.abeg[1]; a < g.abeg[2]; ++a) {
          const int fa = g.rv[a];
          double f = __ldg(cap0 + fa) - g.cap[fa];
          if (f < FLOW_EPS) f = 0.0;
          value += f;
        }
      }
    }
    if (lane == 0) {
      values[b] = value;
      status[b] = st;
    }
    __syncwarp();
  }
}

Slab slab_of(const helio_gpu_ctx* ctx) { return make_slab(ctx->small.V, ctx->small.A); }

}  // namespace

extern "C" int64_t helio_gpu_csr_slab_bytes(const helio_gpu_ctx* ctx) {
  if (!ctx || !ctx->has_cluster) return -1;
  return slab_of(ctx).bytes;
}

extern "C" int helio_gpu_build_csr(helio_gpu_ctx* ctx, const int16_t* d_pl, int64_t B, int allow_partial,
                                   void* d_slabs, int32_t* d_status, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (B < 0 || (B > 0 && (!d_pl || !d_slabs || !d_status))) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (B == 0) return HELIO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const Slab sl = slab_of(ctx);
  const int warps = ctx->small_warps;
  const size_t smem = (size_t)ctx->small.bytes * warps;
  CK(cudaFuncSetAttribute(csr_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(csr_build_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_build_kernel, 32 * warps, smem));
  const int grid = (int)std::min<int64_t>((int64_t)std::max(per_sm, 1) * ctx->sm_count, (B + warps - 1) / warps);
  CK(api_begin(ctx, st));
  CK(cudaMemsetAsync(ctx->d_work + 8, 0, sizeof(unsigned long long), st));
  csr_build_kernel<<<grid, 32 * warps, smem, st>>>(ctx->cd, ctx->small, sl, d_pl, B, allow_partial ? 1 : 0,
                                                   static_cast<char*>(d_slabs), d_status, ctx->d_work + 8);
  CK(cudaGetLastError());
  CK(api_end(ctx, st));
  ctx->launches++;
  return HELIO_OK;
}

extern "C" int helio_gpu_solve_csr(helio_gpu_ctx* ctx, const void* d_slabs, int64_t B, double* d_values,
                                   int32_t* d_status, void* stream) {
  if (!ctx) return HELIO_ERR_INVALID;
  std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);  // contexts serialise their callers
  if (!ctx->has_cluster) return fail(ctx, HELIO_ERR_NO_CLUSTER, "no cluster set");
  if (B < 0 || (B > 0 && (!d_slabs || !d_values || !d_status))) return fail(ctx, HELIO_ERR_INVALID, "bad buffers");
  if (B == 0) return HELIO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const Slab sl = slab_of(ctx);
  const int warps = ctx->small_warps;
  const size_t smem = (size_t)ctx->small.bytes * warps;
  CK(cudaFuncSetAttribute(csr_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(csr_solve_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_solve_kernel, 32 * warps, smem));
  const int grid = (int)std::min<int64_t>((int64_t)std::max(per_sm, 1) * ctx->sm_count, (B + warps - 1) / warps);
  CK(api_begin(ctx, st));
  CK(cudaMemsetAsync(ctx->d_work + 9, 0, sizeof(unsigned long long), st));
  csr_solve_kernel<<<grid, 32 * warps, smem, st>>>(ctx->small, sl, static_cast<const char*>(d_slabs), B, d_values,
                                                   d_status, ctx->d_work + 9);
  CK(cudaGetLastError());
  CK(api_end(ctx, st));
  ctx->launches++;
  return HELIO_OK;
}
