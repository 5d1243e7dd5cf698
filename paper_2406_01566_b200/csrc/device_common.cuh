// device_common.cuh — slot layout and warp helpers shared by the engine's
// device code (included by helio_gpu.cu only).
#pragma once

namespace {


Layout make_layout(int V, int A, int N, int M) {
  Layout l;
  l.V = V; l.A = A; l.N = N; l.M = M;
  int o = 0;
  auto take = [&](int bytes, int align) {
    o = (o + align - 1) / align * align;
    int r = o;
    o += bytes;
    return r;
  };
  l.o_cap = take(8 * A, 16);
  // 16 B per vertex: PARITY's packed VState; SCORE reuses the bytes as a
  // double array (bottleneck) followed by an int16 array (BFS parent arc).
  l.o_vs = take(16 * V, 16);
  l.o_ex = l.o_vs;
  l.o_h = l.o_vs + 8 * V;
  l.o_to = take(2 * A, 2);
  l.o_rv = take(2 * A, 2);
  l.o_abeg = take(2 * (V + 1), 2);
  l.o_cur = take(2 * V, 2);
  l.o_q = take(2 * V, 2);
  l.o_cnt = take(2 * (2 * V + 1), 4);  // SCORE: int32 parent words
  l.o_ps = take(2 * N, 4);
  l.o_pe = take(2 * N, 2);
  l.o_vin = take(2 * N, 2);
  l.o_unode = take(2 * N, 2);
  l.o_efwd = take(2 * M, 2);
  l.o_inq = take(V, 1);
  l.bytes = (o + 15) / 16 * 16;
  return l;
}

// SCORE layout for the general path (N > 64: per-node-list builder + queue
// BFS), which touches only cap/to/rv/abeg/cur/q/h/ex/ps/pe: 12A + 16V + 4N
// bytes instead of 12A + 27V + 8N, so more graphs stay resident per SM.  The
// regions that path never touches alias live ones.
Layout make_layout_score_general(int V, int A, int N) {
  Layout l;
  l.V = V; l.A = A; l.N = N; l.M = 0;
  int o = 0;
  auto take = [&](int bytes, int align) {
    o = (o + align - 1) / align * align;
    int r = o;
    o += bytes;
    return r;
  };
  l.o_cap = take(8 * A, 16);
  l.o_ex = take(8 * V, 16);  // builder: int fill counters; BFS: bottleneck per vertex
  l.o_vs = l.o_ex;
  l.o_to = take(2 * A, 2);
  l.o_rv = take(2 * A, 2);
  l.o_abeg = take(2 * (V + 1), 2);
  l.o_h = take(2 * V, 2);
  l.o_cur = take(2 * V, 2);
  l.o_q = take(2 * V, 2);
  l.o_ps = take(2 * N, 4);
  l.o_pe = take(2 * N, 2);
  l.o_cnt = l.o_q;
  l.o_inq = l.o_ps;  // push-relabel FIFO flags (V <= 4N bytes) over the builder's ps/pe
  l.o_vin = l.o_ps;
  l.o_unode = l.o_ps;
  l.o_efwd = l.o_ps;
  l.bytes = (o + 15) / 16 * 16;
  return l;
}

// SCORE layout of the large-graph path (GEN kernel; series-contracted
// networks, build_graph_score_contract): V and A count the CONTRACTED graph.
// The builder's per-node scratch sits behind the solver arrays: packed
// intervals (4N), int32 in/out degrees (8N; the solver's FIFO flags reuse it),
// int16 kept-vertex ids (4N), int32 unique out-link of a removed out-vertex
// (4N).  12A + 16V + 20N bytes.
Layout make_layout_contract(int V, int A, int N) {
  Layout l;
  l.V = V; l.A = A; l.N = N; l.M = 0;
  int o = 0;
  auto take = [&](int bytes, int align) {
    o = (o + align - 1) / align * align;
    int r = o;
    o += bytes;
    return r;
  };
  l.o_cap = take(8 * A, 16);
  l.o_ex = take(8 * V, 16);  // builder: int degree / slot counters per contracted vertex
  l.o_vs = l.o_ex;
  l.o_to = take(2 * A, 2);
  l.o_rv = take(2 * A, 2);
  l.o_abeg = take(2 * (V + 1), 2);
  l.o_h = take(2 * V, 2);
  l.o_cur = take(2 * V, 2);
  l.o_q = take(2 * V, 2);
  l.o_cnt = l.o_q;
  l.o_ps = take(4 * N, 4);
  l.o_pe = l.o_ps + 2 * N;
  l.o_efwd = take(8 * N, 8);  // din [N], dout [N] (int32)
  l.o_inq = l.o_efwd;         // V <= 2N + 2 <= 8N bytes
  l.o_vin = take(4 * N, 4);   // vin [N], vout [N] (int16, -1 = contracted away)
  l.o_unode = take(4 * N, 4); // succ [N] (int32 link index)
  l.bytes = (o + 15) / 16 * 16;
  return l;
}

// PARITY per-vertex solver state, one 16-byte shared-memory record so a
// discharge loads it with a single LDS.128.
struct __align__(16) VState {
  double ex;     // excess
  int16_t h;     // height
  int16_t cur;   // current-arc index (relative)
  int16_t b;     // first arc
  int16_t deg;   // arc count
};

// Per-warp view of a slot.
struct Gs {
  VState* vs;
  double* cap;
  double* ex;
  int16_t* to;
  int16_t* rv;
  int16_t* abeg;
  int16_t* h;
  int16_t* cur;
  int16_t* q;
  int16_t* cnt;
  uint8_t* inq;
  int16_t* ps;
  int16_t* pe;
  int16_t* vin;
  int16_t* unode;
  int16_t* efwd;
};

__device__ __forceinline__ Gs slot_view(char* base, const Layout& l) {
  Gs g;
  g.vs = reinterpret_cast<VState*>(base + l.o_vs);
  g.cap = reinterpret_cast<double*>(base + l.o_cap);
  g.ex = reinterpret_cast<double*>(base + l.o_ex);
  g.to = reinterpret_cast<int16_t*>(base + l.o_to);
  g.rv = reinterpret_cast<int16_t*>(base + l.o_rv);
  g.abeg = reinterpret_cast<int16_t*>(base + l.o_abeg);
  g.h = reinterpret_cast<int16_t*>(base + l.o_h);
  g.cur = reinterpret_cast<int16_t*>(base + l.o_cur);
  g.q = reinterpret_cast<int16_t*>(base + l.o_q);
  g.cnt = reinterpret_cast<int16_t*>(base + l.o_cnt);
  g.inq = reinterpret_cast<uint8_t*>(base + l.o_inq);
  g.ps = reinterpret_cast<int16_t*>(base + l.o_ps);
  g.pe = reinterpret_cast<int16_t*>(base + l.o_pe);
  g.vin = reinterpret_cast<int16_t*>(base + l.o_vin);
  g.unode = reinterpret_cast<int16_t*>(base + l.o_unode);
  g.efwd = reinterpret_cast<int16_t*>(base + l.o_efwd);
  return g;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// std::min(a, b) == (b < a) ? b : a
__device__ __forceinline__ double ref_min(double a, double b) { return b < a ? b : a; }

}  // namespace
