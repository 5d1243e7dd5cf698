// Counter-based candidate generator G(seed, i) — SURVEY.md §8(d).
//
// Identical integer arithmetic on host and device, so every rank can
// synthesise its own shard of a global batch on device while the CPU
// reference arm scores exactly the same placements.  splitmix64 finaliser
// over (seed, global index, draw number); multiply-shift ranges.
//
// Distribution ("covering chains"):
//   1. a random node permutation (Fisher-Yates, draws 0..N-1);
//   2. each node in turn takes len ~ U[1, k_i] starting at the current layer,
//      truncated at L; after reaching L the chain wraps to layer 0;
//   3. with probability p_uniform_ppm / 1e6 a node instead takes a uniform
//      interval len ~ U[0, k_i], start ~ U[0, L - len] (len 0 = idle).
// Nodes with k_i < 1 stay idle.  Output rows are (start, end) int16 pairs in
// declared node order.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HG_HD __host__ __device__ __forceinline__
#else
#define HG_HD static inline
#endif

#define HG_GOLDEN 0x9E3779B97F4A7C15ull

HG_HD uint64_t hg_fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

HG_HD uint64_t hg_key(uint64_t seed, uint64_t i) {
  return hg_fmix(hg_fmix(seed + HG_GOLDEN) + (i + 1) * HG_GOLDEN);
}

HG_HD uint64_t hg_draw(uint64_t key, uint32_t k) {
  return hg_fmix(key + (uint64_t)(k + 1) * HG_GOLDEN);
}

// uniform integer in [0, m), m >= 1
HG_HD uint32_t hg_uniform(uint64_t x, uint32_t m) {
  return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32);
}

// perm: scratch of N int16; out: [N][2] int16.
HG_HD void hg_candidate(const int32_t* kmax, int32_t N, int32_t L, uint64_t seed, uint64_t i,
                        uint32_t ppm, int16_t* perm, int16_t* out) {
  const uint64_t key = hg_key(seed, i);
  for (int32_t k = 0; k < N; ++k) perm[k] = (int16_t)k;
  for (int32_t k = N - 1; k >= 1; --k) {
    uint32_t r = hg_uniform(hg_draw(key, (uint32_t)k), (uint32_t)(k + 1));
    int16_t t = perm[k];
    perm[k] = perm[r];
    perm[r] = t;
  }
  int32_t cur = 0;
  for (int32_t pos = 0; pos < N; ++pos) {
    int32_t node = perm[pos];
    int32_t k = kmax[node];
    int16_t s = 0, e = 0;
    uint32_t d = (uint32_t)N + 3u * (uint32_t)pos;
    if (k >= 1) {
      if (ppm > 0 && hg_uniform(hg_draw(key, d), 1000000u) < ppm) {
        uint32_t len = hg_uniform(hg_draw(key, d + 1), (uint32_t)k + 1u);
        uint32_t st = hg_uniform(hg_draw(key, d + 2), (uint32_t)(L - (int32_t)len) + 1u);
        s = (int16_t)st;
        e = (int16_t)(st + len);
      } else {
        int32_t len = 1 + (int32_t)hg_uniform(hg_draw(key, d + 1), (uint32_t)k);
        int32_t en = cur + len < L ? cur + len : L;
        s = (int16_t)cur;
        e = (int16_t)en;
        cur = en == L ? 0 : en;
      }
    }
    out[2 * node] = s;
    out[2 * node + 1] = e;
  }
}

// Link-walking chains (mode "walk"): for sparse topologies, where plain
// chains almost never connect.  From the coordinator, repeatedly step to a
// uniformly chosen unused node reachable over a declared link (coordinator
// -> node first), give it len ~ U[1, k]; on reaching L or a dead end,
// restart from the coordinator at layer 0.  Adjacency: succ_beg[N+2] /
// succ[] with row 0 = coordinator, row 1 + k = node k (link order).  `used`
// is scratch of ceil(N/32) words.  Draw numbers follow the chain steps.
HG_HD void hg_candidate_walk(const int32_t* kmax, int32_t N, int32_t L, uint64_t seed, uint64_t i,
                             const int32_t* succ_beg, const int32_t* succ, uint32_t* used,
                             int16_t* out) {
  const uint64_t key = hg_key(seed, i);
  for (int32_t w = 0; w < (N + 31) / 32; ++w) used[w] = 0u;
  for (int32_t k = 0; k < N; ++k) {
    out[2 * k] = 0;
    out[2 * k + 1] = 0;
  }
  int32_t prev = -1, cur = 0;
  uint32_t draw = 0;
  for (int32_t step = 0; step < 2 * N; ++step) {
    const int32_t b = succ_beg[prev + 1], e = succ_beg[prev + 2];
    uint32_t cnt = 0;
    for (int32_t p = b; p < e; ++p) {
      const int32_t j = succ[p];
      if (!((used[j >> 5] >> (j & 31)) & 1u) && kmax[j] >= 1) ++cnt;
    }
    if (cnt == 0) {
      if (prev == -1) break;
      prev = -1;
      cur = 0;
      continue;
    }
    uint32_t r = hg_uniform(hg_draw(key, draw++), cnt);
    int32_t j = -1;
    for (int32_t p = b; p < e; ++p) {
      const int32_t q = succ[p];
      if (!((used[q >> 5] >> (q & 31)) & 1u) && kmax[q] >= 1) {
        if (r == 0) {
          j = q;
          break;
        }
        --r;
      }
    }
    used[j >> 5] |= 1u << (j & 31);
    const int32_t len = 1 + (int32_t)hg_uniform(hg_draw(key, draw++), (uint32_t)kmax[j]);
    const int32_t en = cur + len < L ? cur + len : L;
    out[2 * j] = (int16_t)cur;
    out[2 * j + 1] = (int16_t)en;
    if (en == L) {
      prev = -1;
      cur = 0;
    } else {
      prev = j;
      cur = en;
    }
  }
}
