// Latency probes for the masked-routing replay (one warp): dependent chains
// of DDIV / DMUL / DADD / LDS / VOTE+SHFL, cycles per operation.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, int n, double seed) {
  __shared__ double sm[256];
  for (int i = threadIdx.x; i < 256; i += 32) sm[i] = 1.0 + i * 1e-3;
  __syncwarp();
  double a = seed, b = 1.0 + seed;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = (a + 3.0) / (b + i);            // DADD + DDIV chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = a * 1.0000001 + 1e-9;            // DMUL + DADD chain
  long long t2 = clock64();
  int k = (int)a & 255;
  for (int i = 0; i < n; ++i) k = ((int)sm[k] + k + 1) & 255;      // LDS + F2I chain
  long long t3 = clock64();
  unsigned m = 1;
  for (int i = 0; i < n; ++i) {
    m = __ballot_sync(0xffffffffu, (threadIdx.x + m) & 1);
    m = __shfl_sync(0xffffffffu, m, m & 31) | 1;
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    out[0] = a + k + m;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 8); cudaMalloc(&c, 32);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) probe<<<1, 32>>>(d, c, n, 0.5);
  long long h[4];
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("cycles/op: dadd+ddiv %.1f  dmul+dadd %.1f  lds+f2i %.1f  ballot+shfl %.1f\n", h[0] / (double)n,
         h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
  return 0;
}
