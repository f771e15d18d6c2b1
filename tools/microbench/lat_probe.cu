// Latency probes for the single-CTA small-matrix phases (cycles, clock64):
// dependent chains of double rsqrt, double division, DFMA, LDS round trips,
// __syncthreads, __shfl_sync, with 256 threads active.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, double seed, int n) {
  __shared__ double sm[256 + 64];
  const int t = threadIdx.x;
  sm[t] = seed + t;
  __syncthreads();
  double x = seed + t * 1e-3;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.0;
  long long c1 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
  long long c2 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999, 1e-3);
  long long c3 = clock64();
  for (int i = 0; i < n; ++i) { sm[t] = x; x = sm[(t + 1) & 255] * 0.5 + 1.0; }
  long long c4 = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); }
  long long c5 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (t + 1) & 31) * 0.5 + 1.0;
  long long c6 = clock64();
  for (int i = 0; i < n; ++i) { sm[t] = x; __syncthreads(); x = sm[(t + 8) & 255] * 0.5 + 1.0; }
  long long c7 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  long long c8 = clock64();
  out[blockIdx.x * 256 + t] = x;
  if (t == 0) {
    cyc[0] = (c1 - c0) / n; cyc[1] = (c2 - c1) / n; cyc[2] = (c3 - c2) / n; cyc[3] = (c4 - c3) / n;
    cyc[4] = (c5 - c4) / n; cyc[5] = (c6 - c5) / n; cyc[6] = (c7 - c6) / n; cyc[7] = (c8 - c7) / n;
  }
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 256 * 8 * 2); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<1, 256>>>(d, c, 1.5, 1000);
    long long h[8];
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("rsqrt %lld  div %lld  dfma %lld  sts+lds %lld  syncthreads %lld  shfl %lld  sts+bar+lds %lld  sqrt %lld\n",
           h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
