// Phase timing (clock64) of the one-warp Cholesky + inverse used for l <= 32.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void probe(const double* G, int l, long long* t, double* out) {
  constexpr int LD = 33;
  __shared__ double A[32 * LD], G0[32 * LD];
  __shared__ int tri_i[528], tri_k[528];
  const int lane = threadIdx.x;
  long long t0 = clock64();
  for (int e = lane; e < l * l; e += 32) G0[(e % l) + LD * (e / l)] = G[e];
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) { int q = 0; for (int k = 0; k < l; ++k) for (int i = k; i < l; ++i) { tri_i[q] = i; tri_k[q] = k; ++q; } }
  __syncwarp();
  long long t2 = clock64();
  const bool row = lane < l;
  if (row) for (int k = 0; k <= lane; ++k) A[lane + LD * k] = G0[lane + LD * k];
  __syncwarp();
  int tbase = 0;
  for (int j = 0; j < l; ++j) {
    const double d = A[j + LD * j];
    const double rd = sqrt(d);
    __syncwarp();
    if (lane > j && row) A[lane + LD * j] /= rd;
    if (lane == 0) A[j + LD * j] = rd;
    __syncwarp();
    tbase += l - j;
    const int nt = (l - j - 1) * (l - j) / 2;
    for (int q = lane; q < nt; q += 32) { const int i = tri_i[tbase + q], k = tri_k[tbase + q]; A[i + LD * k] -= A[i + LD * j] * A[k + LD * j]; }
    __syncwarp();
  }
  long long t3 = clock64();
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    double sum = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) sum -= A[i + LD * k] * x[k];
    x[i] = (i < l) ? sum / A[i + LD * i] : 0.0;
  }
  long long t4 = clock64();
  double s = 0; for (int i = 0; i < 32; ++i) s += x[i];
  out[lane] = s;
  if (lane == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; }
}
int main() {
  const int l = 25;
  double h[l * l];
  for (int j = 0; j < l; ++j) for (int i = 0; i < l; ++i) h[i + l * j] = (i == j) ? l + 1.0 : 1.0 / (1 + i + j);
  double *G, *out; long long* t;
  cudaMalloc(&G, sizeof h); cudaMalloc(&out, 256); cudaMalloc(&t, 64);
  cudaMemcpy(G, h, sizeof h, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); probe<<<1, 32>>>(G, l, t, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long ht[4]; cudaMemcpy(ht, t, 32, cudaMemcpyDeviceToHost);
    printf("event %.2f us | load %lld  tri %lld  chol %lld  inverse %lld cycles\n", ms * 1e3, ht[0], ht[1], ht[2], ht[3]);
  }
}
