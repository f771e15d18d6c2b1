// Do DMMA (mma.sync f64) and DFMA share the FP64 datapath on sm_100a?
// Times DMMA-only, DFMA-only and interleaved work of the same amounts.
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF>
__global__ void mix(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  double f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i % 8][0]), "+d"(c[i % 8][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i % 8] = fma(f[i % 8], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <class K>
float run(K k, int iters) {
  double* out; cudaMalloc(&out, 1 << 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148, 512>>>(out, iters); cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); k<<<148, 512>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const int it = 4096;
  float tm = run(mix<8, 0>, it), tf = run(mix<0, 64>, it), tb = run(mix<8, 64>, it);
  // flops: DMMA 8 x 512 per warp-instr per warp; DFMA 64 x 2 per thread
  double fm = 148.0 * 16 * 8 * 512.0 * it, ff = 148.0 * 512 * 64 * 2.0 * it;
  printf("DMMA only: %.3f ms (%.1f TF)\nDFMA only: %.3f ms (%.1f TF)\nboth:      %.3f ms (%.1f TF combined)\n",
         tm, fm / tm / 1e9, tf, ff / tf / 1e9, tb, (fm + ff) / tb / 1e9);
  float tb2 = run(mix<8, 16>, it);
  printf("DMMA + 1/4 DFMA: %.3f ms (%.1f TF combined)\n", tb2, (fm + ff / 4) / tb2 / 1e9);
  return 0;
}
