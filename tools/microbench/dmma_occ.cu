// DMMA throughput vs warps per SM and independent accumulator chains:
// how many DMMAs must be in flight per SMSP to saturate the FP64 pipe.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_chains(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CH, int NF>
__global__ void dmma_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2], x[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(x[i]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CH, int NF>
void runmix(int warps, double* d) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_dfma<CH, NF><<<148, warps * 32>>>(d, iters);
  cudaEventRecord(e0);
  dmma_dfma<CH, NF><<<148, warps * 32>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 148.0 * warps * iters * CH * 512.0;
  printf("warps/SM %2d dmma %d dfma %d : %.3f ms, DMMA part %.1f TFLOP/s\n", warps, CH, NF, ms, fl / (ms * 1e-3) / 1e12);
}

template <int CH>
void run(int warps, double* d) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_chains<CH><<<148, warps * 32>>>(d, iters);
  cudaEventRecord(e0);
  dmma_chains<CH><<<148, warps * 32>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 148.0 * warps * iters * CH * 512.0;
  printf("warps/SM %2d chains %2d : %.1f TFLOP/s\n", warps, CH, fl / (ms * 1e-3) / 1e12);
}

int main() {
  double* d; cudaMalloc(&d, 1 << 20);
  runmix<6, 0>(8, d); runmix<6, 1>(8, d); runmix<6, 2>(8, d); runmix<6, 4>(8, d); runmix<8, 0>(8, d);
  return 0;
}
