// DMMA fed from shared memory (as in pass_kernel): per k-step each warp loads
// NA A fragments + NB B fragments (LDS.64, conflict-free) and issues NA*NB DMMA.
#include <cstdio>
#include <cuda_runtime.h>

template <int NA, int NB, int PREF>
__global__ void __launch_bounds__(256, 1) dmma_lds(double* out, int iters) {
  __shared__ double sm[8 * 512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * 512; i += blockDim.x) sm[i] = 1e-3 * (i & 255);
  __syncthreads();
  double c[NA][NB][2];
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  const double* base = sm + lane;
  for (int it = 0; it < iters; ++it) {
    const double* p = base + (it & 3) * 32 * (NA + NB);
    double a[NA], b[NB];
#pragma unroll
    for (int i = 0; i < NA; ++i) a[i] = p[32 * i];
#pragma unroll
    for (int j = 0; j < NB; ++j) b[j] = p[32 * (NA + j)];
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][j][0]), "+d"(c[i][j][1]) : "d"(a[i]), "d"(b[j]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) s += c[i][j][0] + c[i][j][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NA, int NB>
void run(double* d) {
  const int iters = 8192;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_lds<NA, NB, 0><<<148, 256>>>(d, iters);
  cudaEventRecord(e0);
  dmma_lds<NA, NB, 0><<<148, 256>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 148.0 * 8 * iters * NA * NB * 512.0;
  printf("NA %d NB %d: %.1f TFLOP/s\n", NA, NB, fl / (ms * 1e-3) / 1e12);
}

int main() {
  double* d; cudaMalloc(&d, 1 << 20);
  run<2, 3>(d); run<2, 4>(d); run<4, 3>(d); run<4, 4>(d); run<4, 7>(d);
  return 0;
}
