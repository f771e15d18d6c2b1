// FP64 pipe microbenchmarks for sm_100a: DMMA (mma.sync f64) vs DFMA, and a
// streaming-read kernel.  Used once to pick the pass-kernel design and to set
// the FP64 roofline denominator (MEASURED_PEAKS.json has no fp64 figure).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CH>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dfma_chain(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  double c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void stream_read(const double2* __restrict__ p, size_t n, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(p + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.0) out[0] = acc;
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int ctas_per_sm : {1, 2}) {
      int grid = sms * ctas_per_sm, block = warps * 32;
      float ms = time_it([&] { dmma_m8n8k4<8><<<grid, block>>>(out, iters); }, 5);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid * warps;
      printf("DMMA m8n8k4   warps/cta=%2d ctas/sm=%d : %8.2f TFLOP/s (%.3f ms)\n", warps, ctas_per_sm, flops / ms / 1e9, ms);
      ms = time_it([&] { dmma_m16n8k16<4><<<grid, block>>>(out, iters / 4); }, 5);
      flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (double)grid * warps;
      printf("DMMA m16n8k16 warps/cta=%2d ctas/sm=%d : %8.2f TFLOP/s (%.3f ms)\n", warps, ctas_per_sm, flops / ms / 1e9, ms);
      ms = time_it([&] { dfma_chain<8><<<grid, block>>>(out, iters); }, 5);
      flops = 2.0 * 8.0 * iters * (double)grid * block;
      printf("DFMA          warps/cta=%2d ctas/sm=%d : %8.2f TFLOP/s (%.3f ms)\n", warps, ctas_per_sm, flops / ms / 1e9, ms);
    }
  }
  size_t bytes = (size_t)4 << 30;
  double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  for (int cps : {2, 4, 8}) {
    float ms = time_it([&] { stream_read<<<sms * cps, 512>>>(buf, bytes / 16, out); }, 10);
    printf("stream read 4 GiB ctas/sm=%d: %8.1f GB/s\n", cps, bytes / ms / 1e6);
  }
  return 0;
}
