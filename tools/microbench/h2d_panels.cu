// H2D bandwidth from pinned host memory for a column-major matrix uploaded
// (a) in contiguous column panels, (b) in row panels (cudaMemcpy2DAsync,
// pitch = ld), (c) one contiguous copy.  Decides the streaming order of the
// single-pass host entry points.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 h2d_panels.cu -o h2d_panels
//   ./h2d_panels [rows] [cols] [panels]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

int main(int argc, char** argv) {
  const size_t m = argc > 1 ? atol(argv[1]) : 65536, n = argc > 2 ? atol(argv[2]) : 32768;
  const int np = argc > 3 ? atoi(argv[3]) : 24;
  const size_t bytes = m * n * 8;
  double *h, *d;
  if (cudaHostAlloc(&h, bytes, cudaHostAllocDefault) != cudaSuccess || cudaMalloc(&d, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  for (size_t i = 0; i < bytes / 8; i += 4096) h[i] = 1.0;
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](int mode) {
    cudaEventRecord(a, s);
    if (mode == 0) {
      cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
    } else if (mode == 1) {
      const size_t cp = (n + np - 1) / np;
      for (size_t c0 = 0; c0 < n; c0 += cp) {
        const size_t c1 = c0 + cp < n ? c0 + cp : n;
        cudaMemcpyAsync(d + c0 * m, h + c0 * m, (c1 - c0) * m * 8, cudaMemcpyHostToDevice, s);
      }
    } else {
      const size_t rp = (m + np - 1) / np;
      for (size_t r0 = 0; r0 < m; r0 += rp) {
        const size_t r1 = r0 + rp < m ? r0 + rp : m;
        cudaMemcpy2DAsync(d + r0, m * 8, h + r0, m * 8, (r1 - r0) * 8, n, cudaMemcpyHostToDevice, s);
      }
    }
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  };
  const char* names[3] = {"one contiguous copy", "column panels (contiguous)", "row panels (2D, pitch ld)"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      const float ms = run(mode);
      printf("%-28s %zu x %zu (%.1f GB), %d panels: %.1f ms = %.1f GB/s\n", names[mode], m, n, bytes / 1e9, np,
             ms, bytes / (ms * 1e6));
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
