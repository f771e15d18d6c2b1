// Ablation of the per-step cost of the CTA elimination in cholsmall.cuh:
// which part of a step (pivot store, rsqrt, barrier, shuffle, row update)
// costs the ~800 cycles measured per step.
#include <cstdio>
#include <vector>
#include <cstdlib>

template <int V>
__global__ void run(const double* G, int l, long long* out_cyc, double* out, int reps) {
  constexpr int LD = 33;
  __shared__ double G0[32 * LD], piv[2 * 72];
  for (int e = threadIdx.x; e < 32 * LD; e += 256) G0[e] = 0.0;
  __syncthreads();
  for (int e = threadIdx.x; e < l * l; e += 256) G0[(e % l) + LD * (e / l)] = G[e];
  __syncthreads();
  const int t = threadIdx.x, i = t >> 3, c = t & 7, base = (t & 31) & ~7;
  const bool row = i < l;
  double w[8];
  double acc = 0.0;
  long long c0 = clock64();
#pragma unroll 1
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int p = 8 * c + q;
    double v = 0.0;
    if (row && p < l) v = G0[i + LD * p];
    if (row && p == 32 + i) v = 1.0;
    w[q] = v;
  }
  bool broke = false;
#pragma unroll 1
  for (int jb = 0; jb * 8 < l && !broke; ++jb) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = 8 * jb + jj;
      if (j < l && !broke) {
        double* pv = piv + (j & 1) * 72;
        if (i == j) {
#pragma unroll
          for (int q = 0; q < 8; ++q) pv[8 * c + q] = w[q];
          if (c == jb) {
            const double d = w[jj];
            if (V == 1) {
              pv[64] = 1.0 / d;
            } else {
              const double rs = rsqrt(d);
              pv[64] = rs * rs;
            }
            pv[65] = d;
          }
        }
        if (V == 2) __syncwarp(); else __syncthreads();
        const double d = pv[65];
        if (V != 3 && (!(d > 1e-12 * G0[j + LD * j]) || !(d > 0.0))) {
          broke = true;
        } else {
          const double wij = (V == 4) ? w[jj] : __shfl_sync(0xffffffffu, w[jj], base + jb);
          if (i > j && V != 5) {
            const double f = wij * pv[64];
#pragma unroll
            for (int q = 0; q < 8; ++q) w[q] = fma(-f, pv[8 * c + q], w[q]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) acc += w[q];
  acc += broke;
  }
  long long c1 = clock64();
  out[t] = acc;
  if (t == 0) out_cyc[V] = (c1 - c0) / reps;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 1;
  const int l = 25;
  std::vector<double> g(l * l);
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < l; ++j) g[i + l * j] = (i == j ? l + 1.0 : 1.0 / (1 + i + j));
  double *dG, *dO; long long* dp;
  cudaMalloc(&dG, l * l * 8); cudaMalloc(&dO, 256 * 8); cudaMalloc(&dp, 16 * 8);
  cudaMemcpy(dG, g.data(), l * l * 8, cudaMemcpyHostToDevice);
  const char* names[] = {"full", "div", "syncwarp", "nocheck", "noshfl", "noupdate"};
  for (int k = 0; k < 2; ++k) {
    run<0><<<1, 256>>>(dG, l, dp, dO, reps); run<1><<<1, 256>>>(dG, l, dp, dO, reps);
    run<2><<<1, 256>>>(dG, l, dp, dO, reps); run<3><<<1, 256>>>(dG, l, dp, dO, reps);
    run<4><<<1, 256>>>(dG, l, dp, dO, reps); run<5><<<1, 256>>>(dG, l, dp, dO, reps);
    long long h[16];
    cudaMemcpy(h, dp, sizeof h, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 6; ++v) printf("%s=%lld ", names[v], h[v]);
    printf(" err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
