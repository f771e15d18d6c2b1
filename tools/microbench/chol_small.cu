// Phase timing of cta_chol_inv (cholsmall.cuh) on one CTA, l = 25, a
// well-conditioned SPD Gram; prints cycles of the elimination and the output.
#define CHOL_STEP_PROBE
#include <cstdio>
#include <vector>
#include "../../paper_2402_17794_b200/csrc/cholsmall.cuh"

__global__ void run(const double* G, int l, long long* pr, double* out) {
  constexpr int LD = 33;
  __shared__ double G0[32 * LD], piv[rsvdb::kCholPivScratch], Rs[32 * LD], Ri[32 * LD];
  for (int e = threadIdx.x; e < 32 * LD; e += 256) G0[e] = 0.0;
  __syncthreads();
  for (int e = threadIdx.x; e < l * l; e += 256) G0[(e % l) + LD * (e / l)] = G[e];
  __syncthreads();
  bool sh;
  for (int rep = 0; rep < 4; ++rep) rsvdb::cta_chol_inv(G0, l, 1e-10, piv, Rs, Ri, &sh, pr + 64 * rep);
  for (int e = threadIdx.x; e < 32 * LD; e += 256) out[e] = Rs[e] + Ri[e];
}

int main() {
  const int l = 25;
  std::vector<double> g(l * l);
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < l; ++j) g[i + l * j] = (i == j ? l + 1.0 : 1.0 / (1 + i + j));
  double *dG, *dO; long long* dp;
  cudaMalloc(&dG, l * l * 8); cudaMalloc(&dO, 32 * 33 * 8); cudaMalloc(&dp, 256 * 8);
  cudaMemcpy(dG, g.data(), l * l * 8, cudaMemcpyHostToDevice);
  for (int k = 0; k < 2; ++k) {
    cudaMemset(dp, 0, 256 * 8);
    run<<<1, 256>>>(dG, l, dp, dO);
    long long h[256];
    cudaMemcpy(h, dp, sizeof h, cudaMemcpyDeviceToHost);
    for (int r = 0; r < 4; ++r) printf("[%lld %lld] ", h[64 * r + 1] - h[64 * r], h[64 * r + 2] - h[64 * r + 1]);
    // the probe stamps once per barrier (two pivots): print per barrier
    printf("\n per 2-pivot barrier:");
    for (int j = 0; j < l; j += 2) printf(" %lld", h[64 + 8 + j] - (j ? h[64 + 8 + j - 2] : h[64]));
    printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
