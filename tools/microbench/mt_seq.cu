// Sequential MT19937-64 block generation latency: one 320-thread CTA with a
// barrier per block (rng.cu mt_blocks_kernel) vs a single warp (__syncwarp).
#include <cstdint>
#include <cstdio>
#include <vector>
#include <random>

constexpr uint64_t kMatA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x000000007FFFFFFFULL;
constexpr int kN = 312, kM = 156;

__device__ __forceinline__ uint64_t twist(uint64_t xk, uint64_t xk1) {
  const uint64_t y = (xk & kUpper) | (xk1 & kLower);
  return (y >> 1) ^ ((y & 1ULL) ? kMatA : 0ULL);
}
__device__ __forceinline__ uint64_t next_word(const uint64_t* c, int t) {
  if (t < kN - kM) return c[t + kM] ^ twist(c[t], c[t + 1]);
  if (t < kN - 1) return c[t] ^ twist(c[t - kM], c[t - kM + 1]) ^ twist(c[t], c[t + 1]);
  const uint64_t n0 = c[kM] ^ twist(c[0], c[1]);
  return c[kN - 1] ^ twist(c[kM - 1], c[kM]) ^ twist(c[kN - 1], n0);
}

__global__ void cta_blocks(const uint64_t* init, int64_t nb, uint64_t* out) {
  __shared__ uint64_t S[2][kN];
  const int t = threadIdx.x;
  if (t < kN) { S[0][t] = init[t]; out[t] = init[t]; }
  __syncthreads();
  for (int64_t k = 1; k <= nb; ++k) {
    const uint64_t* c = S[(k - 1) & 1];
    uint64_t* n = S[k & 1];
    if (t < kN) { const uint64_t v = next_word(c, t); n[t] = v; out[k * kN + t] = v; }
    __syncthreads();
  }
}

__global__ void warp_blocks(const uint64_t* init, int64_t nb, uint64_t* out) {
  __shared__ uint64_t S[2][kN];
  const int t = threadIdx.x;
  for (int j = t; j < kN; j += 32) { S[0][j] = init[j]; out[j] = init[j]; }
  __syncwarp();
  for (int64_t k = 1; k <= nb; ++k) {
    const uint64_t* c = S[(k - 1) & 1];
    uint64_t* n = S[k & 1];
    uint64_t v[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const int j = t + 32 * i;
      v[i] = (j < kN) ? next_word(c, j) : 0;
    }
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const int j = t + 32 * i;
      if (j < kN) { n[j] = v[i]; out[k * kN + j] = v[i]; }
    }
    __syncwarp();
  }
}

int main() {
  const int64_t nb = 835;
  std::mt19937_64 g(7);
  std::vector<uint64_t> init(kN);
  // raw initial state of mt19937_64(7): replicate seeding
  init[0] = 7;
  for (int i = 1; i < kN; ++i) init[i] = 6364136223846793005ULL * (init[i - 1] ^ (init[i - 1] >> 62)) + i;
  uint64_t *di, *d1, *d2;
  cudaMalloc(&di, kN * 8); cudaMalloc(&d1, (nb + 1) * kN * 8); cudaMalloc(&d2, (nb + 1) * kN * 8);
  cudaMemcpy(di, init.data(), kN * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e[4]; for (auto& x : e) cudaEventCreate(&x);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e[0]); cta_blocks<<<1, 320>>>(di, nb, d1); cudaEventRecord(e[1]);
    warp_blocks<<<1, 32>>>(di, nb, d2); cudaEventRecord(e[2]); cudaEventSynchronize(e[2]);
    float a, b; cudaEventElapsedTime(&a, e[0], e[1]); cudaEventElapsedTime(&b, e[1], e[2]);
    std::vector<uint64_t> h1((nb + 1) * kN), h2((nb + 1) * kN);
    cudaMemcpy(h1.data(), d1, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), d2, h2.size() * 8, cudaMemcpyDeviceToHost);
    printf("cta %.1f us (%.0f ns/block)  warp %.1f us (%.0f ns/block)  same=%d\n", a * 1e3, a * 1e6 / nb, b * 1e3,
           b * 1e6 / nb, int(h1 == h2));
  }
  return 0;
}
