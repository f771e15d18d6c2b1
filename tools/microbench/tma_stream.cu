// Streaming-read rate of the pass kernel's load path, without the math:
// 148 persistent CTAs stream a column-major 8192 x 8192 fp64 matrix (537 MB)
// through a STAGES-deep mbarrier ring, one producer thread, consumers only
// wait and release.  Variants:
//   tma2d : cp.async.bulk.tensor.2d boxes {16 rows, BK cols}, SWIZZLE_128B,
//           BM/16 boxes per stage (the pass kernel's NN A load)
//   bulk1d: cp.async.bulk (1-D) of one BM-row column chunk (BM * 8 bytes) per
//           column, BK per stage
// Usage: ./tma_stream
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ uint64_t evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int MODE, int BM, int BK, int STAGES>
__global__ void __launch_bounds__(288, 1) stream_kernel(const __grid_constant__ CUtensorMap tm,
                                                        const double* __restrict__ A, int64_t M,
                                                        int64_t K, int64_t* sink) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024 - (su32(smraw) & 1023)) & 1023);
  constexpr int COLB = MODE == 0 ? BM * 8 : BM * 8 + 32;  // bulk1d: padded column stride
  constexpr int STAGE = MODE == 0 ? BM * BK * 8 : COLB * BK;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t mt = M / BM, kt = K / BK, units = mt * kt;
  const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = evict_first();
      for (int64_t u = u0; u < u1; ++u) {
        const int i = int(u - u0), s = i % STAGES;
        if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
        uint8_t* dst = sm + s * STAGE;
        expect_tx(&full[s], BM * BK * 8);
        const int m0 = int(u / kt) * BM, k0 = int(u % kt) * BK;
        if constexpr (MODE == 0) {
#pragma unroll
          for (int b = 0; b < BM / 16; ++b)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(dst + b * (BK * 128))),
                "l"(&tm), "r"(su32(&full[s])), "r"(m0 + 16 * b), "r"(k0), "l"(pol)
                : "memory");
        } else {
          for (int c = 0; c < BK; ++c)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1], %2, [%3], %4;" ::"r"(su32(dst + c * COLB)),
                "l"(A + int64_t(k0 + c) * M + m0), "r"(BM * 8), "r"(su32(&full[s])), "l"(pol)
                : "memory");
        }
      }
    }
    return;
  }
  int64_t acc = 0;
  for (int64_t u = u0; u < u1; ++u) {
    const int i = int(u - u0), s = i % STAGES;
    wait(&full[s], (i / STAGES) & 1);
    acc += reinterpret_cast<const int64_t*>(sm + s * STAGE)[threadIdx.x];
    __syncwarp();
    if (lane == 0) arrive(&empty[s]);
  }
  if (acc == 42) sink[0] = acc;
}

template <int MODE, int BM, int BK, int STAGES>
void run(const double* A, int64_t M, int64_t K, int64_t* sink, const CUtensorMap& tm) {
  constexpr int COLB = MODE == 0 ? BM * 8 : BM * 8 + 32;
  constexpr int STAGE = MODE == 0 ? BM * BK * 8 : COLB * BK;
  const int smem = STAGES * STAGE + 1024 + 2 * STAGES * 8;
  auto k = stream_kernel<MODE, BM, BK, STAGES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    k<<<148, 288, smem>>>(tm, A, M, K, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = ms < best ? ms : best;
  }
  const cudaError_t err = cudaGetLastError();
  std::printf("%-6s BM %3d BK %2d stages %d: %8.1f us  %6.0f GB/s %s\n", MODE == 0 ? "tma2d" : "bulk1d",
              BM, BK, STAGES, best * 1e3, double(M) * K * 8 / (best * 1e-3) / 1e9,
              err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  const int64_t M = 8192, K = 8192;
  double* A;
  int64_t* sink;
  cudaMalloc(&A, M * K * 8);
  cudaMalloc(&sink, 64);
  cudaMemset(A, 0, M * K * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  auto map = [&](int box_k) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(M), cuuint64_t(K)};
    cuuint64_t strides[1] = {cuuint64_t(M) * 8};
    cuuint32_t box[2] = {16, cuuint32_t(box_k)};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
  };
  const CUtensorMap m48 = map(48), m32 = map(32);
  run<0, 128, 48, 3>(A, M, K, sink, m48);
  run<0, 128, 32, 4>(A, M, K, sink, m32);
  run<1, 128, 48, 3>(A, M, K, sink, m48);
  run<1, 128, 32, 4>(A, M, K, sink, m32);
  run<1, 256, 32, 3>(A, M, K, sink, m32);
  run<1, 256, 16, 6>(A, M, K, sink, m32);
  run<1, 512, 16, 3>(A, M, K, sink, m32);
  return 0;
}
