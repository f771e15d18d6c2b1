// tcgen05.mma kind::i8 on sm_100a: descriptor validation and issue-rate
// microbenchmark for the Ozaki-scheme FP64 pass (int8 slices, int32 TMEM
// accumulators).
//   check: one CTA, D[128 x N] = A[128 x K] * B[N x K]^T with TMA-loaded,
//          128B-swizzled operands; A either K-major (row-major int8) or
//          MN-major (column-major int8); compared with a CPU int32 product.
//   rate : 148 CTAs issue long chains of MMAs on resident smem operands
//          (no TMA traffic) for several N: cycles per MMA -> int8 MAC/clk/SM.
// Usage: ./umma_i8
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at line %d\n", cudaGetErrorString(e), __LINE__);             \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  long long t0 = clock64();
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par)
        : "memory");
    if (!ok && clock64() - t0 > (4LL << 30)) __trap();
  }
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 64-bit shared-memory matrix descriptor (sm_100 "version 1")
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout_type) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version
  d |= uint64_t(layout_type) << 61;
  return d;
}
// instruction descriptor for kind::i8, signed x signed -> s32
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_mn_major, int b_mn_major) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn_major) << 15) |
         (uint32_t(b_mn_major) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(dst)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t addr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols)
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(addr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- check
// AMN = 0: A global [128][K] (K contiguous); AMN = 1: A global [K][128] (M contiguous).
// B global [N][K] (K contiguous).  K multiple of 128.
template <int AMN>
__global__ void __launch_bounds__(128, 1)
    check_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int N, int K, int32_t* D) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024 - (su32(smraw) & 1023)) & 1023);
  uint8_t* sA = sm;              // 128 x 128 B = 16 KB
  uint8_t* sB = sm + 16384;      // N x 128 B (<= 32 KB)
  __shared__ uint64_t full, done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  const uint32_t idesc = idesc_i8(128, N, AMN, 0);
  uint32_t ph = 0;
  for (int kb = 0; kb < K / 128; ++kb) {
    if (threadIdx.x == 0) {
      expect_tx(&full, 16384 + N * 128);
      if (AMN == 0) tma_2d(sA, &tmA, &full, kb * 128, 0);   // {k, m}
      else          tma_2d(sA, &tmA, &full, 0, kb * 128);   // {m, k}
      tma_2d(sB, &tmB, &full, kb * 128, 0);
      mbar_wait(&full, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int k = 0; k < 4; ++k) {
        uint64_t ad, bd;
        if (AMN == 0) ad = smem_desc(su32(sA) + k * 32, 0, 1024, 2);
        else          ad = smem_desc(su32(sA) + k * 4096, 16384, 1024, 2);
        bd = smem_desc(su32(sB) + k * 32, 0, 1024, 2);
        umma_i8(tb, ad, bd, idesc, (kb | k) ? 1u : 0u);
      }
      umma_commit(&done);
      mbar_wait(&done, ph);   // operands are reused next iteration
    }
    ph ^= 1;
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    tmem_ld8(tb + (uint32_t(warp * 32) << 16) + c, v);
    for (int j = 0; j < 8; ++j) D[(size_t)threadIdx.x * N + c + j] = int32_t(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 256);
}

// ----------------------------------------------------------------- rate
// STAGES operand buffers rotate; A 16 KB (MN- or K-major), B N*128 B per stage.
template <int AMN>
__global__ void __launch_bounds__(128, 1) rate_kernel(int N, int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024 - (su32(smraw) & 1023)) & 1023);
  constexpr int STAGES = 4;
  __shared__ uint64_t done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < STAGES * 49152 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  const uint32_t idesc = idesc_i8(128, N, AMN, 0);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int st = it % STAGES;
      const uint32_t a0 = su32(sm) + st * 49152, b0 = a0 + 16384;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = AMN == 0 ? smem_desc(a0 + k * 32, 0, 1024, 2) : smem_desc(a0 + k * 4096, 16384, 1024, 2);
        uint64_t bd = smem_desc(b0 + k * 32, 0, 1024, 2);
        umma_i8(tb + (N <= 128 ? ((it * 4 + k) & 3) * 128 : (it & 1) * 256), ad, bd, idesc, 1u);
      }
    }
    umma_commit(&done);
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) cycles[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
}
static CUtensorMap map_u8(const void* p, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                          uint32_t box_in, uint32_t box_out) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_bytes};
  cuuint32_t box[2] = {box_in, box_out};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(p), dims, strides, box,
                     es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); exit(1); }
  return m;
}

template <int AMN>
static void run_check(int N, int K) {
  std::vector<int8_t> a(128 * (size_t)K), b((size_t)N * K);
  uint32_t s = 12345u + AMN;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return int8_t(int((s >> 24) % 129) - 64); };
  for (auto& x : a) x = rnd();
  for (auto& x : b) x = rnd();
  // a is logical A[i][k]; storage depends on AMN
  std::vector<int8_t> ag(a.size());
  for (int i = 0; i < 128; ++i)
    for (int k = 0; k < K; ++k) ag[AMN ? (size_t)k * 128 + i : (size_t)i * K + k] = a[(size_t)i * K + k];
  int8_t *dA, *dB; int32_t* dD;
  CK(cudaMalloc(&dA, ag.size())); CK(cudaMalloc(&dB, b.size())); CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dA, ag.data(), ag.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, b.data(), b.size(), cudaMemcpyHostToDevice));
  CUtensorMap tA = AMN ? map_u8(dA, 128, K, 128, 128, 128) : map_u8(dA, K, 128, K, 128, 128);
  CUtensorMap tB = map_u8(dB, K, N, K, 128, N);
  CK(cudaFuncSetAttribute(check_kernel<AMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768 + 1024));
  check_kernel<AMN><<<1, 128, 16384 + 32768 + 1024>>>(tA, tB, N, K, dD);
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> d(128 * (size_t)N);
  CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t r = 0;
      for (int k = 0; k < K; ++k) r += int32_t(a[(size_t)i * K + k]) * int32_t(b[(size_t)j * K + k]);
      if (r != d[(size_t)i * N + j]) { if (bad < 4) printf("  mismatch (%d,%d): got %d want %d\n", i, j, d[(size_t)i * N + j], r); ++bad; }
    }
  printf("check A %s-major N=%d K=%d: %ld mismatches of %d\n", AMN ? "MN" : "K", N, K, bad, 128 * N);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

static int g_iters = 2048;
template <int AMN>
static void run_rate(int sms) {
  long long* dc; CK(cudaMalloc(&dc, 8));
  CK(cudaFuncSetAttribute(rate_kernel<AMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 49152 + 1024));
  for (int N : {32, 48, 64, 96, 112, 128, 192, 256}) {
    const int iters = g_iters;
    rate_kernel<AMN><<<sms, 128, 4 * 49152 + 1024>>>(N, iters, dc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rate_kernel<AMN><<<sms, 128, 4 * 49152 + 1024>>>(N, iters, dc);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long cyc; CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    double per = double(cyc) / (iters * 4.0);
    double macs = 128.0 * N * 32;
    printf("rate A %s-major N=%3d: %7.1f cyc/MMA  %7.0f MAC/clk/SM  (%.1f%% of 8192)  chip %.0f TOPS (event %.3f ms)\n",
           AMN ? "MN" : "K", N, per, macs / per, 100.0 * macs / per / 8192.0,
           2.0 * macs * iters * 4.0 * sms / (ms * 1e-3) / 1e12, ms);
  }
  cudaFree(dc);
}

int main(int argc, char** argv) {
  if (argc > 1) g_iters = atoi(argv[1]);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_check<0>(64, 256);
  run_check<0>(256, 256);
  run_check<1>(64, 256);
  run_check<1>(256, 384);
  run_check<0>(48, 128);
  run_rate<0>(sms);
  run_rate<1>(sms);
  return 0;
}
