// Streaming passes over A: the tall-skinny FP64 products of the rsvd hot path.
//
//   NN:  C (M x N) = P (M x K) * R (K x N)      Y = A X      (reference
//        rangefinder.hpp:63,73,76,87,91; singlepass.hpp:25,62,121)
//   TN:  C (M x N) = P^T * R, P (K x M)          Z = A^T Y,  B^T = A^T Q
//        (rangefinder.hpp:75,90; factor.hpp:14; singlepass.hpp:30,122) and
//        the l x l inner products Q^T Omega, Q^T Y (singlepass.hpp:65-66,127-128)
//
// B200 design:
//  * FP64 has no tcgen05 kind on sm_100a, so the math is warp-level DMMA
//    (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4), measured at 37.0 TFLOP/s.
//  * Operand tiles are staged by TMA (cp.async.bulk.tensor.2d, SASS UTMALDG)
//    with 128-byte swizzle into a STAGES-deep mbarrier ring; one producer warp
//    issues TMA, eight consumer warps run DMMA.  A is streamed with an
//    evict-first L2 policy, the small operand with evict-last.
//  * The swizzle + (for NN) a permuted K order inside each 8-wide K group make
//    every fragment load exactly 2 shared-memory wavefronts per 256 bytes.
//  * Long reductions are split over K (grid.z) to fill 148 SMs; partial tiles
//    are combined by the last-arriving CTA in FIXED split order, so results
//    are bitwise deterministic run to run (no floating-point atomics).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "pass.cuh"

namespace rsvdb {

// ------------------------------------------------------------ PTX helpers
namespace ptx {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > (20LL << 30)) __trap();
  }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
}  // namespace ptx

// ---------------------------------------------------------------- kernel
constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;

template <bool kNN, int BN, int WMT, int BK, int STAGES>
struct PassCfg {
  static constexpr int BM = kConsumerWarps * WMT * 8;
  static constexpr int NT = BN / 8;
  static constexpr int KH = BK / 16;  // 16-wide (128-byte) swizzle boxes along K
  static constexpr int A_BYTES = BM * BK * 8;
  static constexpr int B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int CPAD = 4;
  static constexpr int CS_BYTES = BN * (BM + CPAD) * 8;
  static constexpr int PIPE_BYTES = STAGES * STAGE_BYTES;
  static constexpr int SMEM = (PIPE_BYTES > CS_BYTES ? PIPE_BYTES : CS_BYTES) + 1024 /*align*/ +
                              2 * STAGES * 8 + 16;
  static_assert(BN % 8 == 0, "BN must be a multiple of 8");
  static_assert(BK % 16 == 0, "BK must be a multiple of 16");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle-128B alignment");
  static_assert(BM <= 256, "TMA box limit");
};

struct PassParams {
  int64_t M, N, K;
  int64_t k_per_split;  // multiple of BK
  int splits;
  double* C;
  int64_t ldc;
  double* partials;
  int* counters;
};

template <bool kNN, int BN, int WMT, int BK, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    pass_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                PassParams p) {
  using Cfg = PassCfg<kNN, BN, WMT, BK, STAGES>;
  constexpr int BM = Cfg::BM, NT = Cfg::NT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(
      smem + (Cfg::PIPE_BYTES > Cfg::CS_BYTES ? Cfg::PIPE_BYTES : Cfg::CS_BYTES));
  uint64_t* empty = full + STAGES;
  int* flag = reinterpret_cast<int*>(empty + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x, m_tile = blockIdx.y, split = blockIdx.z;
  const int64_t m0 = int64_t(m_tile) * BM, n0 = int64_t(n_tile) * BN;
  const int64_t k_begin = int64_t(split) * p.k_per_split;
  const int64_t k_end = min(p.K, k_begin + p.k_per_split);
  const int nkb = k_end > k_begin ? int((k_end - k_begin + BK - 1) / BK) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kConsumerWarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------ TMA producer warp
    if (lane == 0) {
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      const uint64_t pol_a = ptx::policy_evict_first();
      const uint64_t pol_b = ptx::policy_evict_last();
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) ptx::mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* a_st = smem + s * Cfg::STAGE_BYTES;
        uint8_t* b_st = a_st + Cfg::A_BYTES;
        ptx::mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        const int k0 = int(k_begin + int64_t(kb) * BK);
        if constexpr (kNN) {
          // A is M x K, M inner: boxes of 16 (M) x BK (K).
#pragma unroll
          for (int b = 0; b < BM / 16; ++b)
            ptx::tma_load_2d(a_st + b * (BK * 128), &tmA, &full[s], int(m0) + 16 * b, k0, pol_a);
        } else {
          // A is K x M, K inner: boxes of 16 (K) x BM (M).
#pragma unroll
          for (int h = 0; h < Cfg::KH; ++h)
            ptx::tma_load_2d(a_st + h * (BM * 128), &tmA, &full[s], k0 + 16 * h, int(m0), pol_a);
        }
#pragma unroll
        for (int h = 0; h < Cfg::KH; ++h)
          ptx::tma_load_2d(b_st + h * (BN * 128), &tmB, &full[s], k0 + 16 * h, int(n0), pol_b);
      }
    }
  } else {
    // ------------------------------------------------ DMMA consumer warps
    double acc[WMT][NT][2];
#pragma unroll
    for (int i = 0; i < WMT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int r8 = lane >> 2, c4 = lane & 3;
    const int wm0 = warp * WMT * 8;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      ptx::mbar_wait(&full[s], (kb / STAGES) & 1);
      const uint8_t* a_st = smem + s * Cfg::STAGE_BYTES;
      const uint8_t* b_st = a_st + Cfg::A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        double af[WMT], bf[NT];
        int kr;  // K row (0..BK-1) this lane contributes in k-step ks
        if constexpr (kNN) {
          // Permuted K order {0,4,1,5},{2,6,3,7} per 8-group: conflict-free with
          // the M-inner swizzled A tile.
          const int base = (ks >> 1) * 8;
          const int off = (ks & 1) ? ((c4 & 1) ? 6 : 2) + ((c4 >> 1) ? 1 : 0)
                                   : ((c4 & 1) ? 4 : 0) + ((c4 >> 1) ? 1 : 0);
          kr = base + off;
#pragma unroll
          for (int i = 0; i < WMT; ++i) {
            const int m = wm0 + i * 8 + r8;
            const int mm = m & 15;
            const uint8_t* ptr = a_st + (m >> 4) * (BK * 128) + kr * 128 +
                                 ((((mm >> 1)) ^ (kr & 7)) << 4) + ((mm & 1) << 3);
            af[i] = *reinterpret_cast<const double*>(ptr);
          }
        } else {
          kr = ks * 4 + c4;
          const int h = kr >> 4, kk = kr & 15;
#pragma unroll
          for (int i = 0; i < WMT; ++i) {
            const int m = wm0 + i * 8 + r8;
            const uint8_t* ptr = a_st + h * (BM * 128) + m * 128 + (((kk >> 1) ^ (m & 7)) << 4) +
                                 ((kk & 1) << 3);
            af[i] = *reinterpret_cast<const double*>(ptr);
          }
        }
        {
          const int h = kr >> 4, kk = kr & 15;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int n = j * 8 + r8;
            const uint8_t* ptr = b_st + h * (BN * 128) + n * 128 + (((kk >> 1) ^ (n & 7)) << 4) +
                                 ((kk & 1) << 3);
            bf[j] = *reinterpret_cast<const double*>(ptr);
          }
        }
#pragma unroll
        for (int i = 0; i < WMT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) ptx::dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }

    // ------------------------------------------------ epilogue
    ptx::named_bar(1, kConsumerWarps * 32);  // all consumers done reading stages
    double* cs = reinterpret_cast<double*>(smem);
    constexpr int LDC = BM + Cfg::CPAD;
#pragma unroll
    for (int i = 0; i < WMT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int m = wm0 + i * 8 + r8;
        const int n = j * 8 + 2 * c4;
        cs[n * LDC + m] = acc[i][j][0];
        cs[(n + 1) * LDC + m] = acc[i][j][1];
      }
    ptx::named_bar(1, kConsumerWarps * 32);

    const int tid = threadIdx.x;
    constexpr int NCT = kConsumerWarps * 32;
    const int mlim = int(p.M - m0 < BM ? p.M - m0 : BM);
    const int nlim = int(p.N - n0 < BN ? p.N - n0 : BN);
    if (p.splits == 1) {
      for (int n = 0; n < nlim; ++n)
        for (int m = tid; m < mlim; m += NCT) p.C[(n0 + n) * p.ldc + m0 + m] = cs[n * LDC + m];
    } else {
      const int64_t tile = int64_t(m_tile) * gridDim.x + n_tile;
      double* part = p.partials + (tile * p.splits) * (BM * BN);
      double* mine = part + int64_t(split) * (BM * BN);
      for (int e = tid; e < BM * BN; e += NCT) mine[e] = cs[(e / BM) * LDC + (e % BM)];
      __threadfence();
      ptx::named_bar(1, NCT);
      if (tid == 0) {
        const int old = atomicAdd(&p.counters[tile], 1);
        *flag = (old == p.splits - 1);
      }
      ptx::named_bar(1, NCT);
      if (*flag) {
        __threadfence();
        for (int n = 0; n < nlim; ++n)
          for (int m = tid; m < mlim; m += NCT) {
            double v = 0.0;
            for (int z = 0; z < p.splits; ++z) v += __ldcg(part + int64_t(z) * (BM * BN) + n * BM + m);
            p.C[(n0 + n) * p.ldc + m0 + m] = v;
          }
        if (tid == 0) p.counters[tile] = 0;  // self-reset for the next launch
      }
    }
  }
}

// ------------------------------------------------------------- host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) throw Error(RSVD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D column-major fp64 tensor map: dims {inner=rows, outer=cols}.
CUtensorMap make_map(const double* p, int64_t rows, int64_t cols, int64_t ld, int box_inner,
                     int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cuuint64_t(std::max<int64_t>(rows, 1)), cuuint64_t(std::max<int64_t>(cols, 1))};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
  cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(RSVD_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

bool tma_ok(const DMat& x) {
  return (reinterpret_cast<uintptr_t>(x.p) % 16 == 0) && (x.ld % 2 == 0) && x.ld >= x.rows;
}

template <bool kNN, int BN, int WMT, int BK, int STAGES>
void launch(Handle& h, const DMat& P, const DMat& R, DMat C, int64_t M, int64_t N, int64_t K,
            int force_splits) {
  using Cfg = PassCfg<kNN, BN, WMT, BK, STAGES>;
  static bool attr_set = false;
  auto kern = pass_kernel<kNN, BN, WMT, BK, STAGES>;
  if (!attr_set) {
    RSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr_set = true;
  }
  const int64_t mt = ceil_div(M, Cfg::BM), nt = ceil_div(N, BN);
  const int64_t tiles = mt * nt;
  const int64_t kblocks = ceil_div(K, BK);
  // Split K so that the grid fills whole waves of the 148 SMs (1 CTA/SM).
  int splits = 1;
  if (force_splits > 0) {
    splits = force_splits;
  } else {
    const int sms = h.sm_count;
    double best = 1e300;
    const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(kblocks / 4, 64));
    for (int64_t s = 1; s <= smax; ++s) {
      const int64_t ctas = tiles * s;
      const int64_t waves = ceil_div(ctas, sms);
      const double t = double(waves) * double(ceil_div(kblocks, s) + 6) + 0.5 * double(s);
      if (t < best) {
        best = t;
        splits = int(s);
      }
    }
  }
  const int64_t kps = round_up(ceil_div(K, splits), BK);
  splits = int(ceil_div(K, kps));
  if (splits < 1) splits = 1;
  PassParams pp{M, N, K, kps, splits, C.p, C.ld, nullptr, nullptr};
  if (splits > 1) {
    pp.partials = h.ws.alloc(tiles * splits * Cfg::BM * BN);
    pp.counters = tile_counters(h, tiles);
  }
  CUtensorMap ta = kNN ? make_map(P.p, P.rows, P.cols, P.ld, 16, BK)
                       : make_map(P.p, P.rows, P.cols, P.ld, 16, Cfg::BM);
  CUtensorMap tb = make_map(R.p, R.rows, R.cols, R.ld, 16, BN);
  const dim3 grid{unsigned(nt), unsigned(mt), unsigned(splits)};
  kern<<<grid, kThreads, Cfg::SMEM, h.stream>>>(ta, tb, pp);
  RSVD_LAUNCHED(h);
}

// Copy into an aligned, even-ld workspace when TMA cannot address x directly.
DMat tma_view(Handle& h, const DMat& x) {
  if (tma_ok(x)) return x;
  DMat y = h.ws.mat(x.rows, x.cols);
  RSVD_CUDA(cudaMemcpy2DAsync(y.p, y.ld * 8, x.p, x.ld * 8, x.rows * 8, x.cols,
                              cudaMemcpyDeviceToDevice, h.stream));
  return y;
}

}  // namespace

void gemm_nn(Handle& h, const DMat& P, const DMat& R, DMat C, int force_splits) {
  const int64_t M = P.rows, K = P.cols, N = R.cols;
  if (R.rows != K || C.rows != M || C.cols != N) throw_dim("gemm_nn: shape mismatch");
  if (M == 0 || N == 0) return;
  if (K == 0) {
    RSVD_CUDA(cudaMemset2DAsync(C.p, C.ld * 8, 0, M * 8, N, h.stream));
    return;
  }
  DMat Pv = tma_view(h, P), Rv = tma_view(h, R);
  if (N <= 32)
    launch<true, 32, 2, 32, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (N <= 64)
    launch<true, 64, 2, 32, 3>(h, Pv, Rv, C, M, N, K, force_splits);
  else
    launch<true, 56, 4, 16, 4>(h, Pv, Rv, C, M, N, K, force_splits);
}

void gemm_tn(Handle& h, const DMat& P, const DMat& R, DMat C, int force_splits) {
  const int64_t K = P.rows, M = P.cols, N = R.cols;
  if (R.rows != K || C.rows != M || C.cols != N) throw_dim("gemm_tn: shape mismatch");
  if (M == 0 || N == 0) return;
  if (K == 0) {
    RSVD_CUDA(cudaMemset2DAsync(C.p, C.ld * 8, 0, M * 8, N, h.stream));
    return;
  }
  DMat Pv = tma_view(h, P), Rv = tma_view(h, R);
  if (N <= 32)
    launch<false, 32, 2, 32, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (N <= 64)
    launch<false, 64, 2, 32, 3>(h, Pv, Rv, C, M, N, K, force_splits);
  else
    launch<false, 56, 4, 16, 4>(h, Pv, Rv, C, M, N, K, force_splits);
}

}  // namespace rsvdb
