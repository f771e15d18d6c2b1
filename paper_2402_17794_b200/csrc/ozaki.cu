// FP64 streaming-pass products on the INT8 tensor cores (tcgen05.mma
// kind::i8, int32 accumulators in TMEM) by the Ozaki splitting.
//
// FP64 has no tcgen05 kind on sm_100a, so the DMMA passes (pass.cu, fused.cu)
// top out at the 37 TFLOP/s FP64 pipe.  The products of the range finder are
// C = A X with A huge and X skinny (reference rangefinder.hpp:70-79,
// singlepass.hpp:119-122); here each operand is written as
//     a_ik = 2^eA[i] * sum_{s=1..S} d_s(i,k) 2^(2-8s),   |d_s| <= 128
// (d_s: balanced base-256 digits -- int8 -- of the value rounded ONCE to 8S-2
// fractional bits below its row's largest power of two, the leading digit in
// [-64, 64]; X likewise per column), so
//     C_ij = 2^(eA[i]+eX[j]) * sum_{c=2..S+1} 2^(4-8c) * P_c(i,j),
//     P_c  = sum_{s+t=c} D^A_s D^X_t          (exact int32 GEMMs)
// The dropped terms (s+t > S+1) are below 2^(-8S+6) relative to the row /
// column maxima: S = 7 (54 fractional bits, 28 slice products) is at fp64's
// own rounding of the product, S = 6 is 2^-46.  int32 holds a diagonal's sum
// of up to 7 products of |d| <= 128 over 16384 contraction steps (max_k);
// longer contractions are accumulated in chunks.
//
// Pipeline per row panel of A (<= 32768 rows):
//   row_exp -> slice (A read twice from HBM as fp64, slices written once per
//   operand layout) -> apply GEMM (Y rows of the panel) -> Psi' = 2^eA Psi
//   sliced per column -> adjoint GEMM (W += A_panel^T Psi_panel) from the SAME
//   slices of A (MN-major UMMA operand for the apply, K-major for the adjoint).
// The range finder's 2q+2 products of one call share one slicing of A
// (OzCache).
//
// GEMM kernels: warp 0 = TMA producer, warp 1 = MMA issuer + TMEM owner,
// warps 2-5 = epilogue (TMEM -> fp64).  An mbarrier ring of K = 32 steps; each
// step holds every needed slice tile of both operands; the diagonals c are
// accumulated four at a time (4 x 128 TMEM columns), high c first.
//   ozaki_gemm2_kernel: a CTA pair per 256 x {64,96,128} output tile, one
//                       tcgen05.mma.cta_group::2 per slice product (default)
//   ozaki_gemm_kernel : one CTA per 128 x ntile tile (RSVD_OZ_CG2=0)
// DESIGN.md section 3c has the measurements behind each choice.
#include "ozaki.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "pass.cuh"
#include "ptx.cuh"
#include "small.cuh"

namespace rsvdb {

namespace {

constexpr int kBM = 128;           // output rows per CTA (UMMA M)
constexpr int kKS = 32;            // contraction per ring stage = one int8 UMMA K step
constexpr int kStages = 3;
constexpr int kThreads = 192;      // producer warp, MMA warp, 4 epilogue warps
constexpr int kATile = kBM * kKS;  // bytes of one A slice tile
constexpr int kARegion = 8 * kATile;  // A part of a stage (8 slice tiles / 2 quad tiles)
constexpr int kMaxS = 8;
constexpr int kAutoSlices = 7;     // 54 fractional bits: at fp64's own rounding of the product
constexpr int kMaxRows = 32768;    // rows of A sliced at a time (workspace)
// contraction steps one int32 accumulation may cover: (S - 1 or S) products of
// |d| <= 128 per diagonal and step, (S) * K * 2^14 < 2^31
__host__ __device__ constexpr int max_k(int S) { return S >= 8 ? 8192 : 16384; }
// Diagonal groups (four int32 accumulators fit in TMEM beside each other):
// S <= 4: one sweep over c = 2..S+1.  S > 4: sweep 0 takes the high diagonals
// c = 6..S+1 (every slice), sweep 1 the low ones c = 2..5 (slices 1..4 only:
// one quad tile per operand) -- 18 + 10 MMAs per K step for S = 7, both sweeps
// bound by the tensor pipe rather than by their loads.
__host__ __device__ constexpr int grp_c_lo(int S, int g) { return (S > 4 && g == 0) ? 6 : 2; }
__host__ __device__ constexpr int grp_c_hi(int S, int g) { return (S > 4 && g == 1) ? 5 : S + 1; }
__host__ __device__ constexpr int grp_slices(int S, int g) { return (S > 4 && g == 1) ? 4 : S; }

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(map), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(map), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// sm_100 shared-memory matrix descriptor: start address, leading / stride byte
// offsets (all >> 4), version 1, swizzle mode in bits 61-63 (2 = 128 B, 6 = 32 B)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
}
// kind::i8 instruction descriptor: s8 x s8 -> s32, M = 128
__device__ __forceinline__ uint32_t idesc_i8(int n, int a_mn_major) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn_major) << 15) |
         (uint32_t(n >> 3) << 17) | (uint32_t(kBM >> 4) << 24);
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
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          ptx::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// 2^j as a double, j in [-1022, 1023]
__host__ __device__ __forceinline__ double exp2i(int j) {
  const unsigned long long b = (unsigned long long)(j + 1023) << 52;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  std::memcpy(&d, &b, 8);
  return d;
#endif
}
// x * 2^k for |k| up to ~2040 without an overflowing scale factor
__device__ __forceinline__ double scale2(double x, int k) {
  k = max(-2044, min(2046, k));  // beyond this the product under/overflows anyway
  const int k1 = k >> 1;
  return x * exp2i(k1) * exp2i(k - k1);
}

// ----------------------------------------------------------- exponents
__global__ void fill_int_kernel(int* p, int n, int v) {
  RSVD_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
// e[r] = max_c bexp(x[r,c]) - 1022 over this block's column range (|x| < 2^e)
__global__ void __launch_bounds__(256)
    row_exp_kernel(const double* __restrict__ x, int64_t ld, int rows, int64_t cols, int cpb,
                   int* __restrict__ e, int* __restrict__ flags) {
  RSVD_PDL_ENTRY();
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r >= rows) return;
  const int64_t c0 = int64_t(blockIdx.y) * cpb, c1 = min(cols, c0 + cpb);
  const double* p = x + r;
  int mx = 0;
  int64_t c = c0;
  for (; c + 8 <= c1; c += 8) {
    int h[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) h[u] = __double2hiint(__ldg(p + (c + u) * ld));
#pragma unroll
    for (int u = 0; u < 8; ++u) mx = max(mx, h[u] & 0x7ff00000);
  }
  for (; c < c1; ++c) mx = max(mx, __double2hiint(__ldg(p + c * ld)) & 0x7ff00000);
  // Inf / NaN cannot be sliced: the call ends in NumericError, as when a
  // non-finite entry reaches the FP64 pass's outputs
  if (mx == 0x7ff00000) atomicOr(flags, kFlagNonFinite);
  atomicMax(&e[r], (mx >> 20) - 1022);
}
// e[c] = max_r (bexp(x[r,c]) - 1022 + radd[r]) over this block's row range
__global__ void __launch_bounds__(256)
    col_exp_kernel(const double* __restrict__ x, int64_t ld, int rows, int rpb,
                   const int* __restrict__ radd, int* __restrict__ e, int* __restrict__ flags) {
  RSVD_PDL_ENTRY();
  const int c = blockIdx.x;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  const double* p = x + int64_t(c) * ld;
  int mx = INT_MIN;
  for (int r = r0 + threadIdx.x; r < r1; r += 256) {
    const int b = ((__double2hiint(__ldg(p + r)) & 0x7ff00000) >> 20) - 1022;
    if (b == 2047 - 1022) atomicOr(flags, kFlagNonFinite);
    mx = max(mx, b + (radd ? radd[r] : 0));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx != INT_MIN) atomicMax(&e[c], mx);
}

// -------------------------------------------------------------- slicing
// Digit s of q = rint(x[r,c] * 2^(P - rsub[r] + radd[r] - csub[c])), P = 8S-2:
// q = sum_s d_s 256^(S-s), d_s in [-128, 127] (top digit in [-64, 64]).
// Two output layouts (either or both):
//   plain      out[s][c][r]            r contiguous, ld8 bytes per column: the
//              MN-major UMMA operand of a contraction over c (the apply);
//   interleave outi[c][r/32][s][r%32]  ldi bytes per column, 8 slice slots of
//              32 bytes per 32 r: a contraction over r reads it K-major, and a
//              128-byte swizzled TMA box holds FOUR slices of one K = 32 step
//              (the UMMA descriptor picks a slice by a 32-byte start offset),
//              so the K-major operands get the conflict-free 128B swizzle.
// One thread: 4 consecutive r of one column (one 32-bit word per slice).
template <int S>
__global__ void __launch_bounds__(256)
    slice_kernel(const double* __restrict__ x, int64_t ld, int rows, int cols,
                 const int* __restrict__ rsub, const int* __restrict__ radd,
                 const int* __restrict__ csub, uint8_t* __restrict__ out, int64_t ld8,
                 uint8_t* __restrict__ outi, int64_t ldi) {
  RSVD_PDL_ENTRY();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (blockIdx.y * 32 + lane) * 4;  // rows on grid.y (<= 8.3 M), columns on grid.x
  const int c = blockIdx.x * 8 + warp;
  // the interleaved layout is read in whole 32-r groups: zero-fill the last one
  const int rows_w = outi ? ((rows + 31) & ~31) : rows;
  if (r0 >= rows_w || c >= cols) return;
  const double* p = x + int64_t(c) * ld + r0;
  double v[4];
  if (r0 + 3 < rows && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
    const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = r0 + u < rows ? p[u] : 0.0;
  }
  const int kc = 8 * S - 2 - (csub ? csub[c] : 0);
  // Balanced digits without carries: with B = sum_{j < S-1} 128 * 256^j added,
  // the base-256 digits of q + B are d_j + 128 in [0, 255] -- the BYTES of
  // q + B -- and the top one d_top in [-64, 64] is unbiased.  The four rows'
  // bytes of a slice are packed into a word and the bias comes off all four
  // with one XOR (b - 128 = b ^ 0x80 mod 256).
  constexpr long long kBias = [] {
    long long b = 0;
    for (int j = 0; j < S - 1; ++j) b += 128LL << (8 * j);
    return b;
  }();
  uint32_t w[S];
#pragma unroll
  for (int s = 0; s < S; ++s) w[s] = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int k = kc;
    if (r0 + u < rows) {
      if (rsub) k -= rsub[r0 + u];
      if (radd) k += radd[r0 + u];
    }
    const long long qb = __double2ll_rn(scale2(v[u], k)) + kBias;
    const uint32_t lo = uint32_t(qb), hi = uint32_t(uint64_t(qb) >> 32);
#pragma unroll
    for (int j = 0; j < S - 1; ++j) {  // byte j (weight 256^j) belongs to slice S - j
      const uint32_t f = j < 4 ? (lo >> (8 * j)) : (hi >> (8 * (j - 4)));
      w[S - 1 - j] |= (f & 255u) << (8 * u);
    }
    const int top = int(qb >> (8 * (S - 1)));  // arithmetic shift: in [-64, 64]
    w[0] |= (uint32_t(top) & 0xffu) << (8 * u);
  }
#pragma unroll
  for (int s = 1; s < S; ++s) w[s] ^= 0x80808080u;
  if (out && r0 < rows) {
    const int64_t plane = int64_t(cols) * ld8;
    uint8_t* o = out + int64_t(c) * ld8 + r0;
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(o + s * plane) = w[s];
  }
  if (outi) {
    uint8_t* o = outi + int64_t(c) * ldi + int64_t(r0 >> 5) * 256 + (r0 & 31);
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(o + s * 32) = w[s];
  }
}

// ----------------------------------------------------------------- GEMM
struct OzParams {
  int M, N, K;      // output M x N; contraction over K entries starting at k0
  int k0;
  int S;
  int ntile, n_tiles;
  double* C;
  int64_t ldc;
  const int* rexp;  // exponent per output row / column (nullptr = 0)
  const int* cexp;
  int accumulate;   // C += result
  double* scratch;  // per-CTA 128 x ntile partial (S > 4)
  int dbg;          // RSVD_OZ_DBG: 1 = no MMAs (load path alone), 2 = loads only for the first ring fill
};

// AMN = 1: A tiles are MN-major (global [k][m], the apply product of a
// column-major A); AMN = 0: K-major (global [m][k], the adjoint product).
template <int AMN, int S>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, OzParams p) {
  RSVD_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
  __shared__ uint64_t bar_full[kStages], bar_empty[kStages], bar_acc_full, bar_acc_empty;
  __shared__ uint32_t tmem_base_sh;
  const int btile4 = p.ntile * 128;                 // four B slices of one K step
  const int stage_bytes = kARegion + 2 * btile4;    // multiple of 1024 (ntile % 16 == 0)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x / p.n_tiles, nt = blockIdx.x % p.n_tiles;
  const int m0 = mt * kBM, n0 = nt * p.ntile;
  const int nk = (p.K + kKS - 1) / kKS;
  const int ngroups = (S + 3) / 4;
  constexpr int kchunk = max_k(S) / kKS;  // K steps one int32 accumulation may cover
  const int nchunks = (nk + kchunk - 1) / kchunk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&bar_full[s], 1);
      ptx::mbar_init(&bar_empty[s], 1);
    }
    ptx::mbar_init(&bar_acc_full, 1);
    ptx::mbar_init(&bar_acc_empty, 128);
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     ptx::smem_u32(&tmem_base_sh)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      int it = 0;
      for (int g = 0; g < ngroups; ++g) {
        const int Sg = grp_slices(S, g);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          ptx::mbar_wait(&bar_empty[st], ph ^ 1);
          if ((p.dbg & 2) && it >= kStages) {
            ptx::mbar_arrive(&bar_full[st]);
            continue;
          }
          const int nhalf = (Sg + 3) >> 2;
          ptx::mbar_expect_tx(&bar_full[st],
                              uint32_t(AMN ? Sg * kATile : nhalf * 4 * kATile) + uint32_t(nhalf * btile4));
          uint8_t* base = sm + st * stage_bytes;
          const int kc = p.k0 + kb * kKS;   // contraction index
          const int ki = (kc >> 5) * 256;   // byte offset of its 32-group in an interleaved operand
          if (AMN) {
            for (int s = 0; s < Sg; ++s) tma_load_3d(base + s * kATile, &tmA, &bar_full[st], m0, kc, s);
          } else {
            for (int hf = 0; hf < nhalf; ++hf)
              tma_load_2d(base + hf * 4 * kATile, &tmA, &bar_full[st], ki + hf * 128, m0);
          }
          uint8_t* bb = base + kARegion;
          for (int hf = 0; hf < nhalf; ++hf)
            tma_load_2d(bb + hf * btile4, &tmB, &bar_full[st], ki + hf * 128, n0);
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    // The whole warp runs the loop (warp-uniform control flow and operands, so
    // descriptors stay in uniform registers) and one elected lane issues; the
    // schedule of a K step is unrolled at compile time (S is a template
    // parameter).  With a divergent `if (lane == 0)` around the loop the
    // compiler wrapped every tcgen05.mma in an elect loop with four R2UR moves:
    // 128 cycles per MMA, twice the tensor pipe's 60.
    const uint32_t idesc = idesc_i8(p.ntile, AMN);
    const uint64_t ad_fixed = smem_desc(0, AMN ? 4096 : 0, 1024, 2);
    const uint64_t bd_fixed = smem_desc(0, 0, 1024, 2);
    const uint32_t sm0 = ptx::smem_u32(sm);
    int it = 0, drains = 0;
    auto run_group = [&](auto sg_tag) {
      constexpr int G = decltype(sg_tag)::value;
      constexpr int Sg = grp_slices(S, G), c_hi = grp_c_hi(S, G), c_lo = grp_c_lo(S, G);
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int st = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        const bool chunk_start = kb % kchunk == 0;
        if (chunk_start && drains > 0) {  // the epilogue has drained the previous accumulation
          ptx::mbar_wait(&bar_acc_empty, uint32_t(drains - 1) & 1);
          tc_fence_after();
        }
        ptx::mbar_wait(&bar_full[st], ph);
        tc_fence_after();
        const uint32_t a0 = (sm0 + st * stage_bytes) >> 4;
        const uint32_t b0 = a0 + (kARegion >> 4);
        const uint32_t kacc = chunk_start ? 0u : 1u;
        if (elect_one() && !(p.dbg & 1)) {
#pragma unroll
          for (int c = c_hi; c >= c_lo; --c) {
            constexpr int dummy = 0;
            (void)dummy;
            const int s_lo = (c - Sg > 1 ? c - Sg : 1), s_hi = (Sg < c - 1 ? Sg : c - 1);
#pragma unroll
            for (int s = 1; s <= Sg; ++s) {
              if (s < s_lo || s > s_hi) continue;
              const int t = c - s;
              // K-major operands: slice j sits at byte 32 (j % 4) of the 128-byte rows
              // of quad tile j / 4 (128B swizzle, 8-row groups 1024 bytes apart)
              const uint32_t ao = AMN ? uint32_t((s - 1) * kATile)
                                      : uint32_t(((s - 1) >> 2) * 4 * kATile + ((s - 1) & 3) * 32);
              const uint32_t bo = uint32_t(((t - 1) >> 2) * btile4 + ((t - 1) & 3) * 32);
              umma_i8(tb + uint32_t((c - c_lo) * 128), ad_fixed | uint64_t(a0 + (ao >> 4)),
                      bd_fixed | uint64_t(b0 + (bo >> 4)), idesc, s > s_lo ? 1u : kacc);
            }
          }
        }
        __syncwarp();
        if (elect_one()) umma_commit(&bar_empty[st]);
        if (kb % kchunk == kchunk - 1 || kb == nk - 1) {  // int32 headroom: drain per K chunk
          if (elect_one()) umma_commit(&bar_acc_full);
          ++drains;
        }
      }
    };
    run_group(std::integral_constant<int, 0>{});
    if constexpr (S > 4) run_group(std::integral_constant<int, 1>{});
  } else {
    // ---------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may read
    const int row = q * 32 + lane;
    const int64_t grow = int64_t(m0) + row;
    const int re = (p.rexp && grow < p.M) ? p.rexp[grow] : 0;
    double* scr = p.scratch ? p.scratch + int64_t(blockIdx.x) * kBM * p.ntile : nullptr;
    for (int d = 0; d < ngroups * nchunks; ++d) {  // one drain per (diagonal group, K chunk)
      const int g = d / nchunks;
      const int c_hi = grp_c_hi(S, g), c_lo = grp_c_lo(S, g);
      const bool first_d = d == 0, last = d == ngroups * nchunks - 1;
      ptx::mbar_wait(&bar_acc_full, uint32_t(d) & 1);
      tc_fence_after();
      for (int cc = 0; cc < p.ntile; cc += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0.0;
        // all four accumulators' loads in flight before one wait
        uint32_t r[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (c_lo + i <= c_hi) tmem_ld8(tb + (uint32_t(q * 32) << 16) + uint32_t(i * 128 + cc), r[i]);
        tmem_ld_wait();
#pragma unroll
        for (int i = 3; i >= 0; --i) {  // smallest terms (highest c) first
          if (c_lo + i > c_hi) continue;
          const double sc = exp2i(-(8 * (c_lo + i) - 4));
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = fma(double(int(r[i][j])), sc, v[j]);
        }
        if (!first_d) {  // running sum of the earlier drains (this thread's own writes)
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] += scr[int64_t(cc + j) * kBM + row];
        }
        if (!last) {
#pragma unroll
          for (int j = 0; j < 8; ++j) scr[int64_t(cc + j) * kBM + row] = v[j];
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int col = n0 + cc + j;
            if (grow < p.M && col < p.N) {
              double x = v[j];
              x = scale2(x, re + (p.cexp ? p.cexp[col] : 0));
              double* dst = p.C + int64_t(col) * p.ldc + grow;
              *dst = p.accumulate ? *dst + x : x;
            }
          }
        }
      }
      tc_fence_before();
      ptx::mbar_arrive(&bar_acc_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512u)
                 : "memory");
  }
}

// ---------------------------------------------------- CTA-pair variant
// Two CTAs of a cluster (one TPC) run the MMAs as one `cta_group::2`
// instruction of M = 256: each CTA holds its own 128 rows of A and HALF of the
// B tile (64 of the pair's 128 output columns), so a CTA reads 6 KB of
// operands per MMA instead of 7.5 KB for 112 columns -- the single-CTA kernel
// above is bound by shared-memory bandwidth (78 cycles per MMA against the
// tensor pipe's 60).  The leader CTA (cluster rank 0) issues the MMAs and owns
// the full / accumulator-empty barriers; both CTAs' TMA loads signal the
// leader's full barrier, the leader's commits are multicast to both CTAs'
// empty / accumulator-full barriers; each CTA's epilogue drains its own TMEM.
constexpr int kStages2 = 4;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;     // shared::cluster address of the same offset in CTA 0

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma2_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(map), "r"(ptx::smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma2_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(map), "r"(ptx::smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma2_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive (once all earlier MMAs are done) on the barrier at this offset in both CTAs
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar, uint16_t pair_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(ptx::smem_u32(bar)),
      "h"(pair_mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   ptx::smem_u32(bar) & kPeerMask)
               : "memory");
}

template <int AMN, int S>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_gemm2_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, OzParams p) {
  RSVD_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
  __shared__ uint64_t bar_full[kStages2], bar_empty[kStages2], bar_acc_full, bar_acc_empty;
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // launched as clusters of 2 c CTAs (c CTA pairs with consecutive column tiles
  // of one row-tile pair: they start together and share A's tiles through L2)
  const int crank = int(cluster_ctarank());
  const int rank = crank & 1;  // within the pair
  const int pair = blockIdx.x >> 1;
  const int nt = pair % p.n_tiles, mt = 2 * (pair / p.n_tiles) + rank;
  const int NT = p.ntile;                 // output columns per pair: 64, 96 or 128
  const int bhalf4 = (NT / 2) * 128;      // this CTA's half of four B slices of one K step
  const int stage_bytes = kARegion + 2 * bhalf4;
  const int m0 = mt * kBM, n0 = nt * NT;
  const int nk = (p.K + kKS - 1) / kKS;
  constexpr int ngroups = (S + 3) / 4;
  constexpr int kchunk = max_k(S) / kKS;  // K steps one int32 accumulation may cover
  const int nchunks = (nk + kchunk - 1) / kchunk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages2; ++s) {
      ptx::mbar_init(&bar_full[s], 1);
      ptx::mbar_init(&bar_empty[s], 1);
    }
    ptx::mbar_init(&bar_acc_full, 1);
    ptx::mbar_init(&bar_acc_empty, 256);  // both CTAs' epilogue threads (leader's copy is used)
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     ptx::smem_u32(&tmem_base_sh)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tb = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------- TMA producer (both CTAs)
    if (lane == 0) {
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      int it = 0;
      for (int g = 0; g < ngroups; ++g) {
        const int Sg = grp_slices(S, g);
        const int nhalf = (Sg + 3) >> 2;
        const uint32_t bytes = uint32_t(AMN ? Sg * kATile : nhalf * 4 * kATile) + uint32_t(nhalf * bhalf4);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % kStages2;
          const uint32_t ph = (it / kStages2) & 1;
          ptx::mbar_wait(&bar_empty[st], ph ^ 1);
          if (rank == 0) ptx::mbar_expect_tx(&bar_full[st], 2 * bytes);  // both CTAs' loads land here
          uint8_t* base = sm + st * stage_bytes;
          const int kc = p.k0 + kb * kKS;
          const int ki = (kc >> 5) * 256;
          if (AMN) {
            for (int s = 0; s < Sg; ++s) tma2_load_3d(base + s * kATile, &tmA, &bar_full[st], m0, kc, s);
          } else {
            for (int hf = 0; hf < nhalf; ++hf)
              tma2_load_2d(base + hf * 4 * kATile, &tmA, &bar_full[st], ki + hf * 128, m0);
          }
          uint8_t* bb = base + kARegion;
          for (int hf = 0; hf < nhalf; ++hf)
            tma2_load_2d(bb + hf * bhalf4, &tmB, &bar_full[st], ki + hf * 128, n0 + rank * (NT / 2));
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------- MMA issuer (leader CTA)
    if (rank == 0) {
      // M = 256 (the pair), N = NT
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(AMN) << 15) |
                             (uint32_t(NT >> 3) << 17) | (uint32_t(256 >> 4) << 24);
      const uint64_t ad_fixed = smem_desc(0, AMN ? 4096 : 0, 1024, 2);
      const uint64_t bd_fixed = smem_desc(0, 0, 1024, 2);
      const uint32_t sm0 = ptx::smem_u32(sm);
      const uint16_t pair_mask = uint16_t(3u << (crank & ~1));  // this pair's two CTAs in the cluster
      int it = 0, drains = 0;
      auto run_group = [&](auto sg_tag) {
        constexpr int G = decltype(sg_tag)::value;
        constexpr int Sg = grp_slices(S, G), c_hi = grp_c_hi(S, G), c_lo = grp_c_lo(S, G);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % kStages2;
          const uint32_t ph = (it / kStages2) & 1;
          const bool chunk_start = kb % kchunk == 0;
          if (chunk_start && drains > 0) {  // both CTAs' epilogues drained the previous accumulation
            ptx::mbar_wait(&bar_acc_empty, uint32_t(drains - 1) & 1);
            tc_fence_after();
          }
          ptx::mbar_wait(&bar_full[st], ph);
          tc_fence_after();
          const uint32_t a0 = (sm0 + st * stage_bytes) >> 4;
          const uint32_t b0 = a0 + (kARegion >> 4);
          const uint32_t kacc = chunk_start ? 0u : 1u;
          if (elect_one()) {
#pragma unroll
            for (int c = c_hi; c >= c_lo; --c) {
              const int s_lo = (c - Sg > 1 ? c - Sg : 1), s_hi = (Sg < c - 1 ? Sg : c - 1);
#pragma unroll
              for (int s = 1; s <= Sg; ++s) {
                if (s < s_lo || s > s_hi) continue;
                const int t = c - s;
                const uint32_t ao = AMN ? uint32_t((s - 1) * kATile)
                                        : uint32_t(((s - 1) >> 2) * 4 * kATile + ((s - 1) & 3) * 32);
                const uint32_t bo = uint32_t(((t - 1) >> 2) * bhalf4 + ((t - 1) & 3) * 32);
                umma2_i8(tb + uint32_t((c - c_lo) * 128), ad_fixed | uint64_t(a0 + (ao >> 4)),
                         bd_fixed | uint64_t(b0 + (bo >> 4)), idesc, s > s_lo ? 1u : kacc);
              }
            }
          }
          __syncwarp();
          if (elect_one()) umma2_commit_both(&bar_empty[st], pair_mask);
          if (kb % kchunk == kchunk - 1 || kb == nk - 1) {  // int32 headroom: drain per K chunk
            if (elect_one()) umma2_commit_both(&bar_acc_full, pair_mask);
            ++drains;
          }
        }
      };
      run_group(std::integral_constant<int, 0>{});
      if constexpr (S > 4) run_group(std::integral_constant<int, 1>{});
    }
  } else {
    // ------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int64_t grow = int64_t(m0) + row;
    const int re = (p.rexp && grow < p.M) ? p.rexp[grow] : 0;
    double* scr = p.scratch ? p.scratch + int64_t(blockIdx.x) * kBM * NT : nullptr;
    for (int d = 0; d < ngroups * nchunks; ++d) {  // one drain per (diagonal group, K chunk)
      const int g = d / nchunks;
      const int c_hi = grp_c_hi(S, g), c_lo = grp_c_lo(S, g);
      const bool first_d = d == 0, last = d == ngroups * nchunks - 1;
      ptx::mbar_wait(&bar_acc_full, uint32_t(d) & 1);
      tc_fence_after();
      for (int cc = 0; cc < NT; cc += 8) {
        if (n0 + cc >= p.N) break;
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0.0;
        // all four accumulators' loads in flight before one wait
        uint32_t r[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (c_lo + i <= c_hi) tmem_ld8(tb + (uint32_t(q * 32) << 16) + uint32_t(i * 128 + cc), r[i]);
        tmem_ld_wait();
#pragma unroll
        for (int i = 3; i >= 0; --i) {  // smallest terms (highest c) first
          if (c_lo + i > c_hi) continue;
          const double sc = exp2i(-(8 * (c_lo + i) - 4));
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = fma(double(int(r[i][j])), sc, v[j]);
        }
        if (!first_d) {  // running sum of the earlier drains (this thread's own writes)
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] += scr[int64_t(cc + j) * kBM + row];
        }
        if (!last) {
#pragma unroll
          for (int j = 0; j < 8; ++j) scr[int64_t(cc + j) * kBM + row] = v[j];
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int col = n0 + cc + j;
            if (grow < p.M && col < p.N) {
              double x = v[j];
              x = scale2(x, re + (p.cexp ? p.cexp[col] : 0));
              double* dst = p.C + int64_t(col) * p.ldc + grow;
              *dst = p.accumulate ? *dst + x : x;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive_leader(&bar_acc_empty);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512u)
                 : "memory");
  }
}

// ------------------------------------------------------------- host side
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

// Launch with a runtime cluster size (and as a programmatic dependent, like launch_k)
template <typename... KArgs, typename... Args>
void launch_cluster(Handle& h, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                    int csize, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h.stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(csize);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  RSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// 3-D int8 map over slices stored [slice][outer][inner]: dims {inner, outer, S}
CUtensorMap make_map_i8(const uint8_t* p, int64_t inner, int64_t outer, int64_t ld8, int S,
                        int box_inner, int box_outer, bool swizzle128) {
  CUtensorMap m;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(outer), cuuint64_t(S)};
  cuuint64_t strides[2] = {cuuint64_t(ld8), cuuint64_t(ld8) * cuuint64_t(outer)};
  cuuint32_t box[3] = {cuuint32_t(box_inner), cuuint32_t(box_outer), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(p), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(RSVD_ERR_CUDA, "cuTensorMapEncodeTiled (int8) failed (" + std::to_string(int(r)) + ")");
  return m;
}

// 2-D map over an interleaved operand [outer][ldi bytes]: box {128 bytes, rows}
CUtensorMap make_map_inter(const uint8_t* p, int64_t inner_bytes, int64_t outer, int64_t ldi,
                           int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cuuint64_t(inner_bytes), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ldi)};
  cuuint32_t box[2] = {128, cuuint32_t(box_outer)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(p), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(RSVD_ERR_CUDA, "cuTensorMapEncodeTiled (interleaved) failed (" + std::to_string(int(r)) + ")");
  return m;
}

// Sliced operand in device memory (layouts: slice_kernel).  `inner` runs along
// the source's rows (contiguous in the fp64 matrix), `outer` along its columns.
//   plain:      S planes of `outer` columns, ld bytes each
//   interleave: `outer` columns of ld = 256 ceil(inner / 32) bytes
struct Sliced {
  uint8_t* p = nullptr;
  int64_t inner = 0, outer = 0, ld = 0;
};

int64_t ld_plain(int64_t inner) { return round_up(std::max<int64_t>(inner, 16), 16); }
int64_t ld_inter(int64_t inner) { return ceil_div(std::max<int64_t>(inner, 1), 32) * 256; }

uint8_t* alloc_aligned(Handle& h, size_t bytes) {
  uint8_t* p = static_cast<uint8_t*>(h.ws.alloc_bytes(bytes + 1024));
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
}
uint8_t* alloc_plain(Handle& h, int64_t cap_inner, int64_t outer, int S) {
  return alloc_aligned(h, size_t(S) * size_t(outer) * size_t(ld_plain(cap_inner)));
}
uint8_t* alloc_inter(Handle& h, int64_t cap_inner, int64_t outer) {
  return alloc_aligned(h, size_t(outer) * size_t(ld_inter(cap_inner)));
}
Sliced view_plain(uint8_t* p, int64_t inner, int64_t outer) {
  Sliced s;
  s.p = p, s.inner = inner, s.outer = outer, s.ld = ld_plain(inner);
  return s;
}
Sliced view_inter(uint8_t* p, int64_t inner, int64_t outer) {
  Sliced s;
  s.p = p, s.inner = inner, s.outer = outer, s.ld = ld_inter(inner);
  return s;
}

void fill_exp(Handle& h, int* e, int64_t n, int init) {
  if (n < 1) return;
  launch_k(h, fill_int_kernel, unsigned(ceil_div(n, 256)), 256, 0, e, int(n), init);
  RSVD_LAUNCHED(h);
}

// plain and / or inter may be null (p == nullptr)
void launch_slice(Handle& h, const DMat& X, const int* rsub, const int* radd, const int* csub,
                  const Sliced& plain, const Sliced& inter, int S) {
  if (X.rows == 0 || X.cols == 0) return;
  if (ceil_div(X.rows, 128) > 65535) throw_dim("ozaki: operand with more than 8388480 rows per slicing launch");
  dim3 grid(unsigned(ceil_div(X.cols, 8)), unsigned(ceil_div(X.rows, 128)));
#define RSVD_SLICE_CASE(SS)                                                                       \
  case SS:                                                                                        \
    launch_k(h, slice_kernel<SS>, grid, 256, 0, (const double*)X.p, X.ld, int(X.rows), int(X.cols), \
             rsub, radd, csub, plain.p, plain.ld, inter.p, inter.ld);                             \
    break;
  switch (S) {
    RSVD_SLICE_CASE(3)
    RSVD_SLICE_CASE(4)
    RSVD_SLICE_CASE(5)
    RSVD_SLICE_CASE(6)
    RSVD_SLICE_CASE(7)
    RSVD_SLICE_CASE(8)
    default:
      throw_param("ozaki: slices must be in 3..8");
  }
#undef RSVD_SLICE_CASE
  RSVD_LAUNCHED(h);
}

// per-row exponents of X (rows x cols): |x_rc| < 2^e[r]
void row_exponents(Handle& h, const DMat& X, int* e) {
  fill_exp(h, e, X.rows, -1022);
  if (X.rows == 0 || X.cols == 0) return;
  // enough blocks to fill the machine: split the columns
  const int64_t rb = ceil_div(X.rows, 256);
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(ceil_div(X.cols, 64), ceil_div(h.sm_count * 8, rb)));
  const int cpb = int(ceil_div(X.cols, splits));
  splits = ceil_div(X.cols, cpb);
  launch_k(h, row_exp_kernel, dim3(unsigned(rb), unsigned(splits)), 256, 0, (const double*)X.p, X.ld,
           int(X.rows), X.cols, cpb, e, h.d_flags);
  RSVD_LAUNCHED(h);
}

// per-column exponents of diag(2^radd) X: |2^radd[r] x_rc| < 2^e[c]
void col_exponents(Handle& h, const DMat& X, const int* radd, int* e) {
  fill_exp(h, e, X.cols, -1022 - 1100);
  if (X.rows == 0 || X.cols == 0) return;
  const int rpb = 8192;
  launch_k(h, col_exp_kernel, dim3(unsigned(X.cols), unsigned(ceil_div(X.rows, rpb))), 256, 0,
           (const double*)X.p, X.ld, int(X.rows), rpb, radd, e, h.d_flags);
  RSVD_LAUNCHED(h);
}

// CTA-pair kernel (cta_group::2, 128 output columns per pair) unless RSVD_OZ_CG2=0
std::atomic<int> g_pair_kernel{-1};  // -1 = RSVD_OZ_CG2 (default on), 0 / 1 = forced (tests)
bool use_pair_kernel() {
  const int f = g_pair_kernel.load(std::memory_order_relaxed);
  if (f >= 0) return f != 0;
  static const bool on = [] {
    const char* e = std::getenv("RSVD_OZ_CG2");
    return !(e && e[0] == '0');
  }();
  return on;
}
int pick_ntile(int64_t L) {
  if (use_pair_kernel()) {
    // cta_group::2 takes N in multiples of 32: the width that pads L least
    static const int forced = [] { const char* e = std::getenv("RSVD_OZ_NT"); return e ? std::atoi(e) : 0; }();
    if (forced == 64 || forced == 96 || forced == 128) return forced;
    int best = 128;
    for (int w : {96, 64})
      if (round_up(L, w) < round_up(L, best)) best = w;
    return best;
  }
  const int64_t tiles = ceil_div(L, 128);
  return int(round_up(ceil_div(L, tiles), 16));
}
// doubles of per-CTA partial tiles a GEMM with M x N outputs needs (S > 4)
int64_t scratch_doubles(int64_t M, int64_t N, int S) {
  (void)S;  // every launch may drain more than once (diagonal groups, K chunks)
  const int ntile = pick_ntile(N);
  return round_up(ceil_div(M, kBM), 2) * ceil_div(N, ntile) * kBM * ntile;
}

// C (M x N) (+)= sliced A  x  sliced B over K entries.
//   amn = true : As is plain [s][k][m] (M contiguous): the apply product
//   amn = false: As is interleaved [m][k/32][s][k%32]: the adjoint product
// Bs is interleaved [n][k/32][s][k%32].  rexp / cexp: exponents of the output
// rows / columns.
void launch_gemm(Handle& h, bool amn, const Sliced& As, const Sliced& Bs, int64_t M, int64_t N,
                 int64_t K, int S, DMat C, const int* rexp, const int* cexp, bool accumulate,
                 double* scratch) {
  if (M == 0 || N == 0) return;
  if (K < 1) throw_dim("ozaki: empty contraction");
  const int ntile = pick_ntile(N);
  const int n_tiles = int(ceil_div(N, ntile));
  const bool pair = use_pair_kernel();
  const int64_t m_tiles = pair ? round_up(ceil_div(M, kBM), 2) : ceil_div(M, kBM);
  const int64_t grid = m_tiles * n_tiles;
  const int stage_bytes = pair ? kARegion + ntile * 128 : kARegion + 2 * ntile * 128;
  const size_t smem = size_t(pair ? kStages2 : kStages) * stage_bytes + 1024;
  const CUtensorMap ta = amn ? make_map_i8(As.p, As.inner, As.outer, As.ld, S, kBM, kKS, true)
                             : make_map_inter(As.p, As.ld, As.outer, As.ld, kBM);
  const CUtensorMap tb = make_map_inter(Bs.p, Bs.ld, Bs.outer, Bs.ld, pair ? ntile / 2 : ntile);
  // CTA-pair kernel: clusters of 3 pairs (consecutive column tiles of one
  // row-tile pair) when the column tiles allow it, so the pairs sharing A's
  // tiles start together (RSVD_OZ_CLUSTER=2 keeps plain pairs)
  int csize = 2;
  if (pair) {
    static const int forced = [] { const char* e = std::getenv("RSVD_OZ_CLUSTER"); return e ? std::atoi(e) : 0; }();
    if (n_tiles % 3 == 0) csize = 6;
    else if (n_tiles % 2 == 0) csize = 4;
    if (forced == 2 || forced == 4 || forced == 6) csize = (n_tiles * 2) % forced == 0 ? forced : 2;
  }
  // the kernel drains its int32 accumulators every max_k(S) contraction steps;
  // a launch covers up to 2^24 of them (indices stay far inside int)
  const int64_t kmax = int64_t(1) << 24;
  for (int64_t k0 = 0; k0 < K; k0 += kmax) {
    OzParams p;
    p.M = int(M);
    p.N = int(N);
    p.K = int(std::min<int64_t>(kmax, K - k0));
    p.k0 = int(k0);
    p.S = S;
    p.ntile = ntile;
    p.n_tiles = n_tiles;
    p.C = C.p;
    p.ldc = C.ld;
    p.rexp = rexp;
    p.cexp = cexp;
    p.accumulate = (accumulate || k0 > 0) ? 1 : 0;
    p.scratch = scratch;
    static const int dbg = [] { const char* e = std::getenv("RSVD_OZ_DBG"); return e ? std::atoi(e) : 0; }();
    p.dbg = dbg;
    // the kernel's algorithmic work: S(S+1)/2 exact int8 products of M x N x K,
    // every slice byte of both operands read once, the fp64 tile written
    ProfScope prof(h, 4, double(S * (S + 1) / 2) * 2.0 * double(M) * double(N) * double(p.K),
                   double(S) * double(p.K) * double(M + N) + 8.0 * double(M) * double(N));
#define RSVD_OZ_CASE(SS)                                                             \
  case SS:                                                                           \
    if (pair && amn) {                                                               \
      smem_attr(ozaki_gemm2_kernel<1, SS>, smem);                                    \
      launch_cluster(h, ozaki_gemm2_kernel<1, SS>, unsigned(grid), kThreads, smem, csize, ta, tb, p); \
    } else if (pair) {                                                               \
      smem_attr(ozaki_gemm2_kernel<0, SS>, smem);                                    \
      launch_cluster(h, ozaki_gemm2_kernel<0, SS>, unsigned(grid), kThreads, smem, csize, ta, tb, p); \
    } else if (amn) {                                                                \
      smem_attr(ozaki_gemm_kernel<1, SS>, smem);                                     \
      launch_k(h, ozaki_gemm_kernel<1, SS>, unsigned(grid), kThreads, smem, ta, tb, p); \
    } else {                                                                         \
      smem_attr(ozaki_gemm_kernel<0, SS>, smem);                                     \
      launch_k(h, ozaki_gemm_kernel<0, SS>, unsigned(grid), kThreads, smem, ta, tb, p); \
    }                                                                                \
    break;
    switch (S) {
      RSVD_OZ_CASE(3)
      RSVD_OZ_CASE(4)
      RSVD_OZ_CASE(5)
      RSVD_OZ_CASE(6)
      RSVD_OZ_CASE(7)
      RSVD_OZ_CASE(8)
      default:
        throw_param("ozaki: slices must be in 3..8");
    }
#undef RSVD_OZ_CASE
    RSVD_LAUNCHED(h);
    prof.end();
  }
}

// Rows of A sliced at a time: int32 accumulation bounds the adjoint's
// contraction length per launch, not the panel; `copies` layouts of the sub-panel's slices
// (S K bytes per row each) must fit in what the device has left.
int64_t sub_rows(Handle& h, int64_t K, int S, int copies) {
  size_t free_b = 0, total_b = 0;
  RSVD_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double budget = std::min(40.0e9, 0.8 * (double(free_b) + double(h.ws.remaining())));
  int64_t sub = kMaxRows;
  while (sub > 1024 && double(sub) * double(K) * S * copies > budget) sub /= 2;
  return sub;
}

struct StreamSwap {  // launches of this scope go to `s`
  Handle& h;
  cudaStream_t old;
  StreamSwap(Handle& hh, cudaStream_t s) : h(hh), old(hh.stream) { h.stream = s; }
  ~StreamSwap() { h.stream = old; }
};

}  // namespace

void ozaki_force_pair_kernel(int pair) { g_pair_kernel.store(pair < 0 ? -1 : (pair ? 1 : 0)); }

int ozaki_slices(const Handle& h) {
  if (h.ozaki_slices >= 0) return h.ozaki_slices;
  static const int env = [] {
    const char* e = std::getenv("RSVD_OZAKI");
    if (!e) return -1;
    const int v = std::atoi(e);
    return (v >= 3 && v <= kMaxS) ? v : 0;
  }();
  return env;
}

// Default policy of the Alg-6 dual pass (engine.cu op_dual): the sliced INT8
// product with 7 slices (inside the error bound of an fp64 product, see the
// header) when the sketch is wide enough for the tensor pipe to pay for the
// slicing passes (l >= 128: at l = 110 it breaks even with the DMMA pass,
// below that the pass is HBM-bound anyway) and A is large (>= 2^26 entries).
int ozaki_slices_auto(const Handle& h, int64_t rows, int64_t K, int64_t L) {
  const int s = ozaki_slices(h);
  if (s >= 0) return s;
  return (L >= 128 && double(rows) * double(K) >= double(int64_t(1) << 26)) ? kAutoSlices : 0;
}

namespace {
void ensure_state(Handle& h, OzakiState* st, int64_t rows_total, int64_t K, int64_t L, int S,
                  bool need_x, bool need_p) {
  if (st->have) return;
  const int layouts = (need_x ? 1 : 0) + (need_p ? 1 : 0);
  const int64_t want = round_up(std::max<int64_t>(rows_total, 1), 128);
  st->cap = std::min<int64_t>(sub_rows(h, K, S, layouts), want);
  // a second set of panel buffers when it costs no panel size and there is a
  // next panel to slice ahead (the virtual communicator's ranks share a stream)
  st->nbuf = 1;
  if (need_x && need_p && !h.vcomm && rows_total > st->cap &&
      std::min<int64_t>(sub_rows(h, K, S, 2 * layouts), want) == st->cap) {
    static const bool off = [] { const char* e = std::getenv("RSVD_OZ_OVERLAP"); return e && e[0] == '0'; }();
    if (!off) st->nbuf = 2;
  }
  for (int b = 0; b < st->nbuf; ++b) {
    st->e_a[b] = static_cast<int*>(h.ws.alloc_bytes(size_t(st->cap) * 4));
    if (need_x) st->as[b] = alloc_plain(h, st->cap, K, S);
    if (need_p) st->asi[b] = alloc_inter(h, st->cap, K);
  }
  if (need_x) {
    st->xs = alloc_inter(h, K, L);
    st->e_x = static_cast<int*>(h.ws.alloc_bytes(size_t(L) * 4));
  }
  if (need_p) {
    st->ps = alloc_inter(h, st->cap, L);
    st->e_p = static_cast<int*>(h.ws.alloc_bytes(size_t(L) * 4));
  }
  const int64_t sd = std::max(need_x ? scratch_doubles(st->cap, L, S) : 0,
                              need_p ? scratch_doubles(K, L, S) : 0);
  if (sd) st->scratch = h.ws.alloc(sd);
  if (st->nbuf == 2 && !h.oz_stream) {
    RSVD_CUDA(cudaStreamCreateWithFlags(&h.oz_stream, cudaStreamNonBlocking));
    for (auto& e : h.oz_ev) RSVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  st->have = true;
}
}  // namespace

void ozaki_dual_pass(Handle& h, const DMat& A, const DMat& Oc, const DMat& Psi, DMat Y, DMat W,
                     int64_t row0, int64_t row_end, OzakiState* st, bool first, int S) {
  const int64_t K = A.cols, L = Oc.cols;
  if (Oc.rows != K || Psi.rows != A.rows || Psi.cols != L || Y.rows != A.rows || Y.cols != L ||
      W.rows != K || W.cols != L)
    throw_dim("ozaki_dual_pass: shape mismatch");
  if (S < 3 || S > kMaxS) throw_param("ozaki: slices must be in 3..8");
  const double mr = double(row_end - row0);
  ProfScope prof(h, 3, 4.0 * mr * double(K) * double(L),
                 8.0 * (mr * double(K) + 2.0 * double(K) * double(L) + 2.0 * mr * double(L)));
  const Sliced none;
  if (!st->have) {
    ensure_state(h, st, A.rows, K, L, S, true, true);
    col_exponents(h, Oc, nullptr, st->e_x);
    launch_slice(h, Oc, nullptr, nullptr, st->e_x, none, view_inter(st->xs, K, L), S);
  }
  const Sliced xs = view_inter(st->xs, K, L);
  cudaEvent_t* ev_sliced = h.oz_ev + 1;
  cudaEvent_t* ev_free = h.oz_ev + 3;
  const bool two = st->nbuf == 2;
  if (two) RSVD_CUDA(cudaEventRecord(h.oz_ev[0], h.stream));  // this panel's rows are resident
  // exponent scan + slicing of rows [r0, r1): one read of the panel writes both
  // operand layouts of its slices.  With two buffer sets it runs on the second
  // stream, beside the previous sub-panel's GEMMs.
  auto slice_sub = [&](int64_t r0) {
    const int64_t rows = std::min(row_end, r0 + st->cap) - r0;
    const int b = int(st->count % st->nbuf);
    const DMat Ap(A.p + r0, rows, K, A.ld);
    const Sliced as = view_plain(st->as[b], rows, K), asi = view_inter(st->asi[b], rows, K);
    if (two) {
      StreamSwap sw(h, h.oz_stream);
      RSVD_CUDA(cudaStreamWaitEvent(h.oz_stream, h.oz_ev[0], 0));
      if (st->count >= 2) RSVD_CUDA(cudaStreamWaitEvent(h.oz_stream, ev_free[b], 0));
      row_exponents(h, Ap, st->e_a[b]);
      launch_slice(h, Ap, st->e_a[b], nullptr, nullptr, as, asi, S);
      RSVD_CUDA(cudaEventRecord(ev_sliced[b], h.oz_stream));
    } else {
      row_exponents(h, Ap, st->e_a[b]);
      launch_slice(h, Ap, st->e_a[b], nullptr, nullptr, as, asi, S);
    }
    st->count++;
  };
  slice_sub(row0);
  for (int64_t r0 = row0; r0 < row_end; r0 += st->cap) {
    const int64_t r1 = std::min(row_end, r0 + st->cap), rows = r1 - r0;
    const int b = int((st->count - 1) % st->nbuf);  // the set slice_sub(r0) filled
    if (two) RSVD_CUDA(cudaStreamWaitEvent(h.stream, ev_sliced[b], 0));
    if (r1 < row_end) slice_sub(r1);  // ahead of this sub-panel's GEMMs
    const Sliced as = view_plain(st->as[b], rows, K), asi = view_inter(st->asi[b], rows, K);
    // Y[r0:r1, :] = A_p Omega_c
    launch_gemm(h, true, as, xs, rows, L, K, S, DMat(Y.p + r0, rows, L, Y.ld), st->e_a[b], st->e_x,
                false, st->scratch);
    // W (+)= A_p^T Psi_p, with Psi_p' = diag(2^eA) Psi_p so A's row scales cancel
    const DMat Pp(Psi.p + r0, rows, L, Psi.ld);
    col_exponents(h, Pp, st->e_a[b], st->e_p);
    const Sliced ps = view_inter(st->ps, rows, L);
    launch_slice(h, Pp, nullptr, st->e_a[b], st->e_p, none, ps, S);
    launch_gemm(h, false, asi, ps, K, L, rows, S, W, nullptr, st->e_p, !(first && r0 == row0),
                st->scratch);
    if (two) RSVD_CUDA(cudaEventRecord(ev_free[b], h.stream));
  }
  prof.end();
}

void ozaki_gemm(Handle& h, const DMat& A, const DMat& X, DMat C, bool trans, int S) {
  if (S < 3 || S > kMaxS) throw_param("ozaki: slices must be in 3..8");
  const int64_t L = X.cols, K = A.cols;
  if (!trans ? (X.rows != A.cols || C.rows != A.rows || C.cols != L)
             : (X.rows != A.rows || C.rows != A.cols || C.cols != L))
    throw_dim("ozaki_gemm: shape mismatch");
  OzakiState state;
  OzakiState* st = &state;
  ensure_state(h, st, A.rows, K, L, S, !trans, trans);
  const Sliced none;
  if (!trans) {
    col_exponents(h, X, nullptr, st->e_x);
    launch_slice(h, X, nullptr, nullptr, st->e_x, none, view_inter(st->xs, K, L), S);
  }
  for (int64_t r0 = 0; r0 < A.rows; r0 += st->cap) {
    const int64_t rows = std::min<int64_t>(st->cap, A.rows - r0);
    const DMat Ap(A.p + r0, rows, K, A.ld);
    row_exponents(h, Ap, st->e_a[0]);
    if (!trans) {
      const Sliced as = view_plain(st->as[0], rows, K);
      launch_slice(h, Ap, st->e_a[0], nullptr, nullptr, as, none, S);
      launch_gemm(h, true, as, view_inter(st->xs, K, L), rows, L, K, S,
                  DMat(C.p + r0, rows, L, C.ld), st->e_a[0], st->e_x, false, st->scratch);
    } else {
      const Sliced asi = view_inter(st->asi[0], rows, K);
      launch_slice(h, Ap, st->e_a[0], nullptr, nullptr, none, asi, S);
      const DMat Xp(X.p + r0, rows, L, X.ld);
      col_exponents(h, Xp, st->e_a[0], st->e_p);
      const Sliced ps = view_inter(st->ps, rows, L);
      launch_slice(h, Xp, nullptr, st->e_a[0], st->e_p, none, ps, S);
      launch_gemm(h, false, asi, ps, K, L, rows, S, C, nullptr, st->e_p, r0 > 0, st->scratch);
    }
  }
}

bool ozaki_cache_decide(Handle& h, OzCache& c, const DMat& A, int64_t L, int passes) {
  if (c.decided) return c.on;
  c.decided = true;
  c.on = false;
  int S = ozaki_slices(h);
  if (S == 0 || A.rows < 1 || A.cols < 1) return false;
  if (S < 0) {
    // >= 3 products share one slicing pass from l = 96 up; a single product
    // (Alg 5) pays for its own slicing from l ~ 160 up (break-even at l = 110)
    const bool wide = passes >= 3 ? L >= 96 : (passes >= 1 && L >= 160);
    if (!(wide && double(A.rows) * double(A.cols) >= double(int64_t(1) << 26))) return false;
    S = kAutoSlices;
  }
  const int64_t K = A.cols;
  const int64_t cap = std::min<int64_t>(kMaxRows, round_up(A.rows, 128));
  const int64_t nsub = ceil_div(A.rows, cap);
  const double need = double(nsub) * (double(S) * double(K) * double(ld_plain(cap)) +
                                      double(K) * double(ld_inter(cap))) + 64.0e6;
  size_t free_b = 0, total_b = 0;
  RSVD_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (need > 0.8 * (double(free_b) + double(h.ws.remaining()))) return false;
  c.S = S;
  c.cap = cap;
  c.nsub = nsub;
  c.on = true;
  return true;
}

void ozaki_cached_gemm(Handle& h, OzCache& c, const DMat& A, const DMat& X, DMat C, bool trans) {
  const int64_t K = A.cols, L = X.cols;
  const int S = c.S;
  if (!trans ? (X.rows != A.cols || C.rows != A.rows || C.cols != L)
             : (X.rows != A.rows || C.rows != A.cols || C.cols != L))
    throw_dim("ozaki_cached_gemm: shape mismatch");
  const Sliced none;
  const size_t plane_p = size_t(S) * size_t(K) * size_t(ld_plain(c.cap));
  const size_t plane_i = size_t(K) * size_t(ld_inter(c.cap));
  if (!c.built) {
    // one read of A (exponent scan + slicing per sub-panel) for all the passes of the call
    c.as = alloc_aligned(h, plane_p * size_t(c.nsub));
    c.asi = alloc_aligned(h, plane_i * size_t(c.nsub));
    c.e_a = static_cast<int*>(h.ws.alloc_bytes(size_t(A.rows) * 4));
    for (int64_t s = 0; s < c.nsub; ++s) {
      const int64_t r0 = s * c.cap, rows = std::min(c.cap, A.rows - r0);
      const DMat Ap(A.p + r0, rows, K, A.ld);
      row_exponents(h, Ap, c.e_a + r0);
      launch_slice(h, Ap, c.e_a + r0, nullptr, nullptr, view_plain(c.as + plane_p * size_t(s), rows, K),
                   view_inter(c.asi + plane_i * size_t(s), rows, K), S);
    }
    c.built = true;
  }
  if (L > c.Lcap) {
    c.xs = alloc_inter(h, K, L);
    c.ps = alloc_inter(h, c.cap, L);
    c.e_x = static_cast<int*>(h.ws.alloc_bytes(size_t(L) * 4));
    c.e_p = static_cast<int*>(h.ws.alloc_bytes(size_t(L) * 4));
    const int64_t sd = std::max(scratch_doubles(c.cap, L, S), scratch_doubles(K, L, S));
    c.scratch = sd ? h.ws.alloc(sd) : nullptr;
    c.Lcap = L;
  }
  if (!trans) {
    col_exponents(h, X, nullptr, c.e_x);
    const Sliced xs = view_inter(c.xs, K, L);
    launch_slice(h, X, nullptr, nullptr, c.e_x, none, xs, S);
    for (int64_t s = 0; s < c.nsub; ++s) {
      const int64_t r0 = s * c.cap, rows = std::min(c.cap, A.rows - r0);
      launch_gemm(h, true, view_plain(c.as + plane_p * size_t(s), rows, K), xs, rows, L, K, S,
                  DMat(C.p + r0, rows, L, C.ld), c.e_a + r0, c.e_x, false, c.scratch);
    }
  } else {
    for (int64_t s = 0; s < c.nsub; ++s) {
      const int64_t r0 = s * c.cap, rows = std::min(c.cap, A.rows - r0);
      const DMat Xp(X.p + r0, rows, L, X.ld);
      col_exponents(h, Xp, c.e_a + r0, c.e_p);
      const Sliced ps = view_inter(c.ps, rows, L);
      launch_slice(h, Xp, nullptr, c.e_a + r0, c.e_p, none, ps, S);
      launch_gemm(h, false, view_inter(c.asi + plane_i * size_t(s), rows, K), ps, K, L, rows, S, C,
                  nullptr, c.e_p, s > 0, c.scratch);
    }
  }
}

}  // namespace rsvdb
