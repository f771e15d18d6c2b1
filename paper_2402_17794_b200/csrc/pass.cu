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
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>
#include <cstdio>

#include "common.cuh"
#include "pass.cuh"
#include "ptx.cuh"

namespace rsvdb {


// ---------------------------------------------------------------- kernel
// CW consumer warps (DMMA) + one TMA producer warp per CTA.

// XC = 1: the last of the BN/8 loaded column groups holds ONE real column,
// computed with DFMA from the A fragments already in registers instead of a
// padded DMMA n-tile (l = 25 = 3 x 8 + 1: 24 columns on DMMA + 1 on DFMA does
// 25/32 of the FP64-pipe work of padding to 32; DMMA and DFMA share the pipe).
template <bool kNN, int BN, int WMT, int BK, int STAGES, int XC, int CW>
struct PassCfg {
  static constexpr int CWARPS = CW;
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int BM = CW * WMT * 8;
  static constexpr int NT = BN / 8 - XC;  // DMMA n-tiles
  static constexpr int NCOL = NT * 8 + XC;  // output columns per tile
  static constexpr int FRAG = CW * WMT * NT * 64 + XC * CW * WMT * 32;
  static constexpr int KH = BK / 16;  // 16-wide (128-byte) swizzle boxes along K
  static constexpr int A_BYTES = BM * BK * 8;
  static constexpr int B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int PIPE_BYTES = STAGES * STAGE_BYTES;
  static constexpr int SMEM = PIPE_BYTES + 1024 /*align*/ + 2 * STAGES * 8 + 16;
  static_assert(BN % 8 == 0, "BN must be a multiple of 8");
  static_assert(BK % 16 == 0, "BK must be a multiple of 16");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle-128B alignment");
  static_assert(BM <= 256, "TMA box limit");
};

// Work schedule.  A "unit" is one BK-deep slice of one output tile; tiles are
// numbered t = m_tile * nt + n_tile.  Two schedules share one kernel:
//  * split-K:  grid (nt, mt, S); CTA (n, m, s) owns tile (m, n), K slices
//              [s*kps, (s+1)*kps).  Concurrent CTAs of the same m_tile read the
//              same A rows, so A is re-read from L2, not HBM (many-tile passes).
//  * stream-K: 1-D grid of G persistent CTAs; CTA c owns the contiguous unit
//              range [c*U/G, (c+1)*U/G) of the tile-major unit space and may
//              cover several partial tiles ("segments") -- all SMs busy even when
//              there are fewer tiles than SMs (C1/C2 passes, Gram products).
// A tile covered by several segments is reduced by the last-arriving segment's
// CTA, which sums every segment's partial in FIXED segment order (its own from
// registers): bitwise deterministic, no floating-point atomics.
struct PassParams {
  int64_t M, N, K;
  int mt, nt, kb_tile;   // tile grid and BK-slices per tile
  int stream_k;          // schedule
  int splits;            // split-K: S
  int kb_split;          // split-K: BK-slices per split
  int64_t units;         // stream-K: U = mt * nt * kb_tile
  int grid;              // stream-K: G
  int max_seg;           // stream-K: partial slots per CTA
  int nsub;              // stream-K: CTAs c with equal c / nsub walk the same
                         // m-tile / K-slice range, one n-tile each (c % nsub):
                         // the n-tiles of an A block are read at the same time
  double* C;
  int64_t ldc;
  double* partials;
  int* counters;
  unsigned long long* probe;  // debug (RSVD_PROBE_PASS): 16 %globaltimer stamps per CTA
  int defer;             // stream-K: partial tiles are summed by sk_reduce_kernel
};

__device__ __forceinline__ int64_t sk_begin(int c, const PassParams& p) {
  return (int64_t(c) * p.units) / p.grid;
}
__device__ __forceinline__ int sk_cta_of(int64_t u, const PassParams& p) {
  int c = int((u * p.grid) / p.units);
  while (c + 1 < p.grid && sk_begin(c + 1, p) <= u) ++c;
  while (c > 0 && sk_begin(c, p) > u) --c;
  return c;
}

template <bool kNN, int BN, int WMT, int BK, int STAGES, int XC, int CW, bool kGroup>
// CW <= 4: two CTAs per SM (two independent TMA rings), registers capped to fit
__global__ void __launch_bounds__((CW + 1) * 32, (CW <= 4) ? 2 : 1)
    pass_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                PassParams p) {
  RSVD_PDL_ENTRY();
  using Cfg = PassCfg<kNN, BN, WMT, BK, STAGES, XC, CW>;
  constexpr int kConsumerWarps = CW;
  constexpr int BM = Cfg::BM, NT = Cfg::NT, NCOL = Cfg::NCOL;
  constexpr int FRAG = Cfg::FRAG;  // doubles per partial tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Pointer arithmetic on the __shared__ array (no integer round trip) keeps
  // the state space visible to the compiler: fragment loads become LDS.
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::PIPE_BYTES);
  uint64_t* empty = full + STAGES;
  int* flag = reinterpret_cast<int*>(empty + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // This CTA's unit range (tile-major units for stream-K; one segment for split-K).
  int64_t u0, u1;
  int fixed_tile = 0, fixed_kb0 = 0;
  // kGroup: stream-K with nsub > 1 n-tile CTAs per unit range (compile-time,
  // so the common nsub = 1 schedule carries no extra integer work)
  const int grp = (p.stream_k && kGroup) ? int(blockIdx.x) / p.nsub : int(blockIdx.x);
  const int sub = (p.stream_k && kGroup) ? int(blockIdx.x) % p.nsub : 0;
  if (p.stream_k) {
    u0 = sk_begin(grp, p);
    u1 = sk_begin(grp + 1, p);
  } else {
    fixed_tile = blockIdx.y * p.nt + blockIdx.x;
    fixed_kb0 = blockIdx.z * p.kb_split;
    const int kb1 = min(p.kb_tile, fixed_kb0 + p.kb_split);
    u0 = 0;
    u1 = max(0, kb1 - fixed_kb0);
  }
  // stream-K unit u: m-tile-major (u / kb_tile = m-tile when nsub = nt, else
  // the tile itself), K slice u % kb_tile; this CTA's n-tile is `sub`
  auto unit_tile = [&](int64_t u) {
    if constexpr (kGroup) return p.stream_k ? int(u / p.kb_tile) * p.nsub + sub : fixed_tile;
    return p.stream_k ? int(u / p.kb_tile) : fixed_tile;
  };
  auto unit_kb = [&](int64_t u) { return p.stream_k ? int(u % p.kb_tile) : fixed_kb0 + int(u); };

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
      for (int64_t u = u0; u < u1; ++u) {
        const int i = int(u - u0);
        const int s = i % STAGES;
        if (i >= STAGES) ptx::mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        uint8_t* a_st = smem + s * Cfg::STAGE_BYTES;
        uint8_t* b_st = a_st + Cfg::A_BYTES;
        ptx::mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        const int t = unit_tile(u);
        const int m0 = (t / p.nt) * BM, n0 = (t % p.nt) * NCOL;
        const int k0 = unit_kb(u) * BK;
        if constexpr (kNN) {
          // A is M x K, M inner: boxes of 16 (M) x BK (K).
#pragma unroll
          for (int b = 0; b < BM / 16; ++b)
            ptx::tma_load_2d(a_st + b * (BK * 128), &tmA, &full[s], m0 + 16 * b, k0, pol_a);
        } else {
          // A is K x M, K inner: boxes of 16 (K) x BM (M).
#pragma unroll
          for (int h = 0; h < Cfg::KH; ++h)
            ptx::tma_load_2d(a_st + h * (BM * 128), &tmA, &full[s], k0 + 16 * h, m0, pol_a);
        }
#pragma unroll
        for (int h = 0; h < Cfg::KH; ++h)
          ptx::tma_load_2d(b_st + h * (BN * 128), &tmB, &full[s], k0 + 16 * h, n0, pol_b);
      }
    }
    return;
  }

  // -------------------------------------------------- DMMA consumer warps
  const int r8 = lane >> 2, c4 = lane & 3;
  const int wm0 = warp * WMT * 8;
  const int tid = threadIdx.x;
  constexpr int NCT = kConsumerWarps * 32;
  // Per-lane fragment offsets (bytes within a stage).  Shared memory serves a
  // 64-bit warp load as two half-warp wavefronts, so each HALF warp must hit
  // 16 distinct 8-byte bank slots (measured: 4 wavefronts instead of 2 per
  // LDS.64 otherwise).  Inside every 16-wide K block the four DMMA k-steps use
  // the K sets  {0, 3, 12, 15} ^ t,  t in {0, 1, 4, 5}  (lane c4 takes
  // base[c4] ^ t; A and B agree, so the contraction is unchanged):
  //  * K-inner tiles (128B-swizzled rows of 16 K values) need bits 3 and 0 of
  //    k distinct over c4,
  //  * the M-inner NN A tile (rows = K index) needs bits 2..1 of k distinct;
  // {0, 3, 12, 15} satisfies both.  Every lane-dependent term is folded into
  // one register; the k-step enters as an XOR with a compile-time constant on
  // bits 3..10 (disjoint from the immediate box/tile offsets).
  const int kb = (c4 == 0) ? 0 : (c4 == 1) ? 3 : (c4 == 2) ? 12 : 15;
  int offA0;
  if constexpr (kNN)
    // the warp's 8-row tile index parity selects the 16-row box half (WMT odd)
    offA0 = (wm0 >> 4) * (BK * 128) + kb * 128 +
            (((((wm0 >> 3) & 1) << 2 | (r8 >> 1)) ^ (kb & 7)) << 4) + (r8 & 1) * 8;
  else
    offA0 = wm0 * 128 + r8 * 128 + (((kb >> 1) ^ r8) << 4) + (kb & 1) * 8;
  const int offB0 = r8 * 128 + (((kb >> 1) ^ r8) << 4) + (kb & 1) * 8;
  // XC column (row NT*8 of the B tile, swizzle XOR 0): byte k16 * 8
  const int offX0 = kb * 8;
  int64_t u = u0;
  int seg_local = 0;
  unsigned long long* pr = (p.probe && tid == 0) ? p.probe + int64_t(blockIdx.x + blockIdx.y * gridDim.x +
                                                                      blockIdx.z * gridDim.x * gridDim.y) * 16
                                                 : nullptr;
  if (pr) pr[0] = ptx::gtime();
  do {
    double acc[WMT][NT][2];
    double xacc[WMT], xacc2[WMT];  // two K-parity chains for the DFMA column
#pragma unroll
    for (int i = 0; i < WMT; ++i) {
      xacc[i] = xacc2[i] = 0.0;
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    const int t = (u < u1) ? unit_tile(u) : fixed_tile;
    const int tg = (p.stream_k && kGroup) ? t / p.nsub : t;  // unit-space tile (group of n-tiles)
    const int64_t seg_end = p.stream_k ? min(u1, int64_t(tg + 1) * p.kb_tile) : u1;
    for (; u < seg_end; ++u) {
      const int i = int(u - u0);
      const int s = i % STAGES;
      ptx::mbar_wait(&full[s], (i / STAGES) & 1);
      if (pr && i == 0) pr[1] = ptx::gtime();
      const uint8_t* a_st = smem + s * Cfg::STAGE_BYTES;
      const uint8_t* b_st = a_st + Cfg::A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        constexpr int kT[4] = {0, 1, 4, 5};
        const int t = kT[ks & 3], kb16 = ks >> 2;
        const int cB = ((t >> 1) << 4) | ((t & 1) << 3);
        double af[WMT], bf[NT];
        if constexpr (kNN) {
#pragma unroll
          for (int i2 = 0; i2 < WMT; ++i2) {
            const int cA = (t << 7) | (((4 * (i2 & 1)) ^ t) << 4);
            af[i2] = *reinterpret_cast<const double*>(a_st + (offA0 ^ cA) + (i2 >> 1) * (BK * 128) +
                                                      kb16 * 2048);
          }
        } else {
#pragma unroll
          for (int i2 = 0; i2 < WMT; ++i2)
            af[i2] = *reinterpret_cast<const double*>(a_st + (offA0 ^ cB) + kb16 * (BM * 128) +
                                                      i2 * 1024);
        }
#pragma unroll
        for (int j = 0; j < NT; ++j)
          bf[j] = *reinterpret_cast<const double*>(b_st + (offB0 ^ cB) + kb16 * (BN * 128) + j * 1024);
#pragma unroll
        for (int i2 = 0; i2 < WMT; ++i2)
#pragma unroll
          for (int j = 0; j < NT; ++j) ptx::dmma(acc[i2][j][0], acc[i2][j][1], af[i2], bf[j]);
        if constexpr (XC == 1) {
          // lane holds A(m = 8i + r8, k = kr): partial dot product with column NT*8
          const double bx = *reinterpret_cast<const double*>(
              b_st + kb16 * (BN * 128) + NT * 1024 + (offX0 ^ (t * 8)));
#pragma unroll
          for (int i2 = 0; i2 < WMT; ++i2) {
            if (ks & 1)
              xacc2[i2] = fma(af[i2], bx, xacc2[i2]);
            else
              xacc[i2] = fma(af[i2], bx, xacc[i2]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }

    if (pr && seg_local < 4) pr[2 + 3 * seg_local] = ptx::gtime();
    // ---------------------------------------------- segment epilogue (tile t)
    if constexpr (XC == 1) {
      // the 4 lanes of a row hold disjoint K subsets: butterfly sum (identical
      // in all 4 lanes: IEEE addition is commutative)
#pragma unroll
      for (int i2 = 0; i2 < WMT; ++i2) {
        xacc[i2] += xacc2[i2];
        xacc[i2] += __shfl_xor_sync(0xffffffffu, xacc[i2], 1);
        xacc[i2] += __shfl_xor_sync(0xffffffffu, xacc[i2], 2);
      }
    }
    const int64_t m0 = int64_t(t / p.nt) * BM, n0 = int64_t(t % p.nt) * NCOL;
    int nseg, my_seg, c_first = 0;
    if (p.stream_k) {
      c_first = sk_cta_of(int64_t(tg) * p.kb_tile, p);  // CTA groups
      const int c_last = sk_cta_of(int64_t(tg + 1) * p.kb_tile - 1, p);
      nseg = c_last - c_first + 1;
      my_seg = grp - c_first;
    } else {
      nseg = p.splits;
      my_seg = blockIdx.z;
    }
    auto store = [&](double (&v)[WMT][NT][2], double (&vx)[WMT]) {
#pragma unroll
      for (int i2 = 0; i2 < WMT; ++i2) {
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t m = m0 + wm0 + i2 * 8 + r8, n = n0 + j * 8 + 2 * c4 + e;
            if (m < p.M && n < p.N) p.C[n * p.ldc + m] = v[i2][j][e];
          }
        if constexpr (XC == 1) {
          const int64_t m = m0 + wm0 + i2 * 8 + r8, n = n0 + NT * 8;
          if (c4 == 0 && m < p.M && n < p.N) p.C[n * p.ldc + m] = vx[i2];
        }
      }
    };
    if (nseg == 1) {
      store(acc, xacc);
    } else {
      auto slot = [&](int sg) -> int64_t {
        if (!p.stream_k) return int64_t(t) * p.splits + sg;
        const int c2 = c_first + sg;  // group
        const int j2 = tg - int(sk_begin(c2, p) / p.kb_tile);
        return int64_t(kGroup ? c2 * p.nsub + sub : c2) * p.max_seg + j2;
      };
      // partial in fragment-native layout: [warp][i][j][lane][2] (16B / lane, coalesced)
      const bool warp_live = (m0 + wm0) < p.M;
      const int64_t my_slot = p.stream_k ? int64_t(blockIdx.x) * p.max_seg + seg_local
                                         : int64_t(t) * p.splits + my_seg;
      if (warp_live) {
        double2* dst = reinterpret_cast<double2*>(p.partials + my_slot * FRAG) +
                       (warp * WMT * NT) * 32 + lane;
#pragma unroll
        for (int i2 = 0; i2 < WMT; ++i2)
#pragma unroll
          for (int j = 0; j < NT; ++j)
            if (n0 + j * 8 < p.N) dst[(i2 * NT + j) * 32] = make_double2(acc[i2][j][0], acc[i2][j][1]);
        if constexpr (XC == 1) {
          double* dx = p.partials + my_slot * FRAG + kConsumerWarps * WMT * NT * 64 +
                       warp * WMT * 32 + lane;
#pragma unroll
          for (int i2 = 0; i2 < WMT; ++i2) dx[i2 * 32] = xacc[i2];
        }
      }
      if (p.defer) {  // the separate reduction kernel sums this tile (stream-K)
        if (pr && seg_local < 4) pr[3 + 3 * seg_local] = pr[4 + 3 * seg_local] = ptx::gtime();
        ++seg_local;
        continue;
      }
      // Ticket: the consumer warps' partial stores are ordered before thread
      // 0's GPU-scope fence by the CTA barrier (cumulativity), so ONE fence
      // releases them all; the last arriver's thread 0 fences again (acquire)
      // before the barrier that releases its CTA to read the other partials.
      // (Every thread fencing cost ~10 us per small pass: measured on C1.)
      ptx::named_bar(1, NCT);
      if (tid == 0) {
        ptx::fence_acq_rel_gpu();
        const bool last = (atomicAdd(&p.counters[t], 1) == nseg - 1);
        if (last) ptx::fence_acq_rel_gpu();
        *flag = last;
      }
      ptx::named_bar(1, NCT);
      if (pr && seg_local < 4) pr[3 + 3 * seg_local] = ptx::gtime() | (*flag ? 1ull : 0ull);
      if (*flag) {
        // Sum every segment's partial (this CTA's own included, re-read from
        // where it was just written) in segment order: deterministic.
        if (warp_live) {
#pragma unroll
          for (int i2 = 0; i2 < WMT; ++i2) {
            xacc[i2] = 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[i2][j][0] = acc[i2][j][1] = 0.0;
          }
          // RU partials in flight per round trip (summed in order afterwards)
          constexpr int RU = (WMT * NT <= 4) ? 4 : ((WMT * NT <= 8) ? 2 : 1);
          int sg = 0;
          for (; sg + RU <= nseg; sg += RU) {
            double2 v[RU][WMT][NT];
            double vx[RU][WMT];
#pragma unroll
            for (int r = 0; r < RU; ++r) {
              const double2* src = reinterpret_cast<const double2*>(p.partials + slot(sg + r) * FRAG) +
                                   (warp * WMT * NT) * 32 + lane;
#pragma unroll
              for (int i2 = 0; i2 < WMT; ++i2) {
#pragma unroll
                for (int j = 0; j < NT; ++j)
                  v[r][i2][j] = (n0 + j * 8 < p.N) ? __ldcg(src + (i2 * NT + j) * 32)
                                                   : make_double2(0.0, 0.0);
                vx[r][i2] = 0.0;
                if constexpr (XC == 1)
                  vx[r][i2] = __ldcg(p.partials + slot(sg + r) * FRAG +
                                     kConsumerWarps * WMT * NT * 64 + warp * WMT * 32 + lane + i2 * 32);
              }
            }
#pragma unroll
            for (int r = 0; r < RU; ++r)
#pragma unroll
              for (int i2 = 0; i2 < WMT; ++i2) {
                xacc[i2] += vx[r][i2];
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                  acc[i2][j][0] += v[r][i2][j].x;
                  acc[i2][j][1] += v[r][i2][j].y;
                }
              }
          }
          for (; sg < nseg; ++sg) {
            if constexpr (XC == 1) {
              const double* sx = p.partials + slot(sg) * FRAG + kConsumerWarps * WMT * NT * 64 +
                                 warp * WMT * 32 + lane;
#pragma unroll
              for (int i2 = 0; i2 < WMT; ++i2) xacc[i2] += __ldcg(sx + i2 * 32);
            }
            const double2* src = reinterpret_cast<const double2*>(p.partials + slot(sg) * FRAG) +
                                 (warp * WMT * NT) * 32 + lane;
#pragma unroll
            for (int i2 = 0; i2 < WMT; ++i2)
#pragma unroll
              for (int j = 0; j < NT; ++j)
                if (n0 + j * 8 < p.N) {
                  const double2 v = __ldcg(src + (i2 * NT + j) * 32);
                  acc[i2][j][0] += v.x;
                  acc[i2][j][1] += v.y;
                }
          }
          store(acc, xacc);
        }
        if (tid == 0) p.counters[t] = 0;  // self-reset for the next launch
      }
    }
    if (pr && seg_local < 4) pr[4 + 3 * seg_local] = ptx::gtime();
    ++seg_local;
  } while (u < u1);
  if (pr) pr[15] = ptx::gtime();
}

// Stream-K fixup as its own kernel: one CTA per output tile sums the tile's
// segment partials in segment order (the order the in-kernel last-arriver
// reduction used: bitwise the same result) and stores it.  Every partial of
// every tile is loaded in parallel across CTAs instead of one round trip per
// partial by the last-arriving CTA, and the pass kernel's CTAs never wait on
// a ticket (measured with RSVD_PROBE_PASS on C1: ticket 2.1 us per segment,
// in-kernel reduction 3.5-16 us, chained across consecutive tiles).
template <bool kNN, int BN, int WMT, int BK, int STAGES, int XC, int CW, bool kGroup>
__global__ void __launch_bounds__(CW * 32) sk_reduce_kernel(PassParams p) {
  RSVD_PDL_ENTRY();
  using Cfg = PassCfg<kNN, BN, WMT, BK, STAGES, XC, CW>;
  constexpr int BM = Cfg::BM, NT = Cfg::NT, NCOL = Cfg::NCOL, FRAG = Cfg::FRAG;
  const int t = blockIdx.x;
  const int tg = kGroup ? t / p.nsub : t, sub = kGroup ? t % p.nsub : 0;
  const int c_first = sk_cta_of(int64_t(tg) * p.kb_tile, p);
  const int c_last = sk_cta_of(int64_t(tg + 1) * p.kb_tile - 1, p);
  const int nseg = c_last - c_first + 1;
  if (nseg == 1) return;  // stored directly by the pass kernel
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r8 = lane >> 2, c4 = lane & 3, wm0 = warp * WMT * 8;
  const int64_t m0 = int64_t(t / p.nt) * BM, n0 = int64_t(t % p.nt) * NCOL;
  if (m0 + wm0 >= p.M) return;  // no rows of this warp in the tile
  auto slot = [&](int sg) -> int64_t {
    const int c2 = c_first + sg;
    const int j2 = tg - int(sk_begin(c2, p) / p.kb_tile);
    return int64_t(kGroup ? c2 * p.nsub + sub : c2) * p.max_seg + j2;
  };
  double acc[WMT][NT][2], xacc[WMT];
#pragma unroll
  for (int i2 = 0; i2 < WMT; ++i2) {
    xacc[i2] = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i2][j][0] = acc[i2][j][1] = 0.0;
  }
  constexpr int RU = 4;  // partials in flight per thread
  for (int sg0 = 0; sg0 < nseg; sg0 += RU) {
    double2 v[RU][WMT][NT];
    double vx[RU][WMT];
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const bool live = sg0 + r < nseg;
      const int64_t sl = live ? slot(sg0 + r) : 0;
      const double2* src =
          reinterpret_cast<const double2*>(p.partials + sl * FRAG) + (warp * WMT * NT) * 32 + lane;
#pragma unroll
      for (int i2 = 0; i2 < WMT; ++i2) {
#pragma unroll
        for (int j = 0; j < NT; ++j)
          v[r][i2][j] = (live && n0 + j * 8 < p.N) ? __ldcg(src + (i2 * NT + j) * 32) : make_double2(0.0, 0.0);
        vx[r][i2] = 0.0;
        if constexpr (XC == 1)
          if (live)
            vx[r][i2] = __ldcg(p.partials + sl * FRAG + CW * WMT * NT * 64 + warp * WMT * 32 + lane + i2 * 32);
      }
    }
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      if (sg0 + r >= nseg) break;
#pragma unroll
      for (int i2 = 0; i2 < WMT; ++i2) {
        xacc[i2] += vx[r][i2];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          acc[i2][j][0] += v[r][i2][j].x;
          acc[i2][j][1] += v[r][i2][j].y;
        }
      }
    }
  }
#pragma unroll
  for (int i2 = 0; i2 < WMT; ++i2) {
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t m = m0 + wm0 + i2 * 8 + r8, n = n0 + j * 8 + 2 * c4 + e;
        if (m < p.M && n < p.N) p.C[n * p.ldc + m] = acc[i2][j][e];
      }
    if constexpr (XC == 1) {
      const int64_t m = m0 + wm0 + i2 * 8 + r8, n = n0 + NT * 8;
      if (c4 == 0 && m < p.M && n < p.N) p.C[n * p.ldc + m] = xacc[i2];
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

}  // namespace

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

ProfScope::ProfScope(Handle& hh, int kind, double flops, double bytes) : h(hh) {
  if (!h.prof) return;
  on = true;
  for (int i = 0; i < 2; ++i) {
    cudaEvent_t e;
    if (h.prof_pool.empty()) {
      RSVD_CUDA(cudaEventCreate(&e));
    } else {
      e = h.prof_pool.back();
      h.prof_pool.pop_back();
    }
    (i == 0 ? rec.a : rec.b) = e;
  }
  rec.kind = kind;
  rec.flops = flops;
  rec.bytes = bytes;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  RSVD_CUDA(cudaStreamIsCapturing(h.stream, &cap));
  // under capture the event must be an external event-record node to be timeable
  flags = (cap == cudaStreamCaptureStatusActive) ? cudaEventRecordExternal : cudaEventRecordDefault;
  RSVD_CUDA(cudaEventRecordWithFlags(rec.a, h.stream, flags));
}

void ProfScope::end() {
  if (!on) return;
  on = false;
  RSVD_CUDA(cudaEventRecordWithFlags(rec.b, h.stream, flags));
  h.prof_pending.push_back(rec);
}

// Copy into an aligned, even-ld workspace when TMA cannot address x directly.
DMat tma_view(Handle& h, const DMat& x) {
  if (tma_ok(x)) return x;
  DMat y = h.ws.mat(x.rows, x.cols);
  RSVD_CUDA(cudaMemcpy2DAsync(y.p, y.ld * 8, x.p, x.ld * 8, x.rows * 8, x.cols,
                              cudaMemcpyDeviceToDevice, h.stream));
  return y;
}

bool tma_ok(const DMat& x) {
  return (reinterpret_cast<uintptr_t>(x.p) % 16 == 0) && (x.ld % 2 == 0) && x.ld >= x.rows;
}

namespace {

// RSVD_PROBE_PASS: per-CTA %globaltimer stamps of one launch (debug):
// entry, first stage arrival, per segment (main loop end, ticket, epilogue
// end), exit; printed as percentiles over the CTAs, in microseconds.
void probe_report(Handle& h, const unsigned long long* dprobe, int64_t nct, int64_t M, int64_t N,
                  int64_t K, int stream_k) {
  std::vector<unsigned long long> v(size_t(nct) * 16);
  RSVD_CUDA(cudaMemcpyAsync(v.data(), dprobe, v.size() * 8, cudaMemcpyDeviceToHost, h.stream));
  stream_sync(h);
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int64_t c = 0; c < nct; ++c) {
    t0 = std::min(t0, v[size_t(c) * 16]);
    t1 = std::max(t1, v[size_t(c) * 16 + 15]);
  }
  std::vector<double> entry, first, loop0, tick, red_last, red_other, exitv;
  for (int64_t c = 0; c < nct; ++c) {
    const unsigned long long* r = &v[size_t(c) * 16];
    entry.push_back((r[0] - t0) * 1e-3);
    first.push_back((r[1] - r[0]) * 1e-3);
    exitv.push_back((r[15] - t0) * 1e-3);
    for (int sg = 0; sg < 4; ++sg) {
      const unsigned long long le = r[2 + 3 * sg], tk = r[3 + 3 * sg], ee = r[4 + 3 * sg];
      if (!le) break;
      if (sg == 0) loop0.push_back((le - r[1]) * 1e-3);
      if (tk) {
        tick.push_back(((tk & ~1ull) - le) * 1e-3);
        ((tk & 1ull) ? red_last : red_other).push_back((ee - (tk & ~1ull)) * 1e-3);
      }
    }
  }
  auto pct = [](std::vector<double> x) {
    if (x.empty()) return std::string("-");
    std::sort(x.begin(), x.end());
    char b[96];
    std::snprintf(b, sizeof b, "%.2f/%.2f/%.2f", x[x.size() / 10], x[x.size() / 2], x.back());
    return std::string(b);
  };
  std::fprintf(stderr,
               "pass M=%lld N=%lld K=%lld ctas=%lld sk=%d span %.2f us | entry %s | first-data %s | "
               "loop0 %s | ticket %s | reduce(last) %s n=%zu | epi(other) %s | exit %s  (p10/p50/max)\n",
               (long long)M, (long long)N, (long long)K, (long long)nct, stream_k, (t1 - t0) * 1e-3,
               pct(entry).c_str(), pct(first).c_str(), pct(loop0).c_str(), pct(tick).c_str(),
               pct(red_last).c_str(), red_last.size(), pct(red_other).c_str(), pct(exitv).c_str());
}

template <bool kNN, int BN, int WMT, int BK, int STAGES, int XC = 0, int CW = 8>
void launch(Handle& h, const DMat& P, const DMat& R, DMat C, int64_t M, int64_t N, int64_t K,
            int force_splits) {
  using Cfg = PassCfg<kNN, BN, WMT, BK, STAGES, XC, CW>;
  auto kern1 = pass_kernel<kNN, BN, WMT, BK, STAGES, XC, CW, false>;
  auto kernG = pass_kernel<kNN, BN, WMT, BK, STAGES, XC, CW, true>;
  smem_attr(kern1, Cfg::SMEM);
  smem_attr(kernG, Cfg::SMEM);
  const int64_t mt = ceil_div(M, Cfg::BM), nt = ceil_div(N, Cfg::NCOL);
  const int64_t tiles = mt * nt;
  const int64_t kblocks = ceil_div(K, BK);
  constexpr int64_t FRAG = Cfg::FRAG;
  PassParams pp{};
  pp.M = M;
  pp.N = N;
  pp.K = K;
  pp.mt = int(mt);
  pp.nt = int(nt);
  pp.kb_tile = int(kblocks);
  pp.C = C.p;
  pp.ldc = C.ld;
  // resident CTAs per SM for this instantiation (2 for the CW <= 4 configs)
  static int occ = 0;
  if (occ == 0) {
    RSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern1, Cfg::THREADS, Cfg::SMEM));
    occ = std::max(1, occ);
  }
  const int sms = h.sm_count * occ;
  dim3 grid;
  // Few tiles (C1/C2 passes, Gram products): stream-K over all SMs.  Many
  // tiles: split-K grid with n-tiles adjacent for L2 reuse of A.
  const bool stream_k = force_splits <= 0 && tiles < 2 * sms;
  bool split_tiles = false;
  if (stream_k) {
    // n-tiles of one m-tile go to nt adjacent CTAs walking the same unit range
    // (A read once from DRAM; measured 2.44x the algorithmic bytes on C3's
    // adjoint when one CTA swept the n-tiles one after the other)
    const int64_t nsub = (nt > 1 && nt <= sms) ? nt : 1;
    const int64_t units = (tiles / nsub) * kblocks;
    // one CTA per tile at least (short-K products: no partials at all), and
    // >= 4 K slices per CTA when tiles are few (bounds the partials a tile's
    // last segment must reduce)
    static const int64_t min_slices = [] {
      const char* e = std::getenv("RSVD_SK_MIN_SLICES");
      return int64_t(e ? std::max(1, std::atoi(e)) : 4);
    }();
    const int64_t g = std::max<int64_t>(
        1, std::min<int64_t>(sms / nsub, std::max<int64_t>(tiles / nsub, units / min_slices)));
    pp.stream_k = 1;
    pp.nsub = int(nsub);
    pp.units = units;
    pp.grid = int(g);
    pp.max_seg = int(ceil_div(ceil_div(units, g), kblocks) + 1);
    pp.splits = 1;
    pp.kb_split = int(kblocks);
    pp.partials = h.ws.alloc(g * nsub * pp.max_seg * FRAG);
    // partial tiles are summed by sk_reduce_kernel after the pass
    // (RSVD_SK_INKERNEL=1: the last-arriving CTA sums them, ticket per tile)
    static const bool inkernel = std::getenv("RSVD_SK_INKERNEL") != nullptr;
    pp.defer = inkernel ? 0 : 1;
    if (!pp.defer) pp.counters = tile_counters(h, tiles);
    // any tile covered by more than one CTA (group)?  (host copy of sk_cta_of)
    auto begin_of = [&](int64_t c) { return (c * units) / g; };
    auto cta_of = [&](int64_t u) {
      int64_t c = (u * g) / units;
      while (c + 1 < g && begin_of(c + 1) <= u) ++c;
      while (c > 0 && begin_of(c) > u) --c;
      return c;
    };
    for (int64_t tg = 0; tg < tiles / nsub && !split_tiles; ++tg)
      split_tiles = cta_of(tg * kblocks) != cta_of((tg + 1) * kblocks - 1);
    grid = dim3(unsigned(g * nsub), 1, 1);
  } else {
    int splits = 1;
    if (force_splits > 0) {
      splits = force_splits;
    } else {
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
    const int64_t kps = ceil_div(kblocks, splits);
    splits = int(ceil_div(kblocks, kps));
    pp.stream_k = 0;
    pp.splits = splits;
    pp.kb_split = int(kps);
    if (splits > 1) {
      pp.partials = h.ws.alloc(tiles * splits * FRAG);
      pp.counters = tile_counters(h, tiles);
    }
    grid = dim3(unsigned(nt), unsigned(mt), unsigned(splits));
  }
  CUtensorMap ta = kNN ? make_map(P.p, P.rows, P.cols, P.ld, 16, BK)
                       : make_map(P.p, P.rows, P.cols, P.ld, 16, Cfg::BM);
  CUtensorMap tb = make_map(R.p, R.rows, R.cols, R.ld, 16, BN);
  // kinds: 0 = apply pass over A (A X), 1 = adjoint pass (A^T Y), 2 = other
  // skinny products (the lift Q U_B): the streamed operand is A exactly when
  // both of its dimensions dwarf the skinny one
  ProfScope prof(h, (std::min(M, K) > 2 * N) ? (kNN ? 0 : 1) : 2, 2.0 * double(M) * double(N) * double(K),
                 8.0 * (double(M) * K + double(K) * N + double(M) * N));
  static const bool probe_pass = std::getenv("RSVD_PROBE_PASS") != nullptr;
  const int64_t nct = int64_t(grid.x) * grid.y * grid.z;
  if (probe_pass) {
    pp.probe = reinterpret_cast<unsigned long long*>(h.ws.alloc_bytes(size_t(nct) * 16 * 8));
    RSVD_CUDA(cudaMemsetAsync(pp.probe, 0, size_t(nct) * 16 * 8, h.stream));
  }
  if (pp.stream_k && pp.nsub > 1)
    launch_k(h, kernG, grid, Cfg::THREADS, Cfg::SMEM, ta, tb, pp);
  else
    launch_k(h, kern1, grid, Cfg::THREADS, Cfg::SMEM, ta, tb, pp);
  RSVD_LAUNCHED(h);
  if (pp.stream_k && pp.defer && split_tiles) {
    if (pp.nsub > 1)
      launch_k(h, sk_reduce_kernel<kNN, BN, WMT, BK, STAGES, XC, CW, true>, unsigned(tiles), CW * 32, 0, pp);
    else
      launch_k(h, sk_reduce_kernel<kNN, BN, WMT, BK, STAGES, XC, CW, false>, unsigned(tiles), CW * 32, 0, pp);
    RSVD_LAUNCHED(h);
  }
  if (probe_pass) probe_report(h, pp.probe, nct, M, N, K, pp.stream_k);
  prof.end();
}


// Kernel-variant override for tuning experiments (tools/pass_sweep.py); 0 = default.
// Measured on C2 (l = 25), all within 0-9 % slower than the default: BM 256
// (WMT 4), BK 16 x 6 stages, 4 or 6 consumer warps with WMT 4, BK 32 x 4
// stages; a math-free copy of the same TMA load path streams A at 6.4 TB/s
// (tools/microbench/tma_stream.cu), so the pass is bound by the overlap of
// DMMA issue with the 3-stage ring, not by the TMA boxes.
int env_variant(const char* name) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : 0;
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
  static const int v25 = env_variant("RSVD_PASS25_NN");
  static const int vbig = env_variant("RSVD_PASSBIG");
  // N == 25 (C1 / C2): 4 consumer warps, BM 64, two CTAs per SM (two
  // independent TMA rings per SM): C2 passes 124.2 us vs 126.6 us for one
  // 8-warp CTA (BM 128), 926 vs 915 factorizations/s.  BK = 48, 3 stages
  // (measured ~2 % faster than BK = 32 for NN).
  if (N == 25) {
    switch (v25) {
      case 1: launch<true, 32, 4, 32, 3, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 3: launch<true, 32, 4, 16, 6, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 4: launch<true, 32, 4, 32, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 5: launch<true, 32, 2, 32, 4, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 6: launch<true, 32, 4, 32, 3, 1, 6>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 7: launch<true, 32, 4, 48, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 8: launch<true, 32, 2, 32, 4, 1, 7>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 9: launch<true, 32, 2, 48, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 10: launch<true, 32, 2, 32, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 11: launch<true, 32, 1, 48, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 12: launch<true, 32, 2, 48, 3, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      default: launch<true, 32, 2, 48, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits);
    }
  } else if (N <= 32)
    launch<true, 32, 2, 32, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (N <= 64)
    launch<true, 64, 2, 32, 3>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (vbig == 1)
    launch<true, 56, 4, 16, 4, 0, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (vbig == 3 || (vbig == 0 && h.pass_cfg_big == 1))
    launch<true, 56, 4, 16, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else  // two CTAs per SM, BM 64: C3 7.06 -> 6.84 ms, C5-shape 34.8 -> 33.8 ms (apply)
    launch<true, 56, 2, 32, 3, 0, 4>(h, Pv, Rv, C, M, N, K, force_splits);
}

// ---------------------------------------------------------------- small Gram
// C (M x N) = P^T R for tall P (K x M), R (K x N) with M, N <= 64: the l x l
// inner products of the orthonormalization and single-pass cores (Q^T Q,
// Q^T Omega, Q^T Y).  A DMMA tile engine would waste >= 4/5 of its work on
// such outputs.  Each CTA stages one chunk of rows of P and R in shared memory
// with a single round of coalesced loads, forms its M x N partial with DFMA,
// and the last CTA to finish (one atomic ticket) sums the partials in CTA
// order with batched loads: bitwise deterministic, one level, one launch.

__global__ void __launch_bounds__(256) gram_small_kernel(
    const double* __restrict__ P, int64_t ldp, const double* __restrict__ R, int64_t ldr,
    int64_t K, int M, int N, int64_t rows_per_cta, double* __restrict__ part,
    int* __restrict__ counter, double* __restrict__ C, int64_t ldc) {
  RSVD_PDL_ENTRY();
  extern __shared__ double sh[];
  const int RP = int(rows_per_cta);
  double* Ps = sh;                   // [RP][M+1]
  double* Rs = sh + RP * (M + 1);    // [RP][N+1]
  __shared__ int last;
  const int tid = threadIdx.x;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int nr = int(K - r0 < rows_per_cta ? K - r0 : rows_per_cta);
  for (int e = tid; e < RP * M; e += 256) {
    const int r = e % RP, a = e / RP;
    Ps[r * (M + 1) + a] = r < nr ? P[int64_t(a) * ldp + r0 + r] : 0.0;
  }
  for (int e = tid; e < RP * N; e += 256) {
    const int r = e % RP, b = e / RP;
    Rs[r * (N + 1) + b] = r < nr ? R[int64_t(b) * ldr + r0 + r] : 0.0;
  }
  __syncthreads();
  const int MN = M * N;
  double* mine = part + int64_t(blockIdx.x) * MN;
  for (int o = tid; o < MN; o += 256) {
    const int a = o % M, b = o / M;
    double s0 = 0.0, s1 = 0.0;
    int r = 0;
    for (; r + 1 < nr; r += 2) {
      s0 = fma(Ps[r * (M + 1) + a], Rs[r * (N + 1) + b], s0);
      s1 = fma(Ps[(r + 1) * (M + 1) + a], Rs[(r + 1) * (N + 1) + b], s1);
    }
    if (r < nr) s0 = fma(Ps[r * (M + 1) + a], Rs[r * (N + 1) + b], s0);
    mine[o] = s0 + s1;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counter, 1) == int(gridDim.x) - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int G = gridDim.x;
  for (int o = tid; o < MN; o += 256) {
    double v = 0.0;
    int c = 0;
    for (; c + 8 <= G; c += 8) {
      double t[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) t[q] = __ldcg(part + int64_t(c + q) * MN + o);
#pragma unroll
      for (int q = 0; q < 8; ++q) v += t[q];
    }
    for (; c < G; ++c) v += __ldcg(part + int64_t(c) * MN + o);
    C[int64_t(o / M) * ldc + (o % M)] = v;
  }
  if (tid == 0) *counter = 0;
}

void gram_small(Handle& h, const DMat& P, const DMat& R, DMat C) {
  const int64_t K = P.rows;
  const int M = int(P.cols), N = int(R.cols);
  // rows per CTA: ~16 partials for the ordered final sum (its latency, not the
  // DFMA work, dominates these tiny products), at least 64 rows; smem-bounded
  int64_t rp = std::max<int64_t>(64, ceil_div(K, 16));
  const int64_t rp_max = (200 * 1024) / (8 * (M + N + 2));
  rp = std::min(rp, rp_max);
  const int64_t G = ceil_div(K, rp);
  double* part = h.ws.alloc(G * M * N);
  int* cnt = tile_counters(h, 1);
  const size_t smem = size_t(rp) * (M + N + 2) * 8;
  smem_attr(gram_small_kernel, smem);
  launch_k(h, gram_small_kernel, unsigned(G), 256, smem, P.p, P.ld, R.p, R.ld, K, M, N, rp, part,
                                                          cnt, C.p, C.ld);
  RSVD_LAUNCHED(h);
}

void gemm_tn(Handle& h, const DMat& P, const DMat& R, DMat C, int force_splits) {
  const int64_t K = P.rows, M = P.cols, N = R.cols;
  if (R.rows != K || C.rows != M || C.cols != N) throw_dim("gemm_tn: shape mismatch");
  if (M == 0 || N == 0) return;
  if (K == 0) {
    RSVD_CUDA(cudaMemset2DAsync(C.p, C.ld * 8, 0, M * 8, N, h.stream));
    return;
  }
  if (M <= 64 && N <= 64 && force_splits <= 0) {
    gram_small(h, P, R, C);
    return;
  }
  DMat Pv = tma_view(h, P), Rv = tma_view(h, R);
  static const int v25 = env_variant("RSVD_PASS25_TN");
  static const int vbig = env_variant("RSVD_PASSBIG");
  if (N == 25) {  // see gemm_nn
    switch (v25) {
      case 1: launch<false, 32, 4, 32, 3, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 3: launch<false, 32, 4, 16, 6, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 4: launch<false, 32, 4, 32, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 5: launch<false, 32, 2, 48, 3, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 6: launch<false, 32, 4, 32, 3, 1, 6>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 7: launch<false, 32, 4, 48, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 8: launch<false, 32, 2, 32, 4, 1, 7>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 9: launch<false, 32, 2, 32, 4, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 10: launch<false, 32, 2, 32, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 11: launch<false, 32, 1, 48, 3, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits); break;
      case 12: launch<false, 32, 2, 32, 4, 1>(h, Pv, Rv, C, M, N, K, force_splits); break;
      default: launch<false, 32, 2, 32, 4, 1, 4>(h, Pv, Rv, C, M, N, K, force_splits);
    }
  } else if (N <= 32)
    launch<false, 32, 2, 32, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (N <= 64)
    launch<false, 64, 2, 32, 3>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (vbig == 1)
    launch<false, 56, 4, 16, 4, 0, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else if (vbig == 3 || (vbig == 0 && h.pass_cfg_big == 1))
    launch<false, 56, 4, 16, 4>(h, Pv, Rv, C, M, N, K, force_splits);
  else  // two CTAs per SM, BM 64: C3 7.06 -> 6.84 ms, C5-shape 34.8 -> 33.8 ms (apply)
    launch<false, 56, 2, 32, 3, 0, 4>(h, Pv, Rv, C, M, N, K, force_splits);
}

}  // namespace rsvdb
