// Fused single pass of Algorithm 6 (reference spsvd_general,
// singlepass.hpp:119-122; "two sketches formed in one pass"):
//
//     Y = A * Omega_c   (M x L)          W = A^T * Psi   (K x L)
//
// from ONE traversal of A (M x K, column-major) -- each A tile comes from HBM
// once, and the host-buffer entry points can stream A in row panels into a
// single pass (capi.cu).
//
// B200 design.  A is cut into MB x MB macroblocks.  Every macroblock yields
// two kinds of work items of equal size:
//   * apply items  (A Omega_c): one BM-row strip of the macroblock times one
//     NCOL-wide column tile of Omega_c -> a partial Y tile over the
//     macroblock's K range;
//   * adjoint items (A^T Psi):  one BM-column strip of the macroblock times one
//     NCOL-wide column tile of Psi      -> a partial W tile over the
//     macroblock's row range.
// Items are numbered macroblock-major (row-major over macroblocks; inside a
// macroblock apply and adjoint strips alternate) and claimed in that order
// from a global counter by a persistent grid (SMs x resident CTAs).  All items of a macroblock run within
// ~2 waves, so the macroblock (MB^2 x 8 bytes, sized to L2) is read from HBM
// by whichever item touches a tile first and from L2 by the other one.
// The per-item main loop is the pass kernel's (pass.cu): one TMA producer
// warp feeding a 3-stage mbarrier ring with 128-byte-swizzled boxes, four
// DMMA consumer warps; the ring runs on across items, so the producer loads
// the next item while the consumers finish the current one.
// Partial tiles are accumulated IN PLACE in a fixed order: the contribution
// of macroblock column c to a Y tile (row r to a W tile) waits on the tile's
// semaphore until it equals c (r), adds itself to the tile (the first one
// stores), and releases c + 1.  Bitwise deterministic, no floating-point
// atomics, no partial buffers.  Progress: a contribution only waits on a
// LOWER item index, and every lower item has already been claimed by a
// co-resident CTA that is processing it (its own waits are on still lower
// items), so every wait chain ends.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "fused.cuh"
#include "pass.cuh"
#include "ptx.cuh"

namespace rsvdb {

namespace {

constexpr int kBN = 56;     // loaded Omega/Psi columns per tile (7 DMMA n-tiles)
constexpr int kWMT = 2;     // 8-row m-tiles per consumer warp
constexpr int kBK = 32;     // K slice per stage
constexpr int kStages = 3;
constexpr int kCW = 4;      // consumer warps
constexpr int kBM = kCW * kWMT * 8;  // 64 rows (apply) / A columns (adjoint) per item
constexpr int kNT = kBN / 8;
constexpr int kThreads = (kCW + 1) * 32;
constexpr int kABytes = kBM * kBK * 8;
constexpr int kBBytes = kBN * kBK * 8;
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kPipeBytes = kStages * kStageBytes;
constexpr int kItemSlots = 4;  // item ids handed from the producer to the consumers
constexpr int kSmem = kPipeBytes + 1024 + 2 * kStages * 8 + 2 * kItemSlots * 8 + kItemSlots * 8 + 16;
static_assert(kABytes % 1024 == 0 && kBBytes % 1024 == 0, "swizzle-128B alignment");

struct FusedParams {
  int64_t M, K, L;   // A is M x K (rows [row0, row_end) valid in this launch)
  int64_t row0, row_end;
  int MB;            // macroblock edge (multiple of kBM and kBK)
  int mbr, mbc;      // macroblocks in this launch: rows x columns
  int mb_row0;       // global macroblock row of this launch's first one
  int nt;            // column tiles of L
  int strips;        // MB / kBM
  int64_t items;     // mbr * mbc * 2 * strips * nt
  double* Y;
  int64_t ldy;
  double* W;
  int64_t ldw;
  int* semY;         // per Y tile: next macroblock column to add
  int* semW;         // per W tile: next global macroblock row to add
  unsigned long long* next_item;  // dynamic work counter (zeroed per launch)
};

struct Item {
  bool valid;
  bool adj;          // adjoint (W) item
  int64_t m0;        // output row (Y row / W row = A column)
  int64_t k0;        // first K index (A column for apply, A row for adjoint)
  int nkb;           // K slices
  int n0;            // output column
  int idx;           // contribution index (semaphore value to wait for)
  int* sem;
};

__device__ __forceinline__ Item decode(const FusedParams& p, int64_t x) {
  Item it;
  const int64_t per_mb = int64_t(2) * p.strips * p.nt;
  const int64_t mb = x / per_mb;
  const int k = int(x % per_mb);
  const int rl = int(mb / p.mbc), cb = int(mb % p.mbc);
  const int strip = k / (2 * p.nt);
  it.adj = ((k / p.nt) & 1) != 0;
  const int q = k % p.nt;
  it.n0 = q * kBN;
  const int rg = p.mb_row0 + rl;  // global macroblock row
  const int64_t r_lo = int64_t(rg) * p.MB;
  const int64_t r_hi = min(r_lo + p.MB, p.row_end);
  const int64_t c_lo = int64_t(cb) * p.MB;
  const int64_t c_hi = min(c_lo + p.MB, p.K);
  if (!it.adj) {
    it.m0 = r_lo + int64_t(strip) * kBM;
    it.valid = it.m0 < r_hi;
    it.k0 = c_lo;
    it.nkb = int((c_hi - c_lo + kBK - 1) / kBK);
    it.idx = cb;
    it.sem = p.semY + (it.m0 / kBM) * p.nt + q;
  } else {
    it.m0 = c_lo + int64_t(strip) * kBM;
    it.valid = it.m0 < c_hi;
    it.k0 = r_lo;
    it.nkb = int((r_hi - r_lo + kBK - 1) / kBK);
    it.idx = rg;
    it.sem = p.semW + (it.m0 / kBM) * p.nt + q;
  }
  return it;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One BK slice of DMMA on a stage (the pass kernel's fragment scheme, XC = 0).
template <bool kNN>
__device__ __forceinline__ void stage_mma(const uint8_t* a_st, const uint8_t* b_st, int offA0,
                                          int offB0, double (&acc)[kWMT][kNT][2]) {
#pragma unroll
  for (int ks = 0; ks < kBK / 4; ++ks) {
    constexpr int kT[4] = {0, 1, 4, 5};
    const int t = kT[ks & 3], kb16 = ks >> 2;
    const int cB = ((t >> 1) << 4) | ((t & 1) << 3);
    double af[kWMT], bf[kNT];
    if constexpr (kNN) {
#pragma unroll
      for (int i2 = 0; i2 < kWMT; ++i2) {
        const int cA = (t << 7) | (((4 * (i2 & 1)) ^ t) << 4);
        af[i2] = *reinterpret_cast<const double*>(a_st + (offA0 ^ cA) + (i2 >> 1) * (kBK * 128) +
                                                  kb16 * 2048);
      }
    } else {
#pragma unroll
      for (int i2 = 0; i2 < kWMT; ++i2)
        af[i2] = *reinterpret_cast<const double*>(a_st + (offA0 ^ cB) + kb16 * (kBM * 128) +
                                                  i2 * 1024);
    }
#pragma unroll
    for (int j = 0; j < kNT; ++j)
      bf[j] = *reinterpret_cast<const double*>(b_st + (offB0 ^ cB) + kb16 * (kBN * 128) + j * 1024);
#pragma unroll
    for (int i2 = 0; i2 < kWMT; ++i2)
#pragma unroll
      for (int j = 0; j < kNT; ++j) ptx::dmma(acc[i2][j][0], acc[i2][j][1], af[i2], bf[j]);
  }
}

__global__ void __launch_bounds__(kThreads, 2)
    fused_pass_kernel(const __grid_constant__ CUtensorMap tmA_nn,
                      const __grid_constant__ CUtensorMap tmA_tn,
                      const __grid_constant__ CUtensorMap tmOc,
                      const __grid_constant__ CUtensorMap tmPsi, FusedParams p) {
  RSVD_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPipeBytes);
  uint64_t* empty = full + kStages;
  uint64_t* ifull = empty + kStages;      // item-slot ring
  uint64_t* iempty = ifull + kItemSlots;
  int64_t* islot = reinterpret_cast<int64_t*>(iempty + kItemSlots);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kCW);
    }
    for (int s = 0; s < kItemSlots; ++s) {
      ptx::mbar_init(&ifull[s], 1);
      ptx::mbar_init(&iempty[s], kCW);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // Dynamic schedule: the producer claims items in increasing order from a
  // global counter (a faster CTA takes more items, so no CTA's lag can hold
  // the in-order accumulation chains back) and hands each id to the
  // consumers through a small mbarrier ring; -1 ends the CTA.

  if (warp == kCW) {
    // ------------------------------------------------ TMA producer warp
    if (lane == 0) {
      ptx::prefetch_tmap(&tmA_nn);
      ptx::prefetch_tmap(&tmA_tn);
      ptx::prefetch_tmap(&tmOc);
      ptx::prefetch_tmap(&tmPsi);
      const uint64_t pol_b = ptx::policy_evict_last();
      uint64_t pol_a;  // A tiles are read twice (apply + adjoint item): keep them normal
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_a));
      int64_t i = 0;  // ring position, continuous across items
      for (int64_t j = 0;; ++j) {
        int64_t x = int64_t(atomicAdd(p.next_item, 1ull));
        if (x >= p.items) x = -1;
        const int sl = int(j % kItemSlots);
        if (j >= kItemSlots) ptx::mbar_wait(&iempty[sl], int((j / kItemSlots) - 1) & 1);
        islot[sl] = x;
        ptx::mbar_arrive(&ifull[sl]);  // release: the id store is ordered before it
        if (x < 0) break;
        const Item it = decode(p, x);
        if (!it.valid) continue;
        for (int kb = 0; kb < it.nkb; ++kb, ++i) {
          const int s = int(i % kStages);
          if (i >= kStages) ptx::mbar_wait(&empty[s], int((i / kStages) - 1) & 1);
          uint8_t* a_st = smem + s * kStageBytes;
          uint8_t* b_st = a_st + kABytes;
          ptx::mbar_expect_tx(&full[s], kStageBytes);
          const int k0 = int(it.k0) + kb * kBK;
          if (!it.adj) {
#pragma unroll
            for (int b = 0; b < kBM / 16; ++b)
              ptx::tma_load_2d(a_st + b * (kBK * 128), &tmA_nn, &full[s], int(it.m0) + 16 * b, k0,
                               pol_a);
#pragma unroll
            for (int hh = 0; hh < kBK / 16; ++hh)
              ptx::tma_load_2d(b_st + hh * (kBN * 128), &tmOc, &full[s], k0 + 16 * hh, it.n0, pol_b);
          } else {
#pragma unroll
            for (int hh = 0; hh < kBK / 16; ++hh)
              ptx::tma_load_2d(a_st + hh * (kBM * 128), &tmA_tn, &full[s], k0 + 16 * hh, int(it.m0),
                               pol_a);
#pragma unroll
            for (int hh = 0; hh < kBK / 16; ++hh)
              ptx::tma_load_2d(b_st + hh * (kBN * 128), &tmPsi, &full[s], k0 + 16 * hh, it.n0,
                               pol_b);
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------- DMMA consumer warps
  const int r8 = lane >> 2, c4 = lane & 3;
  const int wm0 = warp * kWMT * 8;
  const int tid = threadIdx.x;
  constexpr int NCT = kCW * 32;
  const int kbase = (c4 == 0) ? 0 : (c4 == 1) ? 3 : (c4 == 2) ? 12 : 15;
  const int offA_nn = (wm0 >> 4) * (kBK * 128) + kbase * 128 +
                      (((((wm0 >> 3) & 1) << 2 | (r8 >> 1)) ^ (kbase & 7)) << 4) + (r8 & 1) * 8;
  const int offA_tn = wm0 * 128 + r8 * 128 + (((kbase >> 1) ^ r8) << 4) + (kbase & 1) * 8;
  const int offB0 = r8 * 128 + (((kbase >> 1) ^ r8) << 4) + (kbase & 1) * 8;
  int64_t i = 0;
  for (int64_t j = 0;; ++j) {
    const int sl = int(j % kItemSlots);
    ptx::mbar_wait(&ifull[sl], int(j / kItemSlots) & 1);
    const int64_t x = islot[sl];
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&iempty[sl]);
    if (x < 0) break;
    const Item it = decode(p, x);
    if (!it.valid) continue;
    double acc[kWMT][kNT][2];
#pragma unroll
    for (int a = 0; a < kWMT; ++a)
#pragma unroll
      for (int j = 0; j < kNT; ++j) acc[a][j][0] = acc[a][j][1] = 0.0;
    // The tile's earlier sum is re-read in the epilogue: when its predecessor
    // has already released it (the usual case: it ran ~2 waves earlier), pull
    // its lines into L2 now, so the epilogue's read-modify-write does not pay
    // an HBM round trip.  (A non-blocking peek; prefetches only.)
    const bool released = it.idx == 0 || ld_acquire(it.sem) == it.idx;  // this thread's acquire
    if (it.idx > 0 && released) {
      double* C = it.adj ? p.W : p.Y;
      const int64_t ldc = it.adj ? p.ldw : p.ldy;
      const int64_t mlim = it.adj ? p.K : p.row_end;
      // kBN columns x 4 lines of 128 B (64 rows) per column
      for (int ln = tid; ln < kBN * 4; ln += NCT) {
        const int64_t n = it.n0 + ln / 4, m = it.m0 + 16 * (ln % 4);
        if (n < p.L && m < mlim)
          asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(C + n * ldc + m));
      }
    }
    for (int kb = 0; kb < it.nkb; ++kb, ++i) {
      const int s = int(i % kStages);
      ptx::mbar_wait(&full[s], int(i / kStages) & 1);
      const uint8_t* a_st = smem + s * kStageBytes;
      const uint8_t* b_st = a_st + kABytes;
      if (!it.adj)
        stage_mma<true>(a_st, b_st, offA_nn, offB0, acc);
      else
        stage_mma<false>(a_st, b_st, offA_tn, offB0, acc);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }
    // ordered in-place accumulation into the output tile: every thread
    // acquires the predecessor's release itself (usually already there), so
    // no barrier precedes the read-modify-write
    if (!released) {
      const long long t0 = clock64();
      while (ld_acquire(it.sem) != it.idx) {
        __nanosleep(64);
        if (clock64() - t0 > (40LL << 30)) __trap();  // a schedule bug traps, never hangs
      }
    }
    double* C = it.adj ? p.W : p.Y;
    const int64_t ldc = it.adj ? p.ldw : p.ldy;
    const int64_t mlim = it.adj ? p.K : p.row_end;
    // all of the tile's earlier sum is loaded before any store (one L2 round
    // trip; interleaved load-add-store would serialize 28 of them: the
    // stores may alias later loads as far as the compiler knows)
    if (it.idx > 0) {
      double old[kWMT][kNT][2];
#pragma unroll
      for (int a = 0; a < kWMT; ++a) {
        const int64_t m = it.m0 + wm0 + a * 8 + r8;
#pragma unroll
        for (int j = 0; j < kNT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t n = it.n0 + j * 8 + 2 * c4 + e;
            old[a][j][e] = (m < mlim && n < p.L) ? __ldcg(C + n * ldc + m) : 0.0;
          }
      }
#pragma unroll
      for (int a = 0; a < kWMT; ++a)
#pragma unroll
        for (int j = 0; j < kNT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) acc[a][j][e] = old[a][j][e] + acc[a][j][e];
    }
#pragma unroll
    for (int a = 0; a < kWMT; ++a) {
      const int64_t m = it.m0 + wm0 + a * 8 + r8;
      if (m >= mlim) continue;
#pragma unroll
      for (int j = 0; j < kNT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t n = it.n0 + j * 8 + 2 * c4 + e;
          if (n < p.L) C[n * ldc + m] = acc[a][j][e];
        }
    }
    // every consumer's stores happen-before thread 0's release (bar.sync
    // orders them; st.release is cumulative): no separate fence
    ptx::named_bar(1, NCT);
    if (tid == 0) st_release(it.sem, it.idx + 1);
  }
}

}  // namespace

int fused_macroblock(const Handle& h) {
  static const int env = [] {
    const char* e = std::getenv("RSVD_FUSED_MB");
    return e ? std::atoi(e) : 0;
  }();
  const int v = h.fused_mb > 0 ? h.fused_mb : (env > 0 ? env : 2048);
  return std::max(kBM, (v / kBM) * kBM);
}

void fused_dual_pass(Handle& h, const DMat& A, const DMat& Oc, const DMat& Psi, DMat Y, DMat W,
                     int64_t row0, int64_t row_end, int* sem, bool first) {
  const int64_t M = A.rows, K = A.cols, L = Oc.cols;
  if (Oc.rows != K || Psi.rows != M || Psi.cols != L || Y.rows != M || Y.cols != L ||
      W.rows != K || W.cols != L)
    throw_dim("fused_dual_pass: shape mismatch");
  if (!tma_ok(A) || !tma_ok(Oc) || !tma_ok(Psi)) throw_dim("fused_dual_pass: operand not TMA-addressable");
  const int MB = fused_macroblock(h);
  if (row0 % MB != 0 || row_end <= row0 || row_end > M) throw_dim("fused_dual_pass: bad row panel");
  FusedParams p{};
  p.M = M;
  p.K = K;
  p.L = L;
  p.row0 = row0;
  p.row_end = row_end;
  p.MB = MB;
  p.mbr = int(ceil_div(row_end - row0, MB));
  p.mbc = int(ceil_div(K, MB));
  p.mb_row0 = int(row0 / MB);
  p.nt = int(ceil_div(L, kBN));
  p.strips = MB / kBM;
  p.items = int64_t(p.mbr) * p.mbc * 2 * p.strips * p.nt;
  p.Y = Y.p;
  p.ldy = Y.ld;
  p.W = W.p;
  p.ldw = W.ld;
  const int64_t ny = ceil_div(M, kBM) * p.nt, nw = ceil_div(K, kBM) * p.nt;
  p.semY = sem;
  p.semW = sem + ny;
  // the work counter sits after the semaphores (8-byte aligned), reset per launch
  p.next_item = reinterpret_cast<unsigned long long*>(sem + ((ny + nw + 1) & ~int64_t(1)));
  if (first) RSVD_CUDA(cudaMemsetAsync(sem, 0, size_t(ny + nw) * sizeof(int), h.stream));
  RSVD_CUDA(cudaMemsetAsync(p.next_item, 0, 8, h.stream));
  smem_attr(fused_pass_kernel, kSmem);
  static int occ = 0;
  if (occ == 0) {
    RSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_pass_kernel, kThreads, kSmem));
    occ = std::max(1, occ);
  }
  // co-resident persistent grid (required: see the progress argument above)
  const int64_t grid = std::min<int64_t>(int64_t(h.sm_count) * occ, p.items);
  const CUtensorMap ta_nn = make_map(A.p, A.rows, A.cols, A.ld, 16, kBK);
  const CUtensorMap ta_tn = make_map(A.p, A.rows, A.cols, A.ld, 16, kBM);
  const CUtensorMap tb_oc = make_map(Oc.p, Oc.rows, Oc.cols, Oc.ld, 16, kBN);
  const CUtensorMap tb_ps = make_map(Psi.p, Psi.rows, Psi.cols, Psi.ld, 16, kBN);
  // algorithmic work of this panel (SURVEY 8(d) "fused Alg 6"): 4 m K L flops,
  // 8 (m K + K L + m L + m L + K L) bytes for its m = row_end - row0 rows
  const double mr = double(row_end - row0);
  ProfScope prof(h, 3, 4.0 * mr * double(K) * double(L),
                 8.0 * (mr * double(K) + 2.0 * double(K) * double(L) + 2.0 * mr * double(L)));
  launch_k(h, fused_pass_kernel, unsigned(grid), kThreads, kSmem, ta_nn, ta_tn, tb_oc, tb_ps, p);
  RSVD_LAUNCHED(h);
  prof.end();
}

int64_t fused_semaphores(int64_t M, int64_t K, int64_t L) {
  const int64_t nt = ceil_div(L, kBN);
  return (ceil_div(M, kBM) + ceil_div(K, kBM)) * nt + 4;  // + the work counter
}

}  // namespace rsvdb
