// On-device Gaussian test matrices reproducing the reference's seeded stream.
//
// Reference: gaussian(n, l, rng) (sketch.hpp:48-59) fills column-major with
// Rng::normal() (sketch.hpp:27) = std::normal_distribution<double> over
// std::mt19937_64:
//   * mt19937_64: 312-word state, lazy regeneration (_M_gen_rand) when the
//     index reaches 312, tempering on output (libstdc++ random.tcc);
//   * generate_canonical<double,53>: u = RN((double)x) / 2^64, clamped below 1
//     (libstdc++ random.tcc:3346-3381);
//   * Marsaglia polar (libstdc++ random.tcc:1810-1843): x = 2u-1, y = 2u'-1,
//     r2 = x*x + y*y (no FMA), reject r2 > 1 or r2 == 0, mult =
//     sqrt(-2 log r2 / r2), return y*mult and CACHE x*mult for the next call.
//
// Device pipeline (all exact integer / correctly rounded IEEE arithmetic,
// except log, see ddlog.cuh and "Exact mode" below):
//   1. mt_blocks: regenerate the untempered MT word sequence past the current
//      position (twist = two 156-wide parallel phases per 312 words).
//   2. polar_count: accept flags of every attempt (pair of draws), per-tile
//      counts; scan_counts: exclusive prefix over tiles.
//   3. polar_write: ranks inside each tile by ballot/popc; accepted attempt of
//      rank a writes normals 2a and 2a+1 of the output stream (column-major
//      placement), the attempt that completes the stream records how many
//      draws were consumed and the cached second variate.
//   4. rng_finish: the new MT state (312 words of the block holding the last
//      consumed draw + index, libstdc++'s lazy convention) and the cache.
// The host Rng state is passed in and returned advanced by exactly the draws
// consumed, so a host rsvd::Rng continues bit-identically.
//
// Exact mode (default; RSVD_OMEGA_EXACT=0 turns it off): the device log is
// correctly rounded, glibc's is not, so the two differ on ~0.08 % of polar
// inputs -- always ones whose exact log lies within ~0.02 ulp of a rounding
// midpoint (ddlog.cuh log_near_midpoint; ~1.7 % of inputs fall inside the
// window).  polar_write appends every such accepted pair (stream index, r2, x,
// y) to a pinned, device-mapped list; the host evaluates libstdc++'s
// multiplier sqrt(-2 * std::log(r2) / r2) with the HOST's own glibc log (a
// spinning worker pool for long lists); polar_patch rewrites those normals
// (and the cached variate).  An eager call reads the list's length and
// answers it synchronously before queueing polar_patch.  A CUDA-graph-captured
// call cannot wait mid-graph: there patch_signal publishes the length in the
// list's header, polar_patch spins on the header's release flag, and the host
// thread answers the list right after the graph launch (finish_call); a
// replay re-arms the same headers.  No host node in either form.  The result is the reference's stream
// bit for bit on the host that runs it, whichever glibc ifunc (FMA or SSE2)
// that host selects.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "ddlog.cuh"
#include "mtjump.h"
#include "rng.cuh"
#include "small.cuh"

namespace rsvdb {

__constant__ ddlog::Entry c_log_table[ddlog::kTableSize];

namespace {

constexpr uint64_t kMatA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x000000007FFFFFFFULL;
constexpr int kN = 312, kM = 156;

__device__ __forceinline__ uint64_t twist(uint64_t xk, uint64_t xk1) {
  const uint64_t y = (xk & kUpper) | (xk1 & kLower);
  return (y >> 1) ^ ((y & 1ULL) ? kMatA : 0ULL);
}
__device__ __forceinline__ uint64_t temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}
// generate_canonical<double, 53> for a 64-bit engine.
__device__ __forceinline__ double canonical(uint64_t z) {
  double u = __ull2double_rn(z) * 0x1p-64;
  if (u >= 1.0) u = 0x1.fffffffffffffp-1;  // nextafter(1, 0)
  return u;
}
struct Pair {
  double x, y, r2;
  bool ok;
};
__device__ __forceinline__ Pair polar_pair(uint64_t w1, uint64_t w2) {
  Pair p;
  p.x = __dsub_rn(__dmul_rn(2.0, canonical(temper(w1))), 1.0);
  p.y = __dsub_rn(__dmul_rn(2.0, canonical(temper(w2))), 1.0);
  p.r2 = __dadd_rn(__dmul_rn(p.x, p.x), __dmul_rn(p.y, p.y));
  p.ok = !(p.r2 > 1.0 || p.r2 == 0.0);
  return p;
}
__device__ __forceinline__ double polar_mult_from_log(double r2, double lg) {
  return __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, lg), r2));
}

// 1. block generator (one CTA).  out[0..312) = initial block.  The libstdc++
// twist regenerates block N from block C in place; unrolling its in-place
// dependency (N[j] for j >= 156 reads N[j-156]) expresses every word of N in
// terms of C alone:
//   j <  156: N[j]   = C[j+156] ^ g(C[j], C[j+1])
//   j <  311: N[j]   = C[j] ^ g(C[j-156], C[j-155]) ^ g(C[j], C[j+1])
//   j == 311: N[311] = C[311] ^ g(C[155], C[156]) ^ g(C[311], C[156] ^ g(C[0], C[1]))
// so a whole 312-word block costs one barrier.
__global__ void mt_blocks_kernel(const uint64_t* __restrict__ init, int64_t nb,
                                 uint64_t* __restrict__ out) {
  RSVD_PDL_ENTRY();
  __shared__ uint64_t S[2][kN];
  const int t = threadIdx.x;
  if (t < kN) {
    S[0][t] = init[t];
    out[t] = init[t];
  }
  __syncthreads();
  for (int64_t k = 1; k <= nb; ++k) {
    const uint64_t* c = S[(k - 1) & 1];
    uint64_t* n = S[k & 1];
    if (t < kN) {
      uint64_t v;
      if (t < kN - kM) {
        v = c[t + kM] ^ twist(c[t], c[t + 1]);
      } else if (t < kN - 1) {
        v = c[t] ^ twist(c[t - kM], c[t - kM + 1]) ^ twist(c[t], c[t + 1]);
      } else {
        const uint64_t n0 = c[kM] ^ twist(c[0], c[1]);
        v = c[kN - 1] ^ twist(c[kM - 1], c[kM]) ^ twist(c[kN - 1], n0);
      }
      n[t] = v;
      out[k * kN + t] = v;
    }
    __syncthreads();
  }
}

struct DevState {
  uint64_t mt[kN];
  uint64_t pos;
  int32_t has_cached, pad;
  double cached;
};

// ------------------------------------------------------- parallel stream
// Long streams are generated in segments of kSegWords words, all segments at
// once.  Segment s >= 1 starts from the 312-word window that precedes it,
// obtained by jump-ahead (mtjump.cpp): window[j] = XOR_{k in poly_s} base[k + j],
// base[i] = words[1 + i] (the first 19937 + 312 words, generated sequentially).
// Segment lengths (blocks of 312 words): short segments (more, cheaper jumps,
// short generation chains) up to ~9M words, long ones beyond.
constexpr int64_t kSegBlocksShort = 64;
constexpr int64_t kSegBlocksLong = 1024;
constexpr int kJumpBase = 19937 + kN;  // base words needed by a jump
constexpr int kPolyWords = 312;
constexpr int kSegPerCta = 3;          // segments advanced in lockstep per CTA

// grid (nseg - 1, parts): part p XORs the terms of poly words [w0, w1) into
// the window (XOR is order independent: exact and deterministic).
__global__ void __launch_bounds__(320) mt_jump_kernel(const uint64_t* __restrict__ words,
                                                      const uint64_t* __restrict__ polys,
                                                      int wpp,
                                                      unsigned long long* __restrict__ windows) {
  RSVD_PDL_ENTRY();
  extern __shared__ uint64_t base[];  // 64 * wpp + kN words
  __shared__ uint64_t poly[kPolyWords];
  const int t = threadIdx.x;
  const int s = blockIdx.x + 1;  // segment
  const int w0 = blockIdx.y * wpp, w1 = min(kPolyWords, w0 + wpp);
  if (w0 >= w1) return;
  const int nbase = 64 * (w1 - w0) + kN;
  for (int i = t; i < nbase; i += blockDim.x) {
    const int gi = 64 * w0 + i;
    base[i] = (gi < kJumpBase) ? words[1 + gi] : 0ULL;
  }
  for (int i = t; i < w1 - w0; i += blockDim.x) poly[i] = polys[int64_t(s - 1) * kPolyWords + w0 + i];
  __syncthreads();
  if (t >= kN) return;
  // Only the set bits of the (warp-uniform) polynomial words contribute.
  // Every bit position is tested independently (unrolled, warp-uniform
  // predicate on the load and XOR) into four accumulators: no dependency
  // chain between bits.  (A find-first-set / clear loop serialises ~4
  // dependent integer ops per set bit: measured 31 us for the C2 stream.)
  uint64_t acc[4] = {0, 0, 0, 0};
  for (int w = 0; w < w1 - w0; ++w) {
    const uint64_t bits = poly[w];
    const uint64_t* bw = base + 64 * w + t;
#pragma unroll
    for (int b = 0; b < 64; ++b)
      if ((bits >> b) & 1ull) acc[b & 3] ^= bw[b];
  }
  atomicXor(&windows[int64_t(s) * kN + t],
            static_cast<unsigned long long>((acc[0] ^ acc[1]) ^ (acc[2] ^ acc[3])));
}

// Segment s generates words [s*kSegWords, (s+1)*kSegWords) from its window
// (segment 0 from the initial block, which it also writes).
__global__ void __launch_bounds__(kSegPerCta * kN) mt_segments_kernel(
    const uint64_t* __restrict__ init, const uint64_t* __restrict__ windows, int64_t nseg,
    int64_t seg_blocks, uint64_t* __restrict__ words) {
  RSVD_PDL_ENTRY();
  const int64_t seg_words = seg_blocks * kN;
  __shared__ uint64_t S[kSegPerCta][2][kN];
  const int g = threadIdx.x / kN, t = threadIdx.x % kN;
  const int spc = int(blockDim.x) / kN;  // segments per CTA (1 .. kSegPerCta)
  const int64_t s = int64_t(blockIdx.x) * spc + g;
  const bool live = s < nseg;
  if (live) S[g][0][t] = (s == 0) ? init[t] : windows[s * kN + t];
  if (live && s == 0) words[t] = init[t];
  __syncthreads();
  const int64_t first = (s == 0) ? 1 : 0;  // segment 0's block 0 is the initial block
  for (int64_t k = 0; k < seg_blocks - first; ++k) {
    const uint64_t* c = S[g][k & 1];
    uint64_t* n = S[g][(k + 1) & 1];
    if (live) {
      uint64_t v;
      if (t < kN - kM) {
        v = c[t + kM] ^ twist(c[t], c[t + 1]);
      } else if (t < kN - 1) {
        v = c[t] ^ twist(c[t - kM], c[t - kM + 1]) ^ twist(c[t], c[t + 1]);
      } else {
        const uint64_t n0 = c[kM] ^ twist(c[0], c[1]);
        v = c[kN - 1] ^ twist(c[kM - 1], c[kM]) ^ twist(c[kN - 1], n0);
      }
      n[t] = v;
      words[s * seg_words + (k + first) * kN + t] = v;
    }
    __syncthreads();
  }
}

constexpr int kTile = 256;  // attempts per tile (one per thread): ~4 CTAs per SM
                            // hide the latency of the correctly rounded log

// 2a. accepted-attempt count per tile.
__global__ void polar_count_kernel(const uint64_t* __restrict__ words, const uint64_t* p0p,
                                   int64_t attempts, int* __restrict__ tile_count) {
  RSVD_PDL_ENTRY();
  const int64_t p0 = int64_t(*p0p);
  const int64_t base = int64_t(blockIdx.x) * kTile;
  int c = 0;
  for (int k = 0; k < kTile / 256; ++k) {
    const int64_t j = base + k * 256 + threadIdx.x;
    if (j < attempts) {
      const Pair p = polar_pair(words[p0 + 2 * j], words[p0 + 2 * j + 1]);
      c += p.ok ? 1 : 0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < 8; ++w) s += ws[w];
    tile_count[blockIdx.x] = s;
  }
}

// 2b. exclusive scan of tile counts (single CTA, sequential chunks).
__global__ void scan_counts_kernel(const int* __restrict__ cnt, int64_t ntiles,
                                   int64_t* __restrict__ off, int64_t* __restrict__ total) {
  RSVD_PDL_ENTRY();
  __shared__ int64_t carry;
  __shared__ int64_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < ntiles; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < ntiles ? cnt[i] : 0;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < int(blockDim.x >> 5) ? wsum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int64_t incl = x + (warp > 0 ? wsum[warp - 1] : 0);
    if (i < ntiles) off[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Exact-mode patch list (pinned, device-mapped): written by polar_write,
// completed by the host (patch_service), applied by polar_patch.
struct PatchEntry {
  int64_t e0;  // stream index of the pair's first normal
  double r2, x, y;
};
struct PatchOut {
  double vy, vx;
};
struct PatchList {
  unsigned long long* count;  // device counter (workspace)
  PatchEntry* ent;            // mapped host memory, cap entries
  int64_t cap;
};

struct GaussOut {
  double* out;
  int64_t n, ld;      // rows of the output, leading dimension
  int64_t total;      // n * l normals
  int64_t first;      // 1 if the cached variate was placed at element 0
  int64_t pairs;      // accepted attempts needed
  int64_t row_lo, row_hi;  // only rows in [row_lo, row_hi) are stored (sharded Psi)
};

// 3. write normals; record the completing attempt.
__global__ void polar_write_kernel(const uint64_t* __restrict__ words, const uint64_t* p0p,
                                   int64_t attempts, const int64_t* __restrict__ tile_off,
                                   const int* __restrict__ tile_count, GaussOut g,
                                   int64_t* __restrict__ done_attempt,
                                   double* __restrict__ cache_val, PatchList pl,
                                   int* __restrict__ flags) {
  RSVD_PDL_ENTRY();
  const int64_t p0 = int64_t(*p0p);
  const int64_t base = int64_t(blockIdx.x) * kTile;
  __shared__ int wcnt[8];
  __shared__ int64_t run;
  // the log table in shared memory: lanes index it at random, which the
  // constant cache would serialize (measured: the whole kernel 19 us on C2)
  __shared__ ddlog::Entry tab[ddlog::kTableSize];
  for (int i = threadIdx.x; i < ddlog::kTableSize; i += blockDim.x) tab[i] = c_log_table[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (tile_off) {
    if (threadIdx.x == 0) run = tile_off[blockIdx.x];
  } else {
    // few tiles: this tile's offset is the sum of the counts before it,
    // summed here (no separate scan launch)
    int64_t v = 0;
    for (int i = threadIdx.x; i < int(blockIdx.x); i += blockDim.x) v += tile_count[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ int64_t ws[8];
    if (lane == 0) ws[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) t += ws[w];
      run = t;
    }
  }
  __syncthreads();
  for (int k = 0; k < kTile / 256; ++k) {
    const int64_t j = base + k * 256 + threadIdx.x;
    Pair p{0, 0, 0, false};
    if (j < attempts) p = polar_pair(words[p0 + 2 * j], words[p0 + 2 * j + 1]);
    const unsigned bal = __ballot_sync(0xffffffffu, p.ok);
    if (lane == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    int before = 0;
    for (int w = 0; w < warp; ++w) before += wcnt[w];
    const int64_t rank = run + before + __popc(bal & ((1u << lane) - 1u));
    bool near = false;
    const int64_t e0 = g.first + 2 * rank;
    if (p.ok && rank < g.pairs) {
      const ddlog::dd ls = ddlog::log_dd(p.r2, tab);
      const double lg = ls.hi + ls.lo;
      const double mult = polar_mult_from_log(p.r2, lg);
      const double vy = __dadd_rn(__dmul_rn(p.y, mult), 0.0);
      const double vx = __dadd_rn(__dmul_rn(p.x, mult), 0.0);
      bool used = e0 + 1 >= g.total;  // its second normal becomes the cached variate
      {
        const int64_t r = e0 % g.n, c = e0 / g.n;
        if (r >= g.row_lo && r < g.row_hi) {
          g.out[c * g.ld + (r - g.row_lo)] = vy;
          used = true;
        }
      }
      if (e0 + 1 < g.total) {
        const int64_t r = (e0 + 1) % g.n, c = (e0 + 1) / g.n;
        if (r >= g.row_lo && r < g.row_hi) {
          g.out[c * g.ld + (r - g.row_lo)] = vx;
          used = true;
        }
      }
      if (rank == g.pairs - 1) {
        *done_attempt = j;
        *cache_val = (e0 + 1 < g.total) ? 0.0 : vx;
      }
      near = pl.ent != nullptr && used && ddlog::log_near_midpoint(ls, lg);
    }
    {
      // warp-aggregated append of the near-midpoint pairs
      const unsigned nb = __ballot_sync(0xffffffffu, near);
      if (nb) {
        unsigned long long base = 0;
        if (lane == __ffs(nb) - 1) base = atomicAdd(pl.count, static_cast<unsigned long long>(__popc(nb)));
        base = __shfl_sync(0xffffffffu, base, __ffs(nb) - 1);
        if (near) {
          const int64_t idx = int64_t(base) + __popc(nb & ((1u << lane) - 1u));
          if (idx < pl.cap) {
            // (visible to the host by patch_signal's system-scope fence: it
            // runs after this grid completed -- griddepcontrol.wait -- and
            // fences before publishing the header)
            pl.ent[idx] = PatchEntry{e0, p.r2, p.x, p.y};
          } else {
            atomicOr(flags, kFlagRngPatchOverflow);
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < 8; ++w) s += wcnt[w];
      run += s;
    }
    __syncthreads();
  }
}

// 3b. exact mode: publish the list length to the host (after polar_write).
__global__ void patch_signal_kernel(const unsigned long long* __restrict__ count, PatchHdr* hdr) {
  RSVD_PDL_ENTRY();
  hdr->count = *count;
  __threadfence_system();
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(&hdr->ready), "r"(1u) : "memory");
}

// 3c. exact mode: wait for the host's normals, write them (and the cache).
// CTA 0 polls the host-written header (one PCIe read per ~1 us); the other
// CTAs poll a device-memory gate it opens.  Grid <= SMs, so all CTAs are
// co-resident.  A host that never answers (it died) makes the kernel trap
// after ~60 s rather than hang the GPU.
__global__ void __launch_bounds__(256) polar_patch_kernel(
    const PatchHdr* hdr, unsigned* __restrict__ gate, const PatchEntry* __restrict__ ent,
    const PatchOut* __restrict__ po, int64_t cap, GaussOut g, DevState* st) {
  RSVD_PDL_ENTRY();
  __shared__ unsigned verdict;
  if (threadIdx.x == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned d = 0;
    if (blockIdx.x == 0) {
      for (;;) {
        asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(d) : "l"(&hdr->done) : "memory");
        if (d) break;
        __nanosleep(1000);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 60ull * 1000000000ull) __trap();
      }
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gate), "r"(d) : "memory");
    } else {
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(gate) : "memory");
        if (d) break;
        __nanosleep(500);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 60ull * 1000000000ull) __trap();
      }
    }
    verdict = d;
  }
  __syncthreads();
  if (verdict != 1) return;  // cancelled (the call failed on the host)
  const int64_t n = min(int64_t(hdr->count), cap);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e0 = ent[i].e0;
    const PatchOut v = po[i];
    {
      const int64_t r = e0 % g.n, c = e0 / g.n;
      if (r >= g.row_lo && r < g.row_hi) g.out[c * g.ld + (r - g.row_lo)] = v.vy;
    }
    if (e0 + 1 < g.total) {
      const int64_t r = (e0 + 1) % g.n, c = (e0 + 1) / g.n;
      if (r >= g.row_lo && r < g.row_hi) g.out[c * g.ld + (r - g.row_lo)] = v.vx;
    } else {
      st->cached = v.vx;  // the completing pair's second normal is the cached variate
    }
  }
}

// 4. new state: block holding draw index T-1, pos = T - 312*b (lazy twist).
__global__ void rng_finish_kernel(const uint64_t* __restrict__ words,
                                  const int64_t* __restrict__ done_attempt,
                                  const double* __restrict__ cache_val, int64_t pairs,
                                  int cache_out, DevState* st, int* flags) {
  RSVD_PDL_ENTRY();
  if (pairs == 0) {
    if (threadIdx.x == 0) {
      st->has_cached = cache_out ? 1 : 0;
      if (!cache_out) st->cached = 0.0;
    }
    return;
  }
  const int64_t p0 = int64_t(st->pos);
  const int64_t J = *done_attempt;
  __syncthreads();  // every thread read st->pos before thread 0 rewrites it
  if (J < 0) {
    if (threadIdx.x == 0) atomicOr(flags, kFlagRngExhausted);
    return;
  }
  const int64_t T = p0 + 2 * (J + 1);
  const int64_t b = (T - 1) / kN;
  for (int t = threadIdx.x; t < kN; t += blockDim.x) st->mt[t] = words[b * kN + t];
  if (threadIdx.x == 0) {
    st->pos = uint64_t(T - b * kN);
    st->has_cached = cache_out ? 1 : 0;
    st->cached = cache_out ? *cache_val : 0.0;
  }
}

// ------------------------------------------------ exact mode, host side
// Worker pool for long patch lists.  Workers spin (pause loop) for a while
// after each job so back-to-back calls dispatch in ~0.1 us, then sleep.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  // f(lo, hi) over [0, n) in up to size()+1 chunks; the caller runs one.
  void run(int64_t n, const std::function<void(int64_t, int64_t)>& f) {
    static const int64_t kMinChunk = [] {
      const char* e = std::getenv("RSVD_HOST_MIN_CHUNK");
      return int64_t(e ? std::max(1, std::atoi(e)) : 64);
    }();
    const int nw = int(workers_.size());
    const int parts = int(std::min<int64_t>(nw + 1, (n + kMinChunk - 1) / kMinChunk));
    if (parts <= 1) {
      if (n > 0) f(0, n);
      return;
    }
    // one job at a time: several handles (e.g. the ranks of a virtual
    // communicator, one thread each) may answer their lists concurrently
    std::lock_guard<std::mutex> job(run_mu_);
    fn_ = &f;
    n_ = n;
    parts_ = parts;
    pending_.store(parts - 1, std::memory_order_relaxed);
    next_.store(1, std::memory_order_relaxed);
    epoch_.fetch_add(1, std::memory_order_release);
    if (sleepers_.load(std::memory_order_acquire) > 0) {
      std::lock_guard<std::mutex> lk(m_);
      cv_.notify_all();
    }
    f(0, n / parts);
    while (pending_.load(std::memory_order_acquire) > 0) spin_pause();
    fn_ = nullptr;
  }

 private:
  static void spin_pause() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int nw = int(std::min(8u, hw)) - 1;
    if (const char* e = std::getenv("RSVD_HOST_THREADS")) nw = std::max(0, std::atoi(e) - 1);
    for (int i = 0; i < nw; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    stop_.store(true);
    {
      std::lock_guard<std::mutex> lk(m_);
      cv_.notify_all();
    }
    for (auto& t : workers_) t.join();
  }
  void loop() {
    uint64_t seen = epoch_.load();
    for (;;) {
      // spin ~2 ms for the next job, then sleep
      const auto t0 = std::chrono::steady_clock::now();
      while (epoch_.load(std::memory_order_acquire) == seen && !stop_.load()) {
        spin_pause();
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2)) {
          std::unique_lock<std::mutex> lk(m_);
          sleepers_.fetch_add(1);
          cv_.wait(lk, [&] { return epoch_.load() != seen || stop_.load(); });
          sleepers_.fetch_sub(1);
        }
      }
      if (stop_.load()) return;
      seen = epoch_.load(std::memory_order_acquire);
      for (;;) {
        const int k = next_.fetch_add(1);
        if (k >= parts_) break;
        const int64_t lo = n_ * k / parts_, hi = n_ * (k + 1) / parts_;
        (*fn_)(lo, hi);
        pending_.fetch_sub(1, std::memory_order_release);
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_mu_;
  std::mutex m_;
  std::condition_variable cv_;
  const std::function<void(int64_t, int64_t)>* fn_ = nullptr;
  int64_t n_ = 0;
  int parts_ = 0;
  std::atomic<int> next_{0}, pending_{0}, sleepers_{0};
  std::atomic<uint64_t> epoch_{0};
  std::atomic<bool> stop_{false};
};

bool exact_mode_env() {
  static const bool on = [] {
    const char* e = std::getenv("RSVD_OMEGA_EXACT");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Pinned mapped bytes from the handle's patch chunks (see common.cuh).
char* patch_alloc(Handle& h, size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  while (h.patch_chunk < h.patch_chunks.size()) {
    auto& c = h.patch_chunks[h.patch_chunk];
    if (h.patch_off + bytes <= c.second) {
      char* p = c.first + h.patch_off;
      h.patch_off += bytes;
      return p;
    }
    ++h.patch_chunk;
    h.patch_off = 0;
  }
  const size_t sz = std::max<size_t>(bytes, size_t(1) << 20);
  void* p = nullptr;
  RSVD_CUDA(cudaHostAlloc(&p, sz, cudaHostAllocMapped | cudaHostAllocPortable));
  h.patch_chunks.push_back({static_cast<char*>(p), sz});
  h.patch_chunk = h.patch_chunks.size() - 1;
  h.patch_off = bytes;
  return static_cast<char*>(p);
}

std::once_flag g_table_once;
ddlog::Entry g_host_table[ddlog::kTableSize];

}  // namespace

const ddlog::Entry* host_log_table() {
  std::call_once(g_table_once, [] { ddlog::build_table(g_host_table); });
  return g_host_table;
}

// Answer the exact-mode lists of this call, in queue order (see "Exact mode").
// Called by the host thread before it waits for the stream.
static bool patch_debug() {
  static const bool on = std::getenv("RSVD_PATCH_DEBUG") != nullptr;
  return on;
}

void patch_service(Handle& h) {
  if (h.patch_pending.empty()) return;
  if (patch_debug())
    std::fprintf(stderr, "[patch] rank %d service %zu list(s) first %p\n", h.rank, h.patch_pending.size(),
                 static_cast<void*>(h.patch_pending[0]));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  RSVD_CUDA(cudaStreamIsCapturing(h.stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) return;  // nothing runs before the graph launches
  for (PatchHdr* hdr : h.patch_pending) {
    int polls = 0;
    while (reinterpret_cast<volatile PatchHdr*>(hdr)->ready == 0) {
      if (++polls % 4096 == 0) {
        // the GPU may have failed before reaching the list: do not spin forever
        const cudaError_t q = cudaStreamQuery(h.stream);
        if (q != cudaErrorNotReady) {
          patch_cancel(h);
          if (q != cudaSuccess) RSVD_CUDA(q);
          throw Error(RSVD_ERR_INTERNAL, "exact-mode patch list never published");
        }
      }
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const int64_t n = std::min<int64_t>(int64_t(hdr->count), hdr->cap);
    if (patch_debug()) std::fprintf(stderr, "[patch] rank %d list %p ready, %lld entries\n", h.rank,
                                    static_cast<void*>(hdr), static_cast<long long>(n));
    const PatchEntry* ent = reinterpret_cast<const PatchEntry*>(reinterpret_cast<char*>(hdr) + 64);
    PatchOut* out = reinterpret_cast<PatchOut*>(reinterpret_cast<char*>(hdr) + 64 +
                                                size_t(hdr->cap) * sizeof(PatchEntry));
    // libstdc++ polar multiplier with the host's log (random.tcc:1837:
    // __mult = std::sqrt(-2 * std::log(__r2) / __r2); normal = (y * mult) * 1 + 0)
    HostPool::get().run(n, [ent, out](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        const PatchEntry e = ent[i];
        const double mult = std::sqrt(-2 * std::log(e.r2) / e.r2);
        out[i].vy = e.y * mult * 1.0 + 0.0;
        out[i].vx = e.x * mult * 1.0 + 0.0;
      }
    });
    std::atomic_thread_fence(std::memory_order_release);
    reinterpret_cast<volatile PatchHdr*>(hdr)->done = 1;
    if (patch_debug()) std::fprintf(stderr, "[patch] rank %d list %p done\n", h.rank, static_cast<void*>(hdr));
  }
  h.patch_pending.clear();
}

// Release every pending list without patching (the call failed on the host):
// the waiting patch kernels exit.
void patch_cancel(Handle& h) {
  for (PatchHdr* hdr : h.patch_pending) reinterpret_cast<volatile PatchHdr*>(hdr)->done = 2;
  h.patch_pending.clear();
}

void stream_sync(Handle& h) {
  patch_service(h);
  RSVD_CUDA(cudaStreamSynchronize(h.stream));
}

// Jump polynomials on the device, cached per handle (grown on demand).
static const uint64_t* device_jump_polys(Handle& h, uint64_t L, int count) {
  if (count <= 0) return nullptr;
  if (h.jump_L != L || h.jump_count < count) {
    if (h.jump_L == L) count = std::max(count, 2 * h.jump_count);  // grow geometrically
    const uint64_t* hp = mtjump::jump_polys(L, count);
    if (h.d_jump) {
      stream_sync(h);
      RSVD_CUDA(cudaFree(h.d_jump));
    }
    RSVD_CUDA(cudaMalloc(&h.d_jump, size_t(count) * kPolyWords * 8));
    ++h.generation;
    RSVD_CUDA(cudaMemcpy(h.d_jump, hp, size_t(count) * kPolyWords * 8, cudaMemcpyHostToDevice));
    h.jump_L = L;
    h.jump_count = count;
  }
  return h.d_jump;
}

void rng_init_device(Handle& h) {
  (void)h;
  RSVD_CUDA(cudaMemcpyToSymbol(c_log_table, host_log_table(), sizeof(g_host_table)));
}

DevRng rng_upload(Handle& h, const rsvd_rng_state* st) {
  if (st->pos > uint64_t(kN)) throw_param("rng: invalid state index");
  DevRng r;
  r.d = h.ws.alloc_bytes(sizeof(DevState));
  r.has_cached = st->has_cached ? 1 : 0;
  static_assert(sizeof(DevState) == sizeof(rsvd_rng_state), "state layout");
  // through pinned staging: a graph-capturable copy whose source the replay
  // path refills with the caller's state before each launch
  if (h.h_rng_in != st) std::memcpy(h.h_rng_in, st, sizeof(DevState));
  RSVD_CUDA(cudaMemcpyAsync(r.d, h.h_rng_in, sizeof(DevState), cudaMemcpyHostToDevice, h.stream));
  return r;
}

void rng_download(Handle& h, const DevRng& r, rsvd_rng_state* user) {
  RSVD_CUDA(cudaMemcpyAsync(h.h_rng, r.d, sizeof(DevState), cudaMemcpyDeviceToHost, h.stream));
  h.rng_user_out = user;  // filled from h.h_rng at the call's final synchronization
}

namespace {
__global__ void place_cached_kernel(const DevState* st, double* out) {
  RSVD_PDL_ENTRY(); out[0] = st->cached; }

}  // namespace

void gaussian_dev(Handle& h, int64_t n, int64_t l, DevRng& rng, DMat out, int64_t row_lo,
                  int64_t row_hi) {
  if (n < 1 || l < 1) throw_param("gaussian: dimensions must be positive");
  if (row_hi < 0) {
    row_lo = 0;
    row_hi = n;
  }
  DevState* dst = static_cast<DevState*>(rng.d);
  const int64_t total = n * l;
  const int64_t first = rng.has_cached ? 1 : 0;
  const int64_t remaining = total - first;
  const int64_t pairs = (remaining + 1) / 2;
  const int cache_out = (remaining % 2 == 1) ? 1 : 0;
  // the cached variate (if any) is element 0 of the stream
  if (first && row_lo == 0 && row_hi > 0) {
    launch_k(h, place_cached_kernel, 1, 1, 0, dst, out.p);
    RSVD_LAUNCHED(h);
  }
  if (pairs > 0) {
    // attempt budget: mean pairs/(pi/4) plus > 10 standard deviations
    const double p = 0.78539816339744831;
    const int64_t attempts =
        int64_t(double(pairs) / p + 10.0 * 0.59 * std::sqrt(double(pairs)) + 64.0);
    const int64_t words_needed = kN + 2 * attempts;  // worst-case start index 312
    uint64_t* words;
    const int64_t seg_blocks =
        (words_needed <= 3 * 148 * kSegBlocksShort * kN) ? kSegBlocksShort : kSegBlocksLong;
    const int64_t kSegWords = seg_blocks * kN;
    // One CTA twists a 312-word block in ~220 ns (measured, latency bound);
    // beyond two segments the jump-ahead path (base prefix + jump XORs +
    // parallel segments) is faster.
    if (words_needed <= 2 * kSegWords) {
      const int64_t nb = ceil_div(words_needed, kN) - 1;
      words = reinterpret_cast<uint64_t*>(h.ws.alloc_bytes(size_t(nb + 1) * kN * 8));
      launch_k(h, mt_blocks_kernel, 1, 320, 0, dst->mt, nb, words);
      RSVD_LAUNCHED(h);
    } else {
      // parallel: base prefix (sequential), jump windows, all segments at once
      const int64_t nseg = ceil_div(words_needed, kSegWords);
      words = reinterpret_cast<uint64_t*>(h.ws.alloc_bytes(size_t(nseg) * kSegWords * 8));
      uint64_t* windows = reinterpret_cast<uint64_t*>(h.ws.alloc_bytes(size_t(nseg) * kN * 8));
      const uint64_t* dpolys = device_jump_polys(h, uint64_t(kSegWords), int(nseg - 1));
      const int64_t nb_base = ceil_div(1 + kJumpBase, kN);
      launch_k(h, mt_blocks_kernel, 1, 320, 0, dst->mt, nb_base, words);
      RSVD_LAUNCHED(h);
      // split every jump over `parts` CTAs so all SMs share the XOR work
      const int parts = int(std::max<int64_t>(1, std::min<int64_t>(32, (2 * h.sm_count) / (nseg - 1))));
      const int wpp = (kPolyWords + parts - 1) / parts;
      const size_t jsmem = size_t(64 * wpp + kN) * 8;
      smem_attr(mt_jump_kernel, jsmem);
      RSVD_CUDA(cudaMemsetAsync(windows, 0, size_t(nseg) * kN * 8, h.stream));
      launch_k(h, mt_jump_kernel, dim3(unsigned(nseg - 1), unsigned(parts)), 320, jsmem, 
          words, dpolys, wpp, reinterpret_cast<unsigned long long*>(windows));
      RSVD_LAUNCHED(h);
      // one segment per CTA while that fits the SMs (a 312-thread CTA twists a
      // block in ~220 ns; three in lockstep take ~2x longer per block)
      const int spc = (nseg <= 2 * h.sm_count) ? 1 : kSegPerCta;
      launch_k(h, mt_segments_kernel, unsigned(ceil_div(nseg, spc)), spc * kN, 0, 
          dst->mt, windows, nseg, seg_blocks, words);
      RSVD_LAUNCHED(h);
    }
    const int64_t ntiles = ceil_div(attempts, kTile);
    int* cnt = reinterpret_cast<int*>(h.ws.alloc_bytes(size_t(ntiles) * 4 + 16));
    int64_t* off = reinterpret_cast<int64_t*>(h.ws.alloc_bytes(size_t(ntiles + 4) * 8));
    int64_t* done = off + ntiles;  // [done_attempt, total]
    double* cache = reinterpret_cast<double*>(done + 2);
    RSVD_CUDA(cudaMemsetAsync(done, 0xff, sizeof(int64_t), h.stream));
    launch_k(h, polar_count_kernel, unsigned(ntiles), 256, 0, words, &dst->pos, attempts, cnt);
    RSVD_LAUNCHED(h);
    // up to 4096 tiles each write CTA sums the counts before its tile itself
    // (<= 16 loads per thread); beyond, one scan launch
    const bool self_scan = ntiles <= 4096;
    if (!self_scan) {
      launch_k(h, scan_counts_kernel, 1, 1024, 0, cnt, ntiles, off, done + 1);
      RSVD_LAUNCHED(h);
    }
    GaussOut g{out.p, n, out.ld, total, first, pairs, row_lo, row_hi};
    // exact mode: room for 4 % of the pairs (the window flags ~1.7 %; the
    // count is binomial, so this is > 40 standard deviations for C2's
    // 102400 pairs) -- an overflow raises an error, never a silent mismatch
    PatchList pl{nullptr, nullptr, 0};
    PatchOut* pout = nullptr;
    PatchHdr* hdr = nullptr;
    if (exact_mode_env()) {
      const int64_t stored = (row_hi - row_lo) * l;
      pl.cap = std::min<int64_t>(pairs, (std::min(pairs, stored + 1) * 4) / 100 + 1024);
      char* buf = patch_alloc(h, 64 + size_t(pl.cap) * (sizeof(PatchEntry) + sizeof(PatchOut)));
      hdr = reinterpret_cast<PatchHdr*>(buf);
      hdr->ready = 0;
      hdr->done = 0;
      hdr->cap = pl.cap;
      pl.ent = reinterpret_cast<PatchEntry*>(buf + 64);
      pout = reinterpret_cast<PatchOut*>(buf + 64 + size_t(pl.cap) * sizeof(PatchEntry));
      pl.count = reinterpret_cast<unsigned long long*>(h.ws.alloc_bytes(64));
      RSVD_CUDA(cudaMemsetAsync(pl.count, 0, 16, h.stream));  // count + gate
    }
    launch_k(h, polar_write_kernel, unsigned(ntiles), 256, 0, words, &dst->pos, attempts,
             self_scan ? static_cast<const int64_t*>(nullptr) : static_cast<const int64_t*>(off),
             static_cast<const int*>(cnt), g, done, cache, pl, h.d_flags);
    RSVD_LAUNCHED(h);
    launch_k(h, rng_finish_kernel, 1, 320, 0, words, done, cache, pairs, cache_out, dst,
                                               h.d_flags);
    RSVD_LAUNCHED(h);
    if (hdr) {
      unsigned* gate = reinterpret_cast<unsigned*>(pl.count + 1);
      const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(pl.cap, 1024), h.sm_count)));
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      RSVD_CUDA(cudaStreamIsCapturing(h.stream, &cap));
      if (cap == cudaStreamCaptureStatusNone) {
        // Eager call: the list is answered right here, synchronously (the
        // host is about to wait for the call anyway), and polar_patch is
        // queued with its answer already in place -- no kernel ever waits
        // on the host, so no later implicit device synchronization (a
        // growing workspace's cudaMalloc, another thread sharing the stream)
        // can deadlock with it.
        // (the same kernels as the captured form: counters agree across both)
        launch_k(h, patch_signal_kernel, 1, 32, 0, static_cast<const unsigned long long*>(pl.count), hdr);
        RSVD_LAUNCHED(h);
        stream_sync(h);
        h.patch_pending.push_back(hdr);
        patch_service(h);  // computes the normals, sets done = 1
        launch_k(h, polar_patch_kernel, unsigned(blocks), 256, 0, static_cast<const PatchHdr*>(hdr), gate,
                 static_cast<const PatchEntry*>(pl.ent), static_cast<const PatchOut*>(pout), pl.cap, g, dst);
        RSVD_LAUNCHED(h);
      } else {
        // Captured call: patch_signal publishes the count, polar_patch waits
        // for the host's answer, which finish_call gives after the graph
        // launch (the host does nothing else in between).
        launch_k(h, patch_signal_kernel, 1, 32, 0, static_cast<const unsigned long long*>(pl.count), hdr);
        RSVD_LAUNCHED(h);
        launch_k(h, polar_patch_kernel, unsigned(blocks), 256, 0, static_cast<const PatchHdr*>(hdr), gate,
                 static_cast<const PatchEntry*>(pl.ent), static_cast<const PatchOut*>(pout), pl.cap, g, dst);
        RSVD_LAUNCHED(h);
        h.patch_pending.push_back(hdr);
      }
    }
  } else {
    launch_k(h, rng_finish_kernel, 1, 32, 0, nullptr, nullptr, nullptr, 0, 0, dst, h.d_flags);
    RSVD_LAUNCHED(h);
  }
  rng.has_cached = cache_out;
}

}  // namespace rsvdb

extern "C" double rsvd_debug_log_cr(double x) {
  return rsvdb::ddlog::log_cr(x, rsvdb::host_log_table());
}

// Exact-mode flag test over an array (host evaluation of the device code):
// cr[i] = correctly rounded log(x[i]), flag[i] = 1 where the host log must be
// used (ddlog.cuh log_near_midpoint).
extern "C" void rsvd_debug_log_window(const double* x, int64_t n, double* cr, uint8_t* flag) {
  const rsvdb::ddlog::Entry* t = rsvdb::host_log_table();
  for (int64_t i = 0; i < n; ++i) {
    const rsvdb::ddlog::dd s = rsvdb::ddlog::log_dd(x[i], t);
    const double v = s.hi + s.lo;
    cr[i] = v;
    flag[i] = rsvdb::ddlog::log_near_midpoint(s, v) ? 1 : 0;
  }
}
