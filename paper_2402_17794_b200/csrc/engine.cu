// Pipelines of the rsvd hot path on B200, restating the reference's
// algorithms statement by statement on device-resident data:
//   range finders  rangefinder.hpp:60-105   (Alg 2 / 3 / 4, Stage 1)
//   rsvd           factor.hpp:12-24         (Stage 2)
//   svd_small      core.hpp:111-124, solve_ls core.hpp:166-177,
//   evd_symmetric  core.hpp:130-162
//   spevd_hermitian singlepass.hpp:45-78    (Alg 5, one pass over A)
//   spsvd_general   singlepass.hpp:109-137  (Alg 6, solve_joint_core :84-101)
// A is row-sharded when the handle spans several GPUs: products with A are
// local, and only the n x l / l x l partials are NCCL-allreduced (dist.cu).
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "dist.cuh"
#include "engine.cuh"
#include "pass.cuh"
#include "fused.cuh"
#include "ozaki.cuh"
#include "rng.cuh"
#include "small.cuh"

namespace rsvdb {

// ------------------------------------------------------------------ arena
// RSVD_POISON=<byte>: fill every workspace chunk with that byte at each reset
// and allocation (debug: results must not depend on stale workspace contents).
static int arena_poison() {
  static const int v = [] {
    const char* e = std::getenv("RSVD_POISON");
    return e ? std::atoi(e) & 255 : -1;
  }();
  return v;
}

// RSVD_ARENA_TINY=1: 256 KB chunks, never merged (debug: every call grows
// the arena mid-call many times).
static bool arena_tiny() {
  static const bool v = std::getenv("RSVD_ARENA_TINY") != nullptr;
  return v;
}

Arena::~Arena() {
  for (auto& c : chunks_) cudaFree(c.p);
}

void Arena::reset() {
  size_t cap = 0;
  for (auto& c : chunks_) cap += c.cap;
  if (!arena_tiny() && (chunks_.size() > 1 || (chunks_.size() == 1 && chunks_[0].cap < high_))) {
    for (auto& c : chunks_) cudaFree(c.p);
    chunks_.clear();
    Chunk c{nullptr, size_t(round_up(int64_t(high_), int64_t(1) << 20)), 0};
    RSVD_CUDA(cudaMalloc(&c.p, c.cap));
    chunks_.push_back(c);
    ++gen_;
  }
  for (auto& c : chunks_) c.off = 0;
  if (arena_poison() >= 0)
    for (auto& c : chunks_) RSVD_CUDA(cudaMemset(c.p, arena_poison(), c.cap));
  if (arena_poison() >= 0) RSVD_CUDA(cudaDeviceSynchronize());
  used_total_ = 0;
  (void)cap;
}

void* Arena::alloc_bytes(size_t bytes) {
  bytes = size_t(round_up(int64_t(std::max<size_t>(bytes, 1)), 256));
  // first fit over the chunks already held (an earlier chunk's tail is not
  // lost when a large request opened a new chunk behind it)
  for (auto& c : chunks_) {
    if (c.off + bytes <= c.cap) {
      void* p = c.p + c.off;
      c.off += bytes;
      used_total_ += bytes;
      high_ = std::max(high_, used_total_);
      return p;
    }
  }
  {
    size_t want = std::max<size_t>(bytes, arena_tiny() ? (size_t(256) << 10) : (size_t(64) << 20));
    // geometric growth, bounded: after a matrix-sized chunk the next request
    // must not ask for twice that again
    if (!chunks_.empty() && !arena_tiny())
      want = std::max(want, std::min<size_t>(2 * chunks_.back().cap, size_t(4) << 30));
    Chunk c{nullptr, want, 0};
    cudaError_t e = cudaMalloc(&c.p, c.cap);
    if (e != cudaSuccess) {
      cudaGetLastError();
      // out of memory: give back the chunks this call has not touched (e.g. the
      // previous call's merged high-water chunk, too small for this request)
      for (size_t i = 0; i < chunks_.size();) {
        if (chunks_[i].off == 0) {
          cudaFree(chunks_[i].p);
          chunks_.erase(chunks_.begin() + i);
        } else {
          ++i;
        }
      }
      c.cap = bytes;
      RSVD_CUDA(cudaMalloc(&c.p, c.cap));
    }
    if (arena_poison() >= 0) {
      RSVD_CUDA(cudaMemset(c.p, arena_poison(), c.cap));
      RSVD_CUDA(cudaDeviceSynchronize());
    }
    chunks_.push_back(c);
    ++gen_;
  }
  Chunk& c = chunks_.back();
  void* p = c.p + c.off;
  c.off += bytes;
  used_total_ += bytes;
  high_ = std::max(high_, used_total_);
  return p;
}

int* tile_counters(Handle& h, int64_t n) {
  if (n > h.n_counters) {
    if (h.d_counters) {
      stream_sync(h);
      RSVD_CUDA(cudaFree(h.d_counters));
    }
    const int64_t cap = std::max<int64_t>(n, 4096);
    RSVD_CUDA(cudaMalloc(&h.d_counters, size_t(cap) * sizeof(int)));
    ++h.generation;
    RSVD_CUDA(cudaMemsetAsync(h.d_counters, 0, size_t(cap) * sizeof(int), h.stream));
    h.n_counters = cap;
  }
  return h.d_counters;
}

static cudaEvent_t trace_event(Handle& h) {
  cudaEvent_t e;
  if (h.trace_pool.empty()) {
    RSVD_CUDA(cudaEventCreate(&e));
  } else {
    e = h.trace_pool.back();
    h.trace_pool.pop_back();
  }
  return e;
}

void trace_begin(Handle& h) {
  if (!h.trace) return;
  cudaEvent_t e = trace_event(h);
  RSVD_CUDA(cudaEventRecord(e, h.stream));
  h.trace_ev.push_back({"<call start>", e});
}

void trace_mark(Handle& h, const char* site) {
  cudaEvent_t e = trace_event(h);
  RSVD_CUDA(cudaEventRecord(e, h.stream));
  h.trace_ev.push_back({site, e});
}

void trace_collect(Handle& h) {
  for (size_t i = 1; i < h.trace_ev.size(); ++i) {
    float ms = 0.f;
    RSVD_CUDA(cudaEventElapsedTime(&ms, h.trace_ev[i - 1].second, h.trace_ev[i].second));
    const std::string site = h.trace_ev[i].first;
    bool found = false;
    for (auto& kv : h.trace_acc)
      if (kv.first == site) {
        kv.second.first += 1;
        kv.second.second += ms;
        found = true;
        break;
      }
    if (!found) h.trace_acc.push_back({site, {1, double(ms)}});
  }
  for (auto& kv : h.trace_ev) h.trace_pool.push_back(kv.second);
  h.trace_ev.clear();
}

void finish_call(Handle& h, const char* what) {
  rsvd_rng_state* user = h.rng_user_out;
  h.rng_user_out = nullptr;
  patch_service(h);  // exact-mode Omega lists the queued kernels wait on
  if (h.copy_stream) RSVD_CUDA(cudaStreamSynchronize(h.copy_stream));  // an upload nothing waited on
  check_flags(h, what);  // synchronizes
  if (user) std::memcpy(user, h.h_rng, sizeof(rsvd_rng_state));
  for (auto& r : h.prof_pending) {
    float ms = 0.f;
    RSVD_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    h.prof_ms[r.kind] += ms;
    h.prof_flops[r.kind] += r.flops;
    h.prof_bytes[r.kind] += r.bytes;
    h.prof_count[r.kind] += 1;
    if (!r.graph) {
      h.prof_pool.push_back(r.a);
      h.prof_pool.push_back(r.b);
    }
  }
  h.prof_pending.clear();
  if (h.trace) trace_collect(h);
}

namespace {

// ------------------------------------------------------- small kernels
// Rows i of T scaled by 1/s_i, or zeroed when s_i < max(1e-12 s_max, DBL_MIN)
// (Eigen SVDBase::rank threshold as used by solve_ls, core.hpp:164-176).
__global__ void pinv_rows_kernel(double* T, int64_t rows, int64_t cols, int64_t ld,
                                 const double* s) {
  RSVD_PDL_ENTRY();
  const double thr = fmax(s[0] * 1e-12, DBL_MIN);
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    const double si = s[i];
    T[j * ld + i] = (si >= thr) ? T[j * ld + i] / si : 0.0;
  }
}

// Kronecker-diagonalised joint core: X_ij = (s1_i a_ij + s2_j b_ij) / (s1_i^2 + s2_j^2),
// zero where sqrt(s1_i^2 + s2_j^2) < 1e-12 * sqrt(s1_0^2 + s2_0^2).
__global__ void kron_core_kernel(const double* a, const double* b, int64_t l, int64_t lda,
                                 const double* s1, const double* s2, double* X, int64_t ldx) {
  RSVD_PDL_ENTRY();
  const double smax = sqrt(s1[0] * s1[0] + s2[0] * s2[0]);
  const double thr = fmax(smax * 1e-12, DBL_MIN);
  const int64_t n = l * l;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % l, j = e / l;
    const double x1 = s1[i], x2 = s2[j];
    const double den = x1 * x1 + x2 * x2;
    X[j * ldx + i] =
        (sqrt(den) < thr) ? 0.0 : (x1 * a[j * lda + i] + x2 * b[j * lda + i]) / den;
  }
}

// max|A| and max|A - A^T| over an n x n matrix, one read of A (tile pairs).
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}
// Persistent grid over tile pairs (bi <= bj) of the upper triangle: tile
// (bi, bj) and its mirror (bj, bi) are loaded once each (coalesced columns),
// running maxima stay in registers, one atomic per CTA at the end.  The next
// pair's loads are issued before the current pair is compared (register
// double buffering): one read of A at close to streaming bandwidth.
__device__ __forceinline__ void asym_pair(int64_t t0, int64_t nt, int64_t& bi, int64_t& bj) {
  bi = int64_t((2.0 * nt + 1.0 - sqrt((2.0 * nt + 1.0) * (2.0 * nt + 1.0) - 8.0 * t0)) / 2.0);
  if (bi < 0) bi = 0;
  while (bi > 0 && bi * nt - bi * (bi - 1) / 2 > t0) --bi;
  while ((bi + 1) * nt - (bi + 1) * bi / 2 <= t0) ++bi;
  bj = bi + (t0 - (bi * nt - bi * (bi - 1) / 2));
}

// T x T tiles, 256 threads: thread (tx = row in tile, ty) owns columns ty + (256/T) q.
// T = 64 reads 512-byte column segments (T = 32: 256 bytes).
template <int T>
__global__ void __launch_bounds__(256) asym_kernel(const double* __restrict__ A, int64_t n,
                                                   int64_t lda, double* out) {
  RSVD_PDL_ENTRY();
  constexpr int CS = 256 / T;  // column stride between a thread's elements
  constexpr int E = T / CS;    // elements per thread per tile
  __shared__ double T2[T][T + 1];
  __shared__ double r_abs[8], r_asym[8];
  const int64_t nt = (n + T - 1) / T;
  const int64_t npairs = nt * (nt + 1) / 2;
  const int tx = threadIdx.x % T, ty = threadIdx.x / T;
  double mabs = 0.0, masym = 0.0;
  double a[E], b[E];
  auto load = [&](int64_t t0) {
    int64_t bi, bj;
    asym_pair(t0, nt, bi, bj);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int k = ty + CS * q;
      const int64_t r1 = bi * T + tx, c1 = bj * T + k;  // A(bi*T + tx, bj*T + k)
      a[q] = (r1 < n && c1 < n) ? __ldcs(A + c1 * lda + r1) : 0.0;
      const int64_t r2 = bj * T + tx, c2 = bi * T + k;  // A(bj*T + tx, bi*T + k)
      b[q] = (r2 < n && c2 < n) ? __ldcs(A + c2 * lda + r2) : 0.0;
    }
  };
  int64_t t0 = blockIdx.x;
  if (t0 < npairs) load(t0);
  for (; t0 < npairs; t0 += gridDim.x) {
    double ca[E];
#pragma unroll
    for (int q = 0; q < E; ++q) {
      ca[q] = a[q];
      T2[ty + CS * q][tx] = b[q];
    }
    if (t0 + gridDim.x < npairs) load(t0 + gridDim.x);  // in flight during the compare
    __syncthreads();
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int k = ty + CS * q;
      const double x = ca[q], y = T2[tx][k];  // A(i, j) vs A(j, i)
      mabs = fmax(mabs, fmax(fabs(x), fabs(y)));
      masym = fmax(masym, fabs(x - y));
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    mabs = fmax(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
    masym = fmax(masym, __shfl_xor_sync(0xffffffffu, masym, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    r_abs[w] = mabs;
    r_asym[w] = masym;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) {
      mabs = fmax(mabs, r_abs[i]);
      masym = fmax(masym, r_asym[i]);
    }
    atomic_max_nonneg(&out[0], mabs);
    atomic_max_nonneg(&out[1], masym);
  }
}
__global__ void asym_flag_kernel(const double* mm, int* flags, int bit) {
  RSVD_PDL_ENTRY();
  if (!(mm[1] <= 1e-8 * (1.0 + mm[0]))) atomicOr(flags, bit);
}

// Sharded precondition: max|X - Y^T| (X r x c, Y c x r) and max|X|, max|Y|,
// one read of each: 32 x 32 tiles of X, the matching tile of Y transposed
// through shared memory.  out[0] max|.|, out[1] max asymmetry (atomic max).
__global__ void __launch_bounds__(256) asym_block_kernel(const double* __restrict__ X, int64_t ldx,
                                                        const double* __restrict__ Y, int64_t ldy,
                                                        int64_t r, int64_t c, double* out) {
  RSVD_PDL_ENTRY();
  __shared__ double T[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 row groups
  const int64_t tr = (r + 31) / 32, tc = (c + 31) / 32;
  double mabs = 0.0, masym = 0.0;
  for (int64_t t = blockIdx.x; t < tr * tc; t += gridDim.x) {
    const int64_t bi = t % tr, bj = t / tr;
    // Y tile (rows bj*32.., cols bi*32..) -> T[col][row] = Y^T
    for (int q = ty; q < 32; q += 8) {
      const int64_t yr = bj * 32 + tx, yc = bi * 32 + q;
      const double y = (yr < c && yc < r) ? Y[yc * ldy + yr] : 0.0;
      T[q][tx] = y;  // T[i][j] = Y(bj*32 + j, bi*32 + i) = Y^T(bi*32 + i, bj*32 + j)
      mabs = fmax(mabs, fabs(y));
    }
    __syncthreads();
    for (int q = ty; q < 32; q += 8) {
      const int64_t xr = bi * 32 + tx, xc = bj * 32 + q;
      if (xr < r && xc < c) {
        const double x = X[xc * ldx + xr];
        mabs = fmax(mabs, fabs(x));
        masym = fmax(masym, fabs(x - T[tx][q]));
      }
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    mabs = fmax(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
    masym = fmax(masym, __shfl_xor_sync(0xffffffffu, masym, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(&out[0], mabs);
    atomic_max_nonneg(&out[1], masym);
  }
}

int grid_for(int64_t n, const Handle& h) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 4 * h.sm_count)));
}

}  // namespace

// Asymmetry precondition (core.hpp:135-140 / singlepass.hpp:49-53).
void check_symmetric(Handle& h, const DMat& C, bool dist_unused) {
  (void)dist_unused;
  const int64_t n = C.rows;
  if (n == 0) return;
  double* mm = h.ws.alloc(2);
  RSVD_CUDA(cudaMemsetAsync(mm, 0, 16, h.stream));
  static const int tile_env = std::getenv("RSVD_ASYM_T") ? std::atoi(std::getenv("RSVD_ASYM_T")) : 64;
  if (tile_env == 32 || n < 1024) {
    const int64_t nt = ceil_div(n, 32);
    const int64_t grid = std::min<int64_t>(nt * (nt + 1) / 2, 8 * h.sm_count);
    launch_k(h, asym_kernel<32>, unsigned(grid), 256, 0, C.p, n, C.ld, mm);
  } else {
    const int64_t nt = ceil_div(n, 64);
    const int64_t grid = std::min<int64_t>(nt * (nt + 1) / 2, 6 * h.sm_count);
    launch_k(h, asym_kernel<64>, unsigned(grid), 256, 0, C.p, n, C.ld, mm);
  }
  RSVD_LAUNCHED(h);
  launch_k(h, asym_flag_kernel, 1, 1, 0, mm, h.d_flags, kFlagAsymmetric);
  RSVD_LAUNCHED(h);
}

// Asymmetry precondition of a row-sharded square A (singlepass.hpp:49-53),
// as the separate, uncounted validation pass SURVEY 7.3(9) asks for: rank r
// compares its block A_r[:, R_s] with rank s's block A_s[:, R_r] transposed
// for every s (its own diagonal block included), then max-allreduces
// (max|A|, max|A - A^T|).  The peer blocks move rank to rank (NCCL send /
// recv, one peer per round; the virtual communicator reads them in place):
// the only place A's data crosses GPUs, and it is not part of the single pass.
void check_symmetric_dist(Handle& h, const Problem& P) {
  const int64_t n = P.A.cols, mr = P.A.rows;
  double* mm = h.ws.alloc(2);
  RSVD_CUDA(cudaMemsetAsync(mm, 0, 16, h.stream));
  std::vector<int64_t> rows, offs;
  shard_layout(h, mr, &rows, &offs);
  const int R = h.nranks, me = h.rank;
  auto compare = [&](const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t r, int64_t c) {
    if (r == 0 || c == 0) return;
    const int64_t tiles = ceil_div(r, 32) * ceil_div(c, 32);
    launch_k(h, asym_block_kernel, unsigned(std::min<int64_t>(tiles, 4 * h.sm_count)), 256, 0, X, ldx,
             Y, ldy, r, c, mm);
    RSVD_LAUNCHED(h);
  };
  for (int t = 0; t < R; ++t) {
    const int s = (me + t) % R;       // the peer whose block A_s[:, R_me] this rank checks
    const int d = (me - t + R) % R;   // the peer that checks A_me[:, R_d]
    const int64_t ms = rows[size_t(s)], md = rows[size_t(d)];
    // X = A_me[:, R_s] (mr x ms), Y = A_s[:, R_me] (ms x mr)
    const double* X = P.A.p + offs[size_t(s)] * P.A.ld;
    const double* Y;
    int64_t ldy;
    if (t == 0) {
      Y = P.A.p + offs[size_t(me)] * P.A.ld;
      ldy = P.A.ld;
    } else {
      double* buf = h.ws.alloc(std::max<int64_t>(ms * mr, 1));
      peer_exchange(h, P.A.p + offs[size_t(d)] * P.A.ld, P.A.ld, mr, md, d, buf, ms, mr, s);
      Y = buf;
      ldy = ms;
    }
    compare(X, P.A.ld, Y, ldy, mr, ms);
  }
  (void)n;
  allreduce_max(h, mm, 2);
  launch_k(h, asym_flag_kernel, 1, 1, 0, mm, h.d_flags, kFlagAsymmetric);
  RSVD_LAUNCHED(h);
}

// ------------------------------------------------------------ operators
static void a_ready(Handle& h, const Problem& P) {
  if (P.ready) RSVD_CUDA(cudaStreamWaitEvent(h.stream, P.ready, 0));
  for (const Problem::Panel& pn : P.panels)
    if (pn.ready) RSVD_CUDA(cudaStreamWaitEvent(h.stream, pn.ready, 0));
}

void op_apply(Handle& h, const Problem& P, const DMat& X, DMat Y) {
  if (!P.panels.empty()) {
    // streamed upload: each row panel's rows of Y as soon as the panel lands
    for (const Problem::Panel& pn : P.panels) {
      if (pn.ready) RSVD_CUDA(cudaStreamWaitEvent(h.stream, pn.ready, 0));
      gemm_nn(h, DMat(P.A.p + pn.row0, pn.row1 - pn.row0, P.A.cols, P.A.ld), X,
              DMat(Y.p + pn.row0, pn.row1 - pn.row0, Y.cols, Y.ld));
    }
    h.counters.apply++;
    h.counters.physical_passes++;
    return;
  }
  a_ready(h, P);
  if (ozaki_cache_decide(h, P.oz, P.A, X.cols, P.oz_passes))
    ozaki_cached_gemm(h, P.oz, P.A, X, Y, false);
  else
    gemm_nn(h, P.A, X, Y);
  h.counters.apply++;
  h.counters.physical_passes++;
}

void op_adjoint(Handle& h, const Problem& P, const DMat& Y, DMat Z) {
  a_ready(h, P);
  if (P.panels.empty() && ozaki_cache_decide(h, P.oz, P.A, Y.cols, P.oz_passes))
    ozaki_cached_gemm(h, P.oz, P.A, Y, Z, true);
  else
    gemm_tn(h, P.A, Y, Z);
  if (P.dist) allreduce_mat(h, Z);
  h.counters.adjoint++;
  h.counters.physical_passes++;
}

// Alg 6's two sketches from one traversal of A (fused.cu): counts one apply,
// one adjoint and ONE physical pass (the CountingOperator contract,
// singlepass.hpp:15-40, plus the single-pass property of Alg 6).  A host
// entry point that streams A in row panels runs one launch per panel as it
// lands (P.panels); otherwise one launch covers A.
void op_dual(Handle& h, const Problem& P, const DMat& Oc, const DMat& Psi, DMat Yc, DMat W) {
  const DMat Ov = tma_view(h, Oc), Pv = tma_view(h, Psi);
  DMat A = P.A;
  if (!tma_ok(A)) {
    a_ready(h, P);
    A = tma_view(h, P.A);
  }
  // RSVD_OZAKI / rsvd_set_ozaki_slices: the same dual product on the INT8
  // tensor cores from exact integer slices of each row panel (ozaki.cu)
  const int oz = ozaki_slices_auto(h, P.m_global, A.cols, Oc.cols);
  OzakiState ost;
  int* sem = oz ? nullptr
                : reinterpret_cast<int*>(h.ws.alloc_bytes(size_t(fused_semaphores(A.rows, A.cols, Oc.cols)) * 4));
  auto panel = [&](int64_t r0, int64_t r1, bool first) {
    if (oz) ozaki_dual_pass(h, A, Ov, Pv, Yc, W, r0, r1, &ost, first, oz);
    else fused_dual_pass(h, A, Ov, Pv, Yc, W, r0, r1, sem, first);
  };
  if (P.panels.empty() || A.p != P.A.p) {
    a_ready(h, P);
    panel(0, A.rows, true);
  } else {
    for (size_t i = 0; i < P.panels.size(); ++i) {
      if (P.panels[i].ready) RSVD_CUDA(cudaStreamWaitEvent(h.stream, P.panels[i].ready, 0));
      panel(P.panels[i].row0, P.panels[i].row1, i == 0);
    }
  }
  if (P.dist) allreduce_mat(h, W);
  h.counters.apply++;
  h.counters.adjoint++;
  h.counters.physical_passes++;
}

Problem make_problem(Handle& h, const double* a, int64_t m, int64_t n, int64_t lda) {
  Problem P;
  P.A = DMat(const_cast<double*>(a), m, n, lda);
  P.dist = h.dist();
  shard_rows(h, m, &P.m_global, &P.row_off);
  return P;
}

// ------------------------------------------------- svd_small / solve_ls
// Square l <= 64: M J = W S  =>  M = W S J^T  (U = W, V = J).
// Tall m >= n:   M = Q R, R^T J = W S  =>  M = (Q J) S W^T: U = Q J, V = W.
// Wide m < n:    M^T = Q R, R^T J = W S =>  M = W S (Q J)^T: U = W, V = Q J.
// One-sided Jacobi runs on the TRANSPOSED triangular factor (Drmac-Veselic
// preconditioning): on numerically rank-deficient / strongly graded factors
// it converges in a third of the sweeps (measured on a 1024 x 512 matrix
// with 500 singular values below u: ~40 sweeps on R, 14 on R^T).
void svd_core(Handle& h, const DMat& M, DMat U, double* s, DMat V) {
  const int64_t m = M.rows, n = M.cols;
  if (m == n && n <= 64) {
    jacobi_svd_square(h, M, V, U, s);
  } else if (m >= n) {  // square n > 64 too: residuals and cores can be graded
    DMat Qm = h.ws.mat(m, n), R = h.ws.mat(n, n), Rt = h.ws.mat(n, n), J = h.ws.mat(n, n);
    orthonormalize(h, M, Qm, &R);
    transpose(h, R, Rt);
    jacobi_svd_square(h, Rt, J, V, s);
    gemm_nn(h, Qm, J, U);
  } else {
    DMat Mt = h.ws.mat(n, m), Qm = h.ws.mat(n, m), R = h.ws.mat(m, m), Rt = h.ws.mat(m, m),
         J = h.ws.mat(m, m);
    transpose(h, M, Mt);
    orthonormalize(h, Mt, Qm, &R);
    transpose(h, R, Rt);
    jacobi_svd_square(h, Rt, J, U, s);
    gemm_nn(h, Qm, J, V);
  }
}

void svd_small_impl(Handle& h, const DMat& M, DMat U, double* s, DMat V) {
  check_finite(h, M, kFlagNonFinite);
  svd_core(h, M, U, s, V);
  sign_rule(h, U, &V);
}

void solve_ls_impl(Handle& h, const DMat& G, const DMat& Hm, DMat X) {
  const int64_t m = G.rows, n = G.cols, r = Hm.cols;
  check_finite(h, G, kFlagNonFinite);
  check_finite(h, Hm, kFlagNonFinite);
  const int64_t k = std::min(m, n);
  DMat U = h.ws.mat(m, k), V = h.ws.mat(n, k);
  double* s = h.ws.alloc(k);
  svd_core(h, G, U, s, V);
  DMat T = h.ws.mat(k, r);
  gemm_tn(h, U, Hm, T);  // U^T H
  launch_k(h, pinv_rows_kernel, grid_for(k * r, h), 256, 0, T.p, k, r, T.ld, s);
  RSVD_LAUNCHED(h);
  gemm_nn(h, V, T, X);
}

void evd_symmetric_impl(Handle& h, const DMat& C, DMat U, double* lambda) {
  check_finite(h, C, kFlagNonFinite);
  check_symmetric(h, C, false);
  DMat S = h.ws.mat(C.rows, C.rows);
  sym_part(h, C, S);
  jacobi_evd_sym(h, S, U, lambda);
}

void solve_joint_core_impl(Handle& h, const DMat& G1, const DMat& H1, const DMat& G2,
                           const DMat& H2, DMat C) {
  const int64_t l = G1.rows;
  for (const DMat* x : {&G1, &H1, &G2, &H2}) check_finite(h, *x, kFlagNonFinite);
  DMat U1 = h.ws.mat(l, l), V1 = h.ws.mat(l, l), U2 = h.ws.mat(l, l), V2 = h.ws.mat(l, l);
  double* s1 = h.ws.alloc(l);
  double* s2 = h.ws.alloc(l);
  if (l > 64) {
    // The two SVDs are independent: one batched block-Jacobi launch, on the
    // transposed triangular factors of QR-preconditioned G1, G2 (as
    // svd_core: G = Q R, R^T J = W S  =>  G = (Q J) S W^T): 10 instead of 13
    // outer sweeps on C5's cores (random-like 550 x 550 G1, G2).
    DMat Q1 = h.ws.mat(l, l), R1 = h.ws.mat(l, l), Q2 = h.ws.mat(l, l), R2 = h.ws.mat(l, l);
    orthonormalize(h, G1, Q1, &R1);
    orthonormalize(h, G2, Q2, &R2);
    DMat R1t = h.ws.mat(l, l), R2t = h.ws.mat(l, l), J1 = h.ws.mat(l, l), J2 = h.ws.mat(l, l);
    transpose(h, R1, R1t);
    transpose(h, R2, R2t);
    block_jacobi_svd2(h, R1t, J1, V1, s1, R2t, J2, V2, s2);  // R^T J = W S: V = W
    gemm_nn(h, Q1, J1, U1);
    gemm_nn(h, Q2, J2, U2);
  } else {
    jacobi_svd_square(h, G1, V1, U1, s1);  // G1 V1 = U1 S1
    jacobi_svd_square(h, G2, V2, U2, s2);
  }
  DMat T = h.ws.mat(l, l), a = h.ws.mat(l, l), b = h.ws.mat(l, l), X = h.ws.mat(l, l);
  gemm_tn(h, U1, H1, T);  // U1^T H1
  gemm_nn(h, T, U2, a);   // (U1^T H1) U2
  gemm_tn(h, V1, H2, T);  // V1^T H2
  gemm_nn(h, T, V2, b);   // (V1^T H2) V2
  launch_k(h, kron_core_kernel, grid_for(l * l, h), 256, 0, a.p, b.p, l, a.ld, s1, s2, X.p, X.ld);
  RSVD_LAUNCHED(h);
  DMat U2t = h.ws.mat(l, l);
  transpose(h, U2, U2t);
  gemm_nn(h, V1, X, T);   // V1 X
  gemm_nn(h, T, U2t, C);  // V1 X U2^T
}

// -------------------------------------------------------- range finders
static void check_sketch_shape(const Problem& P, int64_t k, int64_t p, int q) {
  if (k < 1) throw_param("target rank k must be >= 1");
  if (p < 0) throw_param("oversampling p must be >= 0");
  if (q < 0) throw_param("power steps q must be >= 0");
  const int64_t mn = std::min(P.m_global, P.A.cols);
  if (k + p > mn)
    throw_dim("k+p = " + std::to_string(k + p) + " exceeds min(m,n) = " + std::to_string(mn));
}

void range_basis_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                      DevRng& rng, DMat Q) {
  if (mode == RSVD_MODE_BASIC) q = 0;  // SketchConfig::normalized (rangefinder.hpp:37-41)
  if (mode < 0 || mode > 2) throw_param("unknown range mode");
  check_sketch_shape(P, k, p, q);
  const int64_t n = P.A.cols, ml = P.A.rows, l = k + p;
  if (P.oz_passes == 0) P.oz_passes = 2 * q + 1;
  DMat Omega = h.ws.mat(n, l);
  gaussian_dev(h, n, l, rng, Omega);
  DMat Y = h.ws.mat(ml, l);
  op_apply(h, P, Omega, Y);  // Y = A Omega
  if (mode == RSVD_MODE_POWER) {
    DMat Z = h.ws.mat(n, l);
    for (int j = 0; j < q; ++j) {  // rangefinder.hpp:74-77
      op_adjoint(h, P, Y, Z);
      op_apply(h, P, Z, Y);
    }
    orthonormalize(h, Y, Q, nullptr, P.dist);
  } else if (mode == RSVD_MODE_POWER_ORTHO) {
    orthonormalize(h, Y, Q, nullptr, P.dist);
    DMat Z = h.ws.mat(n, l), W = h.ws.mat(n, l);
    for (int j = 0; j < q; ++j) {  // rangefinder.hpp:89-92
      op_adjoint(h, P, Q, Z);
      orthonormalize(h, Z, W, nullptr, false);  // replicated n x l
      op_apply(h, P, W, Y);
      orthonormalize(h, Y, Q, nullptr, P.dist);
    }
  } else {
    orthonormalize(h, Y, Q, nullptr, P.dist);
  }
}

// Stage 2 after B^T = Z = A^T Q (factor.hpp:14-16): svd_small(B) through the
// QR of Z and a one-sided Jacobi on the TRANSPOSED l x l factor:
//   Z = Qb Rb,  Rb^T J = W S  =>  B = Rb^T Qb^T = W S (Qb J)^T,
//   U_B = W, V = Qb J;  then the sign rule on U_B (core.hpp:115-122) and U = Q U_B.
// On C1's slowly decaying spectrum Jacobi on Rb^T converges in 7 sweeps instead
// of 8 on Rb (C1 3565 vs 3468 factorizations/s); RSVD_STAGE2_RT=0 restores Rb.
void rsvd_stage2(Handle& h, const DMat& Q, const DMat& Z, DMat U, double* sigma, DMat V) {
  const int64_t n = Z.rows, l = Z.cols;
  DMat Qb = h.ws.mat(n, l), Rb = h.ws.mat(l, l), J = h.ws.mat(l, l), W = h.ws.mat(l, l);
  orthonormalize(h, Z, Qb, &Rb, false);
  static const bool rt = [] {
    const char* e = std::getenv("RSVD_STAGE2_RT");
    return !(e && e[0] == '0');
  }();
  if (rt) {
    DMat Rt = h.ws.mat(l, l);
    transpose(h, Rb, Rt);
    jacobi_svd_square(h, Rt, J, W, sigma);
    gemm_nn(h, Qb, J, V);
    sign_rule(h, W, &V);
    gemm_nn(h, Q, W, U);
  } else {  // Rb J = W S  =>  B = J S (Qb W)^T: U_B = J, V = Qb W
    jacobi_svd_square(h, Rb, J, W, sigma);
    gemm_nn(h, Qb, W, V);
    sign_rule(h, J, &V);
    gemm_nn(h, Q, J, U);
  }
}

void rsvd_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode, DevRng& rng,
               DMat U, double* sigma, DMat V) {
  const int64_t n = P.A.cols, ml = P.A.rows, l = k + p;
  check_sketch_shape(P, k, p, mode == RSVD_MODE_BASIC ? 0 : q);
  DMat Q = h.ws.mat(ml, l);
  P.oz_passes = 2 * (mode == RSVD_MODE_BASIC ? 0 : q) + 2;  // the range finder's and Stage 2's
  range_basis_impl(h, P, k, p, q, mode, rng, Q);
  // Stage 2 (factor.hpp:14-16): B = Q^T A is formed transposed, Z = A^T Q.
  DMat Z = h.ws.mat(n, l);
  op_adjoint(h, P, Q, Z);
  rsvd_stage2(h, Q, Z, U, sigma, V);  // svd_small(B), B = Z^T
}

// --------------------------------------------------------- single pass
void spevd_impl(Handle& h, const Problem& P, int64_t k, int64_t p, DevRng& rng, bool check_sym,
                DMat U, double* lambda) {
  const int64_t n = P.A.cols, ml = P.A.rows;
  if (P.m_global != n) throw_dim("spevd_hermitian: matrix is not square");
  if (k < 1) throw_param("spevd_hermitian: k must be >= 1");
  if (p < 0) throw_param("spevd_hermitian: p must be >= 0");
  if (k + p > n) throw_dim("spevd_hermitian: k+p exceeds n");
  // Reference singlepass.hpp:49-53: an uncounted precondition read of A.  It
  // raises a sticky device flag that the call's final check turns into the
  // reference's NumericError (no mid-call host wait, so the call stays
  // graph-replayable); a streamed upload checks once every panel has landed.
  const bool sym_first = check_sym && P.panels.empty();
  if (sym_first) {
    a_ready(h, P);
    if (P.dist)
      check_symmetric_dist(h, P);
    else
      check_symmetric(h, P.A, false);
  }
  const int64_t l = k + p;
  DMat Omega = h.ws.mat(n, l);
  gaussian_dev(h, n, l, rng, Omega);
  DMat Y = h.ws.mat(ml, l);
  {
    struct Cfg {  // see Handle::pass_cfg_big; restored on exceptions too
      Handle& h;
      ~Cfg() { h.pass_cfg_big = 0; }
    } cfg_scope{h};
    h.pass_cfg_big = 1;
    // one product with A: wide sketches (C4: l = 220) take the INT8 path, whose
    // exact integer accumulation does not depend on a summation order (C4's
    // Ritz values sit within 2e-11 of the oracle with it, 5e-11 with DMMA)
    if (P.oz_passes == 0) P.oz_passes = 1;
    op_apply(h, P, Omega, Y);  // the single pass over A
  }
  if (check_sym && !sym_first) {  // streamed upload: once every panel has landed
    a_ready(h, P);
    if (P.dist)
      check_symmetric_dist(h, P);
    else
      check_symmetric(h, P.A, false);
  }
  DMat Q = h.ws.mat(ml, l);
  orthonormalize(h, Y, Q, nullptr, P.dist);
  DMat Oloc(Omega.p + P.row_off, ml, l, Omega.ld);
  DMat g = h.ws.mat(l, l), hm = h.ws.mat(l, l);
  gemm_tn(h, Q, Oloc, g);  // g = Q^T Omega
  gemm_tn(h, Q, Y, hm);    // h = Q^T Y
  if (P.dist) {
    allreduce_mat(h, g);
    allreduce_mat(h, hm);
  }
  DMat gt = h.ws.mat(l, l), ht = h.ws.mat(l, l), X = h.ws.mat(l, l), c = h.ws.mat(l, l);
  transpose(h, g, gt);
  transpose(h, hm, ht);
  solve_ls_impl(h, gt, ht, X);  // C g = h via g^T C^T = h^T
  sym_part(h, X, c);            // c = X^T; c = (c + c^T)/2
  DMat Uc = h.ws.mat(l, l);
  double* lam = h.ws.alloc(l);
  evd_symmetric_impl(h, c, Uc, lam);
  gemm_nn(h, Q, DMat(Uc.p, l, k, Uc.ld), U);
  RSVD_CUDA(cudaMemcpyAsync(lambda, lam, size_t(k) * 8, cudaMemcpyDeviceToDevice, h.stream));
}

void spsvd_impl(Handle& h, const Problem& P, int64_t k, int64_t p, DevRng& rng, DMat U,
                double* sigma, DMat V) {
  const int64_t n = P.A.cols, ml = P.A.rows, m = P.m_global;
  if (k < 1) throw_param("spsvd_general: k must be >= 1");
  if (p < 0) throw_param("spsvd_general: p must be >= 0");
  if (k + p > std::min(m, n)) throw_dim("spsvd_general: k+p exceeds min(m,n)");
  const int64_t l = k + p;
  DMat Oc = h.ws.mat(n, l);
  gaussian_dev(h, n, l, rng, Oc);  // Omega_c
  DMat Psi = h.ws.mat(ml, l);
  gaussian_dev(h, m, l, rng, Psi, P.row_off, P.row_off + ml);  // Omega_r (local rows)
  DMat Yc = h.ws.mat(ml, l), W = h.ws.mat(n, l);
  op_dual(h, P, Oc, Psi, Yc, W);  // Y_c = A Omega_c and Y_r = A^T Omega_r, ONE pass over A
  DMat Qc = h.ws.mat(ml, l), Qr = h.ws.mat(n, l);
  orthonormalize(h, Yc, Qc, nullptr, P.dist);
  orthonormalize(h, W, Qr, nullptr, false);
  DMat G1 = h.ws.mat(l, l), H1 = h.ws.mat(l, l), G2 = h.ws.mat(l, l), H2 = h.ws.mat(l, l);
  gemm_tn(h, Psi, Qc, G1);  // Omega_r^T Q_c
  gemm_tn(h, W, Qr, H1);    // Y_r^T Q_r
  gemm_tn(h, Qr, Oc, G2);   // Q_r^T Omega_c
  gemm_tn(h, Qc, Yc, H2);   // Q_c^T Y_c
  if (P.dist) {
    allreduce_mat(h, G1);
    allreduce_mat(h, H2);
  }
  DMat C = h.ws.mat(l, l);
  solve_joint_core_impl(h, G1, H1, G2, H2, C);
  DMat Uc = h.ws.mat(l, l), Vc = h.ws.mat(l, l);
  double* s = h.ws.alloc(l);
  svd_small_impl(h, C, Uc, s, Vc);
  gemm_nn(h, Qc, DMat(Uc.p, l, k, Uc.ld), U);
  gemm_nn(h, Qr, DMat(Vc.p, l, k, Vc.ld), V);
  RSVD_CUDA(cudaMemcpyAsync(sigma, s, size_t(k) * 8, cudaMemcpyDeviceToDevice, h.stream));
}

}  // namespace rsvdb
