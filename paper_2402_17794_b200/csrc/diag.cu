// Residual and subspace diagnostics on the GPU:
//
//   singular_values        reference core.hpp:180-183
//   spectral_norm          reference core.hpp:188-221  (dense route for
//                          min(m,n) <= 512, else power iteration on M^T M from
//                          the reference's LCG start vector, tol 1e-10, cap 5000)
//   computed_range_error   reference bounds.hpp:107-120 (||A - Q Q^T A||_2)
//   canonical_sines        reference angles.hpp:42-60   (projection route)
//   check_orthonormal      reference angles.hpp:24-35 / bounds.hpp:111-117
//
// B200 mapping.  The residual R = A - Q (A^T Q)^T is one streaming pass for
// A^T Q (pass.cu) plus one rank-l update kernel that reads A once and writes
// R once.  The power iteration is ONE cooperative kernel for all iterations:
// per iteration two HBM-bound matrix-vector sweeps over R (y = R x with
// column chunks, x' = R^T y with one warp per column slice), fixed-order
// reductions between grid barriers, and the convergence test evaluated
// identically in every CTA -- no host round trip per iteration.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "diag.cuh"
#include "engine.cuh"
#include "pass.cuh"
#include "small.cuh"

namespace cg = cooperative_groups;

namespace rsvdb {
namespace {

constexpr int kSnThreads = 256;
constexpr int kSnWarps = kSnThreads / 32;
constexpr int kSnMaxIter = 5000;       // core.hpp:88
constexpr double kSnTol = 1e-10;       // core.hpp:87
constexpr int64_t kSnDenseLimit = 512;  // core.hpp:86

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

// max_ij |G_ij - delta_ij|  (reference: (gram - I).cwiseAbs().maxCoeff())
__global__ void dev_identity_kernel(const double* __restrict__ G, int64_t k, int64_t ld,
                                    double* out) {
  RSVD_PDL_ENTRY();
  double v = 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < k * k;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % k, j = e / k;
    const double d = fabs(G[j * ld + i] - (i == j ? 1.0 : 0.0));
    v = (d > v || d != d) ? d : v;  // NaN propagates like maxCoeff's comparison fails
  }
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, v);
}

// R = A - Q Z^T  (A m x n, Q m x l, Z n x l): one read of A, one write of R.
// 64 x 64 output tile per CTA; thread t owns row t % 64 and 16 columns
// (t / 64) * 16 ...; Q^T / Z panels of 32 along l staged in shared memory.
constexpr int kRT = 64, kRK = 32;
__global__ void __launch_bounds__(256) residual_lowrank_kernel(
    const double* __restrict__ A, int64_t lda, const double* __restrict__ Q, int64_t ldq,
    const double* __restrict__ Z, int64_t ldz, int64_t m, int64_t n, int64_t l,
    double* __restrict__ R, int64_t ldr) {
  RSVD_PDL_ENTRY();
  __shared__ double Qs[kRK][kRT];      // Qs[k][row]
  __shared__ double Zs[kRT][kRK + 1];  // Zs[col][k]
  const int tid = threadIdx.x;
  const int r = tid % kRT, cgp = tid / kRT;
  const int64_t i0 = int64_t(blockIdx.x) * kRT, j0 = int64_t(blockIdx.y) * kRT;
  double acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0.0;
  for (int64_t k0 = 0; k0 < l; k0 += kRK) {
    for (int e = tid; e < kRT * kRK; e += 256) {
      const int rr = e % kRT, kk = e / kRT;
      const int64_t gi = i0 + rr, gk = k0 + kk;
      Qs[kk][rr] = (gi < m && gk < l) ? Q[gk * ldq + gi] : 0.0;
      const int64_t gj = j0 + rr;
      Zs[rr][kk] = (gj < n && gk < l) ? Z[gk * ldz + gj] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kRK; ++kk) {
      const double q = Qs[kk][r];
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = fma(q, Zs[cgp * 16 + c][kk], acc[c]);
    }
    __syncthreads();
  }
  const int64_t gi = i0 + r;
  if (gi >= m) return;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int64_t gj = j0 + cgp * 16 + c;
    if (gj < n) R[gj * ldr + gi] = A[gj * lda + gi] - acc[c];
  }
}

// Fixed-order CTA sum (every CTA that calls it with the same data gets the
// same bits): warp 0 reduces the G values in a fixed lane/shuffle pattern.
__device__ double cta_fixed_sum(const double* __restrict__ v, int G, double* sh) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    double s = 0.0;
    for (int b = tid; b < G; b += 32) s += __ldcg(v + b);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (tid == 0) sh[0] = s;
  }
  __syncthreads();
  const double s = sh[0];
  __syncthreads();
  return s;
}

// CTA sum of per-thread values, result in thread 0 (fixed order).
__device__ double cta_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kSnWarps; ++i) s += sh[i];
  __syncthreads();
  return s;
}

struct SnParams {
  const double* R;
  int64_t m, n, ld;
  int cc;        // column chunks of y = R x
  int64_t ccw;   // columns per chunk
  int rc;        // row chunks of x' = R^T y
  int64_t rcw;   // rows per chunk
  double* x;     // n
  double* xp;    // n
  double* y;     // m
  double* ypart;  // cc x m
  double* xpart;  // rc x n
  double* red;    // 2 x gridDim
  double* out;    // [0] result, [1] iterations
  int* flags;
  int flag_cap;
};

// Power iteration of reference core.hpp:194-220, all iterations in one launch.
__global__ void __launch_bounds__(kSnThreads) spectral_power_kernel(SnParams p) {
  RSVD_PDL_ENTRY();
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kSnWarps + 2];
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t gtid = int64_t(blockIdx.x) * kSnThreads + tid, gthreads = int64_t(G) * kSnThreads;
  const int64_t gwarp = int64_t(blockIdx.x) * kSnWarps + warp, gwarps = int64_t(G) * kSnWarps;
  const double* __restrict__ R = p.R;
  const int64_t m = p.m, n = p.n, ld = p.ld;

  // start vector: LCG fill (core.hpp:196-201), serial by construction; then x /= ||x||
  if (blockIdx.x == 0 && tid == 0) {
    uint64_t state = 0x9e3779b97f4a7c15ULL;
    for (int64_t i = 0; i < n; ++i) {
      state = state * 6364136223846793005ULL + 1442695040888963407ULL;
      p.xp[i] = double(state >> 11) / 9007199254740992.0 - 0.5;
    }
  }
  grid.sync();
  {
    double s = 0.0;
    for (int64_t j = gtid; j < n; j += gthreads) s += p.xp[j] * p.xp[j];
    s = cta_sum(s, sh);
    if (tid == 0) p.red[G + blockIdx.x] = s;
  }
  grid.sync();
  {
    const double xn = sqrt(cta_fixed_sum(p.red + G, G, sh));
    if (xn == 0.0) {
      if (blockIdx.x == 0 && tid == 0) p.out[0] = 0.0;
      return;
    }
    for (int64_t j = gtid; j < n; j += gthreads) p.x[j] = p.xp[j] / xn;
  }
  double sigma = 0.0;
  const int64_t row_tiles = (m + 2 * kSnThreads - 1) / (2 * kSnThreads);
  for (int iter = 0; iter < kSnMaxIter; ++iter) {
    grid.sync();
    // ---- y partials: item = (row tile of 512 rows, column chunk)
    for (int64_t it = blockIdx.x; it < row_tiles * p.cc; it += G) {
      const int64_t rt = it % row_tiles, c = it / row_tiles;
      const int64_t i0 = rt * 2 * kSnThreads + tid, i1 = i0 + kSnThreads;
      const int64_t j0 = c * p.ccw, j1 = min(n, j0 + p.ccw);
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      int64_t j = j0;
      for (; j + 1 < j1; j += 2) {
        const double x0 = __ldcg(p.x + j), x1 = __ldcg(p.x + j + 1);
        if (i0 < m) {
          a0 = fma(__ldg(R + j * ld + i0), x0, a0);
          b0 = fma(__ldg(R + (j + 1) * ld + i0), x1, b0);
        }
        if (i1 < m) {
          a1 = fma(__ldg(R + j * ld + i1), x0, a1);
          b1 = fma(__ldg(R + (j + 1) * ld + i1), x1, b1);
        }
      }
      if (j < j1) {
        const double x0 = __ldcg(p.x + j);
        if (i0 < m) a0 = fma(__ldg(R + j * ld + i0), x0, a0);
        if (i1 < m) a1 = fma(__ldg(R + j * ld + i1), x0, a1);
      }
      if (i0 < m) p.ypart[c * m + i0] = a0 + b0;
      if (i1 < m) p.ypart[c * m + i1] = a1 + b1;
    }
    grid.sync();
    // ---- y = sum of chunks (fixed order), ||y||^2 partials
    {
      double s = 0.0;
      for (int64_t i = gtid; i < m; i += gthreads) {
        double v = 0.0;
        for (int c = 0; c < p.cc; ++c) v += __ldcg(p.ypart + c * m + i);
        p.y[i] = v;
        s += v * v;
      }
      s = cta_sum(s, sh);
      if (tid == 0) p.red[blockIdx.x] = s;
    }
    grid.sync();
    const double est = sqrt(cta_fixed_sum(p.red, G, sh));
    if (est == 0.0) {
      if (blockIdx.x == 0 && tid == 0) {
        p.out[0] = 0.0;
        p.out[1] = iter + 1;
      }
      return;
    }
    if (iter > 0 && fabs(est - sigma) <= kSnTol * est) {
      if (blockIdx.x == 0 && tid == 0) {
        p.out[0] = est;
        p.out[1] = iter + 1;
      }
      return;
    }
    sigma = est;
    // ---- x' partials: item = (column, row chunk), one warp each
    for (int64_t it = gwarp; it < n * p.rc; it += gwarps) {
      const int64_t j = it % n, rchunk = it / n;
      const int64_t r0 = rchunk * p.rcw, r1 = min(m, r0 + p.rcw);
      const double* col = R + j * ld;
      double a = 0.0, b = 0.0;
      int64_t i = r0 + lane;
      for (; i + 32 < r1; i += 64) {
        a = fma(__ldg(col + i), __ldcg(p.y + i), a);
        b = fma(__ldg(col + i + 32), __ldcg(p.y + i + 32), b);
      }
      if (i < r1) a = fma(__ldg(col + i), __ldcg(p.y + i), a);
      a += b;
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) p.xpart[rchunk * n + j] = a;
    }
    grid.sync();
    {
      double s = 0.0;
      for (int64_t j = gtid; j < n; j += gthreads) {
        double v = 0.0;
        for (int c = 0; c < p.rc; ++c) v += __ldcg(p.xpart + c * n + j);
        p.xp[j] = v;
        s += v * v;
      }
      s = cta_sum(s, sh);
      if (tid == 0) p.red[G + blockIdx.x] = s;
    }
    grid.sync();
    const double nx = sqrt(cta_fixed_sum(p.red + G, G, sh));
    if (nx == 0.0) {
      if (blockIdx.x == 0 && tid == 0) {
        p.out[0] = est;
        p.out[1] = iter + 1;
      }
      return;
    }
    for (int64_t j = gtid; j < n; j += gthreads) p.x[j] = __ldcg(p.xp + j) / nx;
  }
  if (blockIdx.x == 0 && tid == 0) {
    p.out[0] = sigma;
    p.out[1] = kSnMaxIter;
    atomicOr(p.flags, p.flag_cap);
  }
}

// out[i] = clamp(sv[count - 1 - i], 0, 1): ascending sines (angles.hpp:53-57)
__global__ void reverse_clamp01_kernel(const double* sv, int64_t count, double* out) {
  RSVD_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = fmin(fmax(sv[count - 1 - i], 0.0), 1.0);
}

// sum of squares of an m x n matrix: per-CTA partials (fixed order), then one
// CTA sums them in CTA order -- deterministic.
__global__ void sumsq_partial_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                                     int64_t lda, double* __restrict__ part) {
  RSVD_PDL_ENTRY();
  __shared__ double sh[kSnWarps + 2];
  double s = 0.0;
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const double v = A[(e / m) * lda + (e % m)];
    s = fma(v, v, s);
  }
  s = cta_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void sum_kernel(const double* __restrict__ part, int G, double* out) {
  RSVD_PDL_ENTRY();
  __shared__ double sh[kSnWarps + 2];
  const double s = cta_fixed_sum(part, G, sh);
  if (threadIdx.x == 0) *out = s;
}

double read_scalar(Handle& h, const double* d) {
  double v = 0.0;
  RSVD_CUDA(cudaMemcpyAsync(&v, d, sizeof(double), cudaMemcpyDeviceToHost, h.stream));
  stream_sync(h);
  return v;
}

}  // namespace

// ------------------------------------------------------------------ host side
void singular_values_impl(Handle& h, const DMat& M, double* s) {
  const int64_t r = std::min(M.rows, M.cols);
  if (r == 0) return;
  check_finite(h, M, kFlagNonFinite);
  DMat U = h.ws.mat(M.rows, r), V = h.ws.mat(M.cols, r);
  svd_core(h, M, U, s, V);
}

double orthonormal_deviation(Handle& h, const DMat& X) {
  const int64_t k = X.cols;
  if (k == 0) return 0.0;
  DMat G = h.ws.mat(k, k);
  gemm_tn(h, X, X, G);
  return gram_deviation(h, G);
}

void gram_deviation_dev(Handle& h, const DMat& G, double* d) {
  const int64_t k = G.rows;
  if (k == 0) return;
  const int blocks = int(std::min<int64_t>(ceil_div(k * k, 256), 2 * h.sm_count));
  launch_k(h, dev_identity_kernel, blocks, 256, 0, G.p, k, G.ld, d);
  RSVD_LAUNCHED(h);
}

double gram_deviation(Handle& h, const DMat& G) {
  const int64_t k = G.rows;
  if (k == 0) return 0.0;
  double* d = h.ws.alloc(1);
  RSVD_CUDA(cudaMemsetAsync(d, 0, sizeof(double), h.stream));
  gram_deviation_dev(h, G, d);
  return read_scalar(h, d);
}

void residual_lowrank(Handle& h, const DMat& A, const DMat& Q, const DMat& Z, DMat R) {
  if (A.rows == 0 || A.cols == 0) return;
  dim3 grid(unsigned(ceil_div(A.rows, kRT)), unsigned(ceil_div(A.cols, kRT)));
  launch_k(h, residual_lowrank_kernel, grid, 256, 0, A.p, A.ld, Q.p, Q.ld, Z.p, Z.ld, A.rows,
                                                       A.cols, Q.cols, R.p, R.ld);
  RSVD_LAUNCHED(h);
}

double frobenius_impl(Handle& h, const DMat& M) {
  if (M.rows == 0 || M.cols == 0) return 0.0;
  const int G = int(std::min<int64_t>(ceil_div(M.rows * M.cols, 256), 4 * h.sm_count));
  double* part = h.ws.alloc(G + 1);
  launch_k(h, sumsq_partial_kernel, G, kSnThreads, 0, M.p, M.rows, M.cols, M.ld, part);
  RSVD_LAUNCHED(h);
  launch_k(h, sum_kernel, 1, kSnThreads, 0, part, G, part + G);
  RSVD_LAUNCHED(h);
  return std::sqrt(read_scalar(h, part + G));
}

void reconstruction_error_impl(Handle& h, const DMat& A, const DMat& U, const double* s,
                               const DMat& V, double* rel_fro, double* rel_spec) {
  const int64_t r = U.cols;
  if (U.rows != A.rows || V.rows != A.cols || V.cols != r)
    throw_dim("reconstruction_error: factor shapes do not match A");
  check_finite(h, A, kFlagNonFinite);
  check_flags(h, "reconstruction_error");
  DMat R = h.ws.mat(A.rows, A.cols);
  if (r == 0) {
    copy(h, A, R);
  } else {
    DMat US = h.ws.mat(A.rows, r);
    copy(h, U, US);
    scale_cols(h, US, s, false);
    residual_lowrank(h, A, US, V, R);  // A - (U diag(s)) V^T
  }
  // drivers.hpp:147-151: ||A - recon||_F / ||A||_F and sigma_max(A - recon) / sigma_max(A)
  const double fro = frobenius_impl(h, A);
  *rel_fro = frobenius_impl(h, R) / (fro > 0.0 ? fro : 1.0);
  const double sa = spectral_norm_impl(h, A, nullptr);
  *rel_spec = spectral_norm_impl(h, R, nullptr) / (sa > 0.0 ? sa : 1.0);
}

double spectral_norm_impl(Handle& h, const DMat& M, int64_t* iterations) {
  const int64_t m = M.rows, n = M.cols;
  if (iterations) *iterations = 0;
  check_finite(h, M, kFlagNonFinite);
  check_flags(h, "spectral_norm");
  if (m == 0 || n == 0) return 0.0;
  if (std::min(m, n) <= kSnDenseLimit) {  // core.hpp:190-192
    double* s = h.ws.alloc(std::min(m, n));
    DMat U = h.ws.mat(m, std::min(m, n)), V = h.ws.mat(n, std::min(m, n));
    svd_core(h, M, U, s, V);
    return read_scalar(h, s);
  }
  int per_sm = 0;
  RSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spectral_power_kernel,
                                                          kSnThreads, 0));
  const int G = std::max(1, std::min(per_sm, 4)) * h.sm_count;
  SnParams p{};
  p.R = M.p;
  p.m = m;
  p.n = n;
  p.ld = M.ld;
  // y = R x: enough (row tile, column chunk) items for ~2 per CTA
  const int64_t row_tiles = ceil_div(m, 2 * kSnThreads);
  p.cc = int(std::max<int64_t>(1, std::min<int64_t>(n, ceil_div(2 * G, row_tiles))));
  p.ccw = ceil_div(n, p.cc);
  p.cc = int(ceil_div(n, p.ccw));
  // x' = R^T y: enough (column, row chunk) warp items for ~2 per warp
  const int64_t warps = int64_t(G) * kSnWarps;
  p.rc = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), ceil_div(2 * warps, n))));
  p.rcw = ceil_div(m, p.rc);
  p.rc = int(ceil_div(m, p.rcw));
  p.x = h.ws.alloc(n);
  p.xp = h.ws.alloc(n);
  p.y = h.ws.alloc(m);
  p.ypart = h.ws.alloc(int64_t(p.cc) * m);
  p.xpart = h.ws.alloc(int64_t(p.rc) * n);
  p.red = h.ws.alloc(2 * G);
  p.out = h.ws.alloc(2);
  p.flags = h.d_flags;
  p.flag_cap = kFlagPowerCap;
  void* args[] = {&p};
  RSVD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(spectral_power_kernel),
                                        dim3(unsigned(G)), dim3(kSnThreads), args, 0, h.stream));
  RSVD_LAUNCHED(h);
  check_flags(h, "spectral_norm");  // the 5000-step cap (core.hpp:220)
  double out[2];
  RSVD_CUDA(cudaMemcpyAsync(out, p.out, sizeof out, cudaMemcpyDeviceToHost, h.stream));
  stream_sync(h);
  if (iterations) *iterations = int64_t(out[1]);
  return out[0];
}

double computed_range_error_impl(Handle& h, const DMat& A, const DMat& Q, DMat* resid) {
  if (Q.rows != A.rows) throw_dim("computed_range_error: row counts differ");
  const double dev = orthonormal_deviation(h, Q);
  if (dev > 1e-8 || dev != dev) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", dev);
    throw_numeric(std::string("computed_range_error: Q is not orthonormal (deviation ") + buf + ")");
  }
  DMat R = resid ? *resid : h.ws.mat(A.rows, A.cols);
  if (Q.cols == 0) {
    copy(h, A, R);
  } else {
    DMat Z = h.ws.mat(A.cols, Q.cols);
    gemm_tn(h, A, Q, Z);  // (Q^T A)^T
    residual_lowrank(h, A, Q, Z, R);
  }
  return spectral_norm_impl(h, R, nullptr);
}

void canonical_sines_impl(Handle& h, const DMat& X, const DMat& Y, double* out) {
  if (X.rows != Y.rows) throw_dim("canonical_sines: ambient dimensions differ");
  for (int w = 0; w < 2; ++w) {
    const DMat& M = w ? Y : X;
    const double dev = orthonormal_deviation(h, M);
    if (dev > 1e-8 || dev != dev) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%f", dev);
      throw_numeric(std::string("canonical_sines: ") + (w ? "Y" : "X") +
                    ": columns are not orthonormal (deviation " + buf + ")");
    }
  }
  const int64_t count = std::min(X.cols, Y.cols);
  if (count == 0) return;
  // residual = Y - X (X^T Y) = Y - X Z^T with Z = Y^T X
  DMat Rs = h.ws.mat(Y.rows, Y.cols);
  if (X.cols == 0) {
    copy(h, Y, Rs);
  } else {
    DMat Z = h.ws.mat(Y.cols, X.cols);
    gemm_tn(h, Y, X, Z);
    residual_lowrank(h, Y, X, Z, Rs);
  }
  const int64_t r = std::min(Rs.rows, Rs.cols);
  double* sv = h.ws.alloc(std::max<int64_t>(r, 1));
  DMat U = h.ws.mat(Rs.rows, r), V = h.ws.mat(Rs.cols, r);
  svd_core(h, Rs, U, sv, V);
  launch_k(h, reverse_clamp01_kernel, unsigned(std::min<int64_t>(ceil_div(count, 256), 64)), 256, 0, 
      sv, count, out);
  RSVD_LAUNCHED(h);
}

}  // namespace rsvdb
