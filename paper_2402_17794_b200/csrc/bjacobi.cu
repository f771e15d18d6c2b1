// Block one-sided Jacobi SVD for l x l factors with l > 64 (BASELINE C3-C5:
// l = 110, 220, 550), replacing the single-CTA kernel whose l - 1 rounds per
// sweep each cost a full block barrier over one SM.
//
//   M J = W diag(sigma):  columns of M are grouped in blocks of kBJ; a sweep is
//   a round-robin over block pairs (nb/2 pairs per round, one CTA each, all in
//   parallel).  A CTA loads its two blocks (l x 2kBJ) into shared memory, runs
//   one inner sweep of one-sided Jacobi on those columns while accumulating
//   the 2kBJ x 2kBJ rotation V, writes the columns back and applies V to the
//   same two block-columns of J.  Rounds are separated by a grid-wide barrier
//   (cooperative launch); a sweep with no rotation above the threshold ends
//   the iteration.  Deterministic: the pair schedule and every reduction are
//   fixed, no atomics on data.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "small.cuh"

namespace cg = cooperative_groups;

namespace rsvdb {
namespace {

constexpr int kBJ = 16;
constexpr int kBJW = 2 * kBJ;
constexpr int kBJThreads = 512;
constexpr int kBJMaxSweeps = 40;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// circle-method partner slots for pair `pr` of round `round` over `np` slots
__device__ __forceinline__ void circle(int pr, int round, int np, int& a, int& b) {
  int ia = pr - 1 + round;
  if (ia >= np - 1) ia -= np - 1;
  int ib = np - 2 - pr + round;
  if (ib >= np - 1) ib -= np - 1;
  a = (pr == 0) ? 0 : 1 + ia;
  b = 1 + ib;
}

__global__ void __launch_bounds__(kBJThreads) bjacobi_kernel(double* __restrict__ X,
                                                            double* __restrict__ Jm, int l,
                                                            int nb, int* __restrict__ changed) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  double* Xb = sm;                            // l x kBJW, ld = l
  double* V = sm + size_t(l) * kBJW;          // kBJW x kBJW, ld = kBJW
  __shared__ int colmap[kBJW];
  __shared__ int any;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const int nbp = nb + (nb & 1);
  // rotation threshold: the rounding noise of an l-term dot product is ~sqrt(l) eps,
  // so a fixed 1e-15 would never report convergence for large l
  const double tol = fmax(1e-15, 2.0 * sqrt(double(l)) * 1.1102230246251565e-16);
  for (int sweep = 0; sweep < kBJMaxSweeps; ++sweep) {
    for (int round = 0; round < nbp - 1; ++round) {
      for (int pr = blockIdx.x; pr < nbp / 2; pr += gridDim.x) {
        int a, b;
        circle(pr, round, nbp, a, b);
        const int I = min(a, b), K = max(a, b);
        if (K >= nb) continue;  // dummy block
        const int wI = min(kBJ, l - I * kBJ), wK = min(kBJ, l - K * kBJ);
        const int w = wI + wK;
        if (tid < w) colmap[tid] = (tid < wI) ? I * kBJ + tid : K * kBJ + (tid - wI);
        if (tid == 0) any = 0;
        __syncthreads();
        for (int e = tid; e < l * w; e += blockDim.x) {
          const int r = e % l, c = e / l;
          Xb[c * l + r] = X[int64_t(colmap[c]) * l + r];
        }
        for (int e = tid; e < kBJW * kBJW; e += blockDim.x)
          V[e] = ((e % kBJW) == (e / kBJW)) ? 1.0 : 0.0;
        __syncthreads();
        // one inner sweep over the w columns, one warp per column pair
        const int wp = w + (w & 1);
        for (int r2 = 0; r2 < wp - 1; ++r2) {
          for (int q = warp; q < wp / 2; q += nwarps) {
            int pa, pb;
            circle(q, r2, wp, pa, pb);
            const int p0 = min(pa, pb), q0 = max(pa, pb);
            if (q0 >= w) continue;
            double al = 0, be = 0, ga = 0;
            for (int i = lane; i < l; i += 32) {
              const double xp = Xb[p0 * l + i], xq = Xb[q0 * l + i];
              al = fma(xp, xp, al);
              be = fma(xq, xq, be);
              ga = fma(xp, xq, ga);
            }
            al = wsum(al);
            be = wsum(be);
            ga = wsum(ga);
            if (fabs(ga) > tol * sqrt(al * be) && ga != 0.0) {
              const double d = be - al, g2 = 2.0 * ga;
              const double t = copysign(1.0, d) * g2 / (fabs(d) + sqrt(d * d + g2 * g2));
              const double c = rsqrt(1.0 + t * t), s = c * t;
              for (int i = lane; i < l; i += 32) {
                const double xp = Xb[p0 * l + i], xq = Xb[q0 * l + i];
                Xb[p0 * l + i] = c * xp - s * xq;
                Xb[q0 * l + i] = s * xp + c * xq;
              }
              if (lane < w) {
                const double vp = V[p0 * kBJW + lane], vq = V[q0 * kBJW + lane];
                V[p0 * kBJW + lane] = c * vp - s * vq;
                V[q0 * kBJW + lane] = s * vp + c * vq;
              }
              if (lane == 0) any = 1;
            }
          }
          __syncthreads();
        }
        for (int e = tid; e < l * w; e += blockDim.x) {
          const int r = e % l, c = e / l;
          X[int64_t(colmap[c]) * l + r] = Xb[c * l + r];
        }
        // J(:, block cols) <- J(:, block cols) * V, one row per thread
        for (int r = tid; r < l; r += blockDim.x) {
          double jr[kBJW];
#pragma unroll
          for (int c = 0; c < kBJW; ++c) jr[c] = (c < w) ? Jm[int64_t(colmap[c]) * l + r] : 0.0;
#pragma unroll 4
          for (int c = 0; c < kBJW; ++c) {
            if (c >= w) break;
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < kBJW; ++k) acc = fma(jr[k], V[c * kBJW + k], acc);
            Jm[int64_t(colmap[c]) * l + r] = acc;
          }
        }
        if (tid == 0 && any) atomicOr(&changed[sweep], 1);
        __syncthreads();
      }
      grid.sync();
    }
    const int done = (*reinterpret_cast<volatile int*>(&changed[sweep]) == 0);
    if (done) return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) changed[kBJMaxSweeps] = 1;  // no convergence
}

// column norms (sigma), stable descending order, permuted outputs
__global__ void bj_norms_kernel(const double* __restrict__ X, int l, double* __restrict__ nrm) {
  const int c = blockIdx.x;
  double s = 0;
  for (int i = threadIdx.x; i < l; i += blockDim.x) s = fma(X[int64_t(c) * l + i], X[int64_t(c) * l + i], s);
  __shared__ double red[8];
  s = wsum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    nrm[c] = sqrt(t);
  }
}

__global__ void bj_order_kernel(const double* __restrict__ nrm, int l, int* __restrict__ order,
                                double* __restrict__ sigma) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < l; j += gridDim.x * blockDim.x) {
    const double v = nrm[j];
    int rank = 0;
    for (int k = 0; k < l; ++k) {
      const double u = nrm[k];
      if (u > v || (u == v && k < j)) ++rank;
    }
    order[rank] = j;
    sigma[rank] = v;
  }
}

__global__ void bj_permute_kernel(const double* __restrict__ X, const double* __restrict__ Jm,
                                  const double* __restrict__ nrm, const int* __restrict__ order,
                                  int l, double* __restrict__ Jout, int64_t ldj,
                                  double* __restrict__ Wout, int64_t ldw, int* __restrict__ nzero) {
  const int jn = blockIdx.x;
  const int src = order[jn];
  const double smax = nrm[order[0]];
  const double s = nrm[src];
  const bool valid = s > 0.0 && s > smax * 1e-300;
  for (int i = threadIdx.x; i < l; i += blockDim.x) {
    Jout[int64_t(jn) * ldj + i] = Jm[int64_t(src) * l + i];
    Wout[int64_t(jn) * ldw + i] = valid ? X[int64_t(src) * l + i] / s : 0.0;
  }
  if (!valid && threadIdx.x == 0) atomicAdd(nzero, 1);
}

// Complete zero columns of W to an orthonormal set (rank-deficient factors):
// candidate unit vectors, two Gram-Schmidt passes.  Runs only when needed.
__global__ void bj_complete_kernel(const double* __restrict__ sigma, int l, double* __restrict__ W,
                                   int64_t ldw, const int* __restrict__ nzero) {
  if (*nzero == 0) return;
  const int lane = threadIdx.x;
  const double smax = sigma[0];
  for (int jn = 0; jn < l; ++jn) {
    const double s = sigma[jn];
    if (s > 0.0 && s > smax * 1e-300) continue;
    double bestn = -1.0;
    int besti = 0;
    for (int cand = 0; cand < l; ++cand) {
      double part = 0.0;
      for (int k = lane; k < l; k += 32) {
        if (k == jn) continue;
        const double sk = sigma[k];
        const bool valid = (k < jn) || (sk > 0.0 && sk > smax * 1e-300);
        if (valid) part += W[int64_t(k) * ldw + cand] * W[int64_t(k) * ldw + cand];
      }
      const double r2 = 1.0 - wsum(part);
      if (r2 > bestn + 1e-12) {
        bestn = r2;
        besti = cand;
      }
    }
    for (int i = lane; i < l; i += 32) W[int64_t(jn) * ldw + i] = (i == besti) ? 1.0 : 0.0;
    __syncwarp();
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = 0; k < l; ++k) {
        if (k == jn) continue;
        const double sk = sigma[k];
        const bool valid = (k < jn) || (sk > 0.0 && sk > smax * 1e-300);
        if (!valid) continue;
        double d = 0;
        for (int i = lane; i < l; i += 32) d += W[int64_t(k) * ldw + i] * W[int64_t(jn) * ldw + i];
        d = wsum(d);
        for (int i = lane; i < l; i += 32) W[int64_t(jn) * ldw + i] -= d * W[int64_t(k) * ldw + i];
        __syncwarp();
      }
      double nn = 0;
      for (int i = lane; i < l; i += 32) nn += W[int64_t(jn) * ldw + i] * W[int64_t(jn) * ldw + i];
      nn = sqrt(wsum(nn));
      for (int i = lane; i < l; i += 32) W[int64_t(jn) * ldw + i] /= nn;
      __syncwarp();
    }
  }
}

__global__ void bj_init_kernel(const double* __restrict__ Rm, int64_t ldr, int l,
                               double* __restrict__ X, double* __restrict__ Jm) {
  const int64_t n = int64_t(l) * l;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e % l), j = int(e / l);
    X[e] = Rm[int64_t(j) * ldr + i];
    Jm[e] = (i == j) ? 1.0 : 0.0;
  }
}

__global__ void bj_flag_kernel(const int* changed, int* flags) {
  if (changed[kBJMaxSweeps]) atomicOr(flags, kFlagJacobiNoConv);
}

// mu >= max_i sum_j |c_ij| >= |lambda|_max (Gershgorin): C + mu I is PSD.
__global__ void gershgorin_kernel(const double* __restrict__ C, int64_t ldc, int l,
                                  double* __restrict__ mu) {
  __shared__ double red[32];
  double m = 0.0;
  for (int i = threadIdx.x; i < l; i += blockDim.x) {
    double sacc = 0.0;
    for (int j = 0; j < l; ++j) sacc += fabs(C[int64_t(j) * ldc + i]);
    m = fmax(m, sacc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    *mu = 1.0625 * t + 1e-300;
  }
}

__global__ void shift_copy_kernel(const double* __restrict__ C, int64_t ldc, int l,
                                  const double* __restrict__ mu, double* __restrict__ T) {
  const int64_t n = int64_t(l) * l;
  const double m = *mu;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e % l), j = int(e / l);
    T[e] = C[int64_t(j) * ldc + i] + (i == j ? m : 0.0);
  }
}

// lambda = sigma - mu, reordered by |lambda| descending; exact ties: positive
// first (see evd_symmetric in small.cu / the oracle).
__global__ void evd_order_kernel(const double* __restrict__ sigma, const double* __restrict__ mu,
                                 const double* __restrict__ Jm, int64_t ldj, int l,
                                 double* __restrict__ U, int64_t ldu, double* __restrict__ lambda,
                                 int* __restrict__ order) {
  const double m = *mu;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < l; j += gridDim.x * blockDim.x) {
    const double v = sigma[j] - m;
    int rank = 0;
    for (int k = 0; k < l; ++k) {
      const double u = sigma[k] - m;
      if (fabs(u) > fabs(v) || (fabs(u) == fabs(v) && (u > v || (u == v && k < j)))) ++rank;
    }
    order[rank] = j;
    lambda[rank] = v;
  }
}

__global__ void evd_permute_kernel(const double* __restrict__ Jm, int64_t ldj, int l,
                                   const int* __restrict__ order, double* __restrict__ U,
                                   int64_t ldu) {
  const int jn = blockIdx.x, src = order[jn];
  for (int i = threadIdx.x; i < l; i += blockDim.x) U[int64_t(jn) * ldu + i] = Jm[int64_t(src) * ldj + i];
}

}  // namespace

void block_jacobi_svd(Handle& h, const DMat& Rm, DMat J, DMat W, double* sigma) {
  const int l = int(Rm.rows);
  const int nb = (l + kBJ - 1) / kBJ;
  double* X = h.ws.alloc(int64_t(l) * l);
  double* Jm = h.ws.alloc(int64_t(l) * l);
  double* nrm = h.ws.alloc(l);
  int* order = reinterpret_cast<int*>(h.ws.alloc_bytes(size_t(l) * 4 + 16));
  int* changed = reinterpret_cast<int*>(h.ws.alloc_bytes((kBJMaxSweeps + 2) * 4));
  int* nzero = changed + kBJMaxSweeps + 1;
  RSVD_CUDA(cudaMemsetAsync(changed, 0, (kBJMaxSweeps + 2) * 4, h.stream));
  bj_init_kernel<<<std::max(1, std::min(4 * h.sm_count, (l * l + 255) / 256)), 256, 0, h.stream>>>(
      Rm.p, Rm.ld, l, X, Jm);
  RSVD_LAUNCHED(h);
  const size_t smem = (size_t(l) * kBJW + kBJW * kBJW) * 8;
  if (smem > 227 * 1024) throw_dim("block_jacobi_svd: l too large for one block pair in shared memory");
  static size_t cur = 0;
  if (smem > cur) {
    RSVD_CUDA(cudaFuncSetAttribute(bjacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
    cur = smem;
  }
  int nbv = nb;
  int lv = l;
  const int nbp = nb + (nb & 1);
  int grid = std::max(1, std::min(nbp / 2, h.sm_count));
  void* args[] = {&X, &Jm, &lv, &nbv, &changed};
  RSVD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bjacobi_kernel), dim3(grid),
                                        dim3(kBJThreads), args, smem, h.stream));
  RSVD_LAUNCHED(h);
  bj_flag_kernel<<<1, 1, 0, h.stream>>>(changed, h.d_flags);
  RSVD_LAUNCHED(h);
  bj_norms_kernel<<<l, 256, 0, h.stream>>>(X, l, nrm);
  RSVD_LAUNCHED(h);
  bj_order_kernel<<<(l + 255) / 256, 256, 0, h.stream>>>(nrm, l, order, sigma);
  RSVD_LAUNCHED(h);
  bj_permute_kernel<<<l, 128, 0, h.stream>>>(X, Jm, nrm, order, l, J.p, J.ld, W.p, W.ld, nzero);
  RSVD_LAUNCHED(h);
  bj_complete_kernel<<<1, 32, 0, h.stream>>>(sigma, l, W.p, W.ld, nzero);
  RSVD_LAUNCHED(h);
}

// Symmetric EVD for l > 64: the SVD of the positive semidefinite C + mu I
// (right singular vectors = eigenvectors, sigma = lambda + mu).  Eigenvalues
// carry an absolute error ~eps * ||C||, the accuracy class of the reference's
// tridiagonal-QR eigensolver.
void evd_shifted(Handle& h, const DMat& C, DMat U, double* lambda) {
  const int l = int(C.rows);
  double* mu = h.ws.alloc(1);
  gershgorin_kernel<<<1, 256, 0, h.stream>>>(C.p, C.ld, l, mu);
  RSVD_LAUNCHED(h);
  DMat T = h.ws.mat(l, l), Jm = h.ws.mat(l, l), W = h.ws.mat(l, l);
  shift_copy_kernel<<<std::max(1, std::min(4 * h.sm_count, (l * l + 255) / 256)), 256, 0, h.stream>>>(
      C.p, C.ld, l, mu, T.p);
  RSVD_LAUNCHED(h);
  double* sg = h.ws.alloc(l);
  block_jacobi_svd(h, DMat(T.p, l, l, l), Jm, W, sg);
  int* order = reinterpret_cast<int*>(h.ws.alloc_bytes(size_t(l) * 4 + 16));
  evd_order_kernel<<<(l + 255) / 256, 256, 0, h.stream>>>(sg, mu, Jm.p, Jm.ld, l, U.p, U.ld, lambda,
                                                         order);
  RSVD_LAUNCHED(h);
  evd_permute_kernel<<<l, 128, 0, h.stream>>>(Jm.p, Jm.ld, l, order, U.p, U.ld);
  RSVD_LAUNCHED(h);
}

}  // namespace rsvdb
