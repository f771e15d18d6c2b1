// Blocked Cholesky + triangular inverse of an l x l Gram on the whole GPU, for
// the CholeskyQR of wide sketches (l > 32: C3 l = 110, C4 l = 220, C5 l = 550),
// replacing a one-CTA right-looking kernel whose l sequential steps each swept
// the trailing matrix through L2 (15 ms at l = 550).
//
// One cooperative launch, 32 x 32 blocks (nb = ceil(l / 32)):
//   for k: [CTA 0] factor A_kk = L_kk L_kk^T and invert it (cta_chol_inv:
//          elimination across the CTA), | grid barrier |
//          [all]   L_ik = A_ik L_kk^-T                  (row blocks i > k),
//          | grid barrier |
//          [all]   A_ij -= L_ik L_jk^T                  (k < j <= i),
//          | grid barrier |
//   then L^-1 by block anti-diagonals d = i - j:
//          X_ij = -X_ii sum_{m=j}^{i-1} L_im X_mj        (all j of one d at once)
//   and R = L^T, R^-1 = (L^-1)^T.
// Shift policy as chol_inv_kernel (small.cu): every pivot is tested against
// 1e-12 of its original diagonal; on breakdown the whole factorization
// restarts once with s = shift_coef * trace(G) added to the diagonal.  All
// decisions are grid-uniform (read after a grid barrier); the block products
// run in a fixed order, so the result is bitwise reproducible.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "cholsmall.cuh"
#include "common.cuh"
#include "small.cuh"

namespace cg = cooperative_groups;

namespace rsvdb {
namespace {

constexpr int kB = 32;
constexpr int kLD = 33;
constexpr int kT = kCholThreads;  // 256: cta_chol_inv runs on the whole CTA

// dst(r, c) (ld kLD) = src(r, c) (trans = false) or src(c, r) (trans = true),
// src column-major with leading dimension ld, rows x cols valid, zero elsewhere.
__device__ __forceinline__ void load_blk(double* dst, const double* src, int64_t ld, int rows, int cols,
                                         bool trans) {
  for (int e = threadIdx.x; e < kB * kB; e += kT) {
    const int r = e & 31, c = e >> 5;
    double v = 0.0;
    if (!trans) {
      if (r < rows && c < cols) v = src[r + ld * c];
    } else {
      if (c < rows && r < cols) v = src[c + ld * r];
    }
    dst[r + kLD * c] = v;
  }
}

// acc[q] += sum_k As(lane, k) Bs(k, warp + 8 q)
__device__ __forceinline__ void mm_acc(double (&acc)[4], const double* As, const double* Bs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 8
  for (int k = 0; k < kB; ++k) {
    const double a = As[lane + kLD * k];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = fma(a, Bs[k + kLD * (warp + 8 * q)], acc[q]);
  }
}

__global__ void __launch_bounds__(kT) chol_blocked_kernel(const double* __restrict__ G, int64_t ldg, int l,
                                                         double shift_coef, double* __restrict__ A,
                                                         double* __restrict__ X, double* __restrict__ R,
                                                         int64_t ldr, double* __restrict__ Rinv, int64_t ldri,
                                                         int* __restrict__ shift_used, int* __restrict__ flags,
                                                         int* __restrict__ status) {
  RSVD_PDL_ENTRY();
  cg::grid_group grid = cg::this_grid();
  __shared__ double S0[kB * kLD], S1[kB * kLD], Rs[kB * kLD], Ri[kB * kLD], piv[2 * 136], orig[kB];
  __shared__ double red[kT / 32];
  const int nb = (l + kB - 1) / kB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t L = l;
  const int64_t gstride = int64_t(gridDim.x) * kT;
  // trace(G), identical in every CTA (fixed reduction order)
  double tr = 0.0;
  for (int j = tid; j < l; j += kT) tr += G[j + ldg * j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
  if (lane == 0) red[warp] = tr;
  __syncthreads();
  tr = 0.0;
  for (int w = 0; w < kT / 32; ++w) tr += red[w];

  int attempt = 0;
  bool broke = true;
  for (; attempt < 2 && broke; ++attempt) {
    const double shift = attempt ? shift_coef * tr : 0.0;
    for (int64_t e = int64_t(blockIdx.x) * kT + tid; e < L * L; e += gstride) {
      const int64_t i = e % L, j = e / L;
      A[e] = (i >= j) ? G[i + ldg * j] + (i == j ? shift : 0.0) : 0.0;
      X[e] = 0.0;
    }
    grid.sync();
    broke = false;
    for (int k = 0; k < nb && !broke; ++k) {
      const int k0 = kB * k, wk = min(kB, l - k0);
      if (blockIdx.x == 0) {
        // symmetric diagonal block from the lower triangle; padding = identity
        for (int e = tid; e < kB * kB; e += kT) {
          const int r = e & 31, c = e >> 5;
          double v = (r == c) ? 1.0 : 0.0;
          if (r < wk && c < wk) v = A[(k0 + max(r, c)) + L * (k0 + min(r, c))];
          S0[r + kLD * c] = v;
        }
        if (tid < kB) orig[tid] = (tid < wk) ? G[(k0 + tid) * (ldg + 1)] + shift : 1.0;
        __syncthreads();
        bool sh;
        const bool ok = cta_chol_inv(S0, kB, 0.0, piv, Rs, Ri, &sh, nullptr, orig, 1);
        if (!ok) {
          if (tid == 0) status[attempt] = 1;
        } else {
          // L_kk = Rs^T, L_kk^-1 = Ri^T (lower)
          for (int e = tid; e < kB * kB; e += kT) {
            const int r = e & 31, c = e >> 5;
            if (r < wk && c < wk && r >= c) {
              A[(k0 + r) + L * (k0 + c)] = Rs[c + kLD * r];
              X[(k0 + r) + L * (k0 + c)] = Ri[c + kLD * r];
            }
          }
        }
      }
      grid.sync();
      broke = *reinterpret_cast<volatile int*>(&status[attempt]) != 0;  // grid-uniform
      if (broke) break;
      // L_ik = A_ik X_kk^T
      for (int ib = k + 1 + blockIdx.x; ib < nb; ib += gridDim.x) {
        const int i0 = kB * ib, wi = min(kB, l - i0);
        load_blk(S0, A + i0 + L * k0, L, wi, wk, false);
        load_blk(S1, X + k0 + L * k0, L, wk, wk, true);  // S1(k, c) = X_kk(c, k)
        __syncthreads();
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        mm_acc(acc, S0, S1);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = warp + 8 * q;
          if (lane < wi && c < wk) A[(i0 + lane) + L * (k0 + c)] = acc[q];
        }
        __syncthreads();
      }
      grid.sync();
      // A_ij -= L_ik L_jk^T for k < jb <= ib (pairs enumerated row by row)
      const int n = nb - k - 1, npairs = n * (n + 1) / 2;
      for (int pidx = blockIdx.x; pidx < npairs; pidx += gridDim.x) {
        int a = int((sqrt(8.0 * pidx + 1.0) - 1.0) * 0.5);
        while (a * (a + 1) / 2 > pidx) --a;
        while ((a + 1) * (a + 2) / 2 <= pidx) ++a;
        const int ib = k + 1 + a, jb = k + 1 + (pidx - a * (a + 1) / 2);
        const int i0 = kB * ib, j0 = kB * jb, wi = min(kB, l - i0), wj = min(kB, l - j0);
        load_blk(S0, A + i0 + L * k0, L, wi, wk, false);
        load_blk(S1, A + j0 + L * k0, L, wj, wk, true);  // S1(k, c) = L_jk(c, k)
        __syncthreads();
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        mm_acc(acc, S0, S1);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = warp + 8 * q;
          if (lane < wi && c < wj && (ib != jb || lane >= c)) A[(i0 + lane) + L * (j0 + c)] -= acc[q];
        }
        __syncthreads();
      }
      grid.sync();
    }
  }
  if (broke) {  // failed after the shifted retry
    if (blockIdx.x == 0 && tid == 0) atomicOr(flags, kFlagCholBreakdown);
    return;
  }
  if (attempt == 2 && blockIdx.x == 0 && tid == 0 && shift_used) *shift_used = 1;
  // L^-1, block anti-diagonal by anti-diagonal
  for (int d = 1; d < nb; ++d) {
    for (int jb = blockIdx.x; jb + d < nb; jb += gridDim.x) {
      const int ib = jb + d;
      const int i0 = kB * ib, j0 = kB * jb, wi = min(kB, l - i0), wj = min(kB, l - j0);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int mb = jb; mb < ib; ++mb) {  // S = sum_m L_im X_mj
        const int m0 = kB * mb, wm = min(kB, l - m0);
        load_blk(S0, A + i0 + L * m0, L, wi, wm, false);
        load_blk(S1, X + m0 + L * j0, L, wm, wj, false);
        __syncthreads();
        mm_acc(acc, S0, S1);
        __syncthreads();
      }
      // X_ij = -X_ii S
#pragma unroll
      for (int q = 0; q < 4; ++q) S1[lane + kLD * (warp + 8 * q)] = acc[q];
      load_blk(S0, X + i0 + L * i0, L, wi, wi, false);
      __syncthreads();
      double out[4] = {0.0, 0.0, 0.0, 0.0};
      mm_acc(out, S0, S1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = warp + 8 * q;
        if (lane < wi && c < wj) X[(i0 + lane) + L * (j0 + c)] = -out[q];
      }
      __syncthreads();
    }
    grid.sync();
  }
  // R = L^T, R^-1 = X^T (upper triangular, zero below)
  for (int64_t e = int64_t(blockIdx.x) * kT + tid; e < L * L; e += gstride) {
    const int64_t i = e % L, c = e / L;
    R[i + ldr * c] = (c >= i) ? A[c + L * i] : 0.0;
    Rinv[i + ldri * c] = (c >= i) ? X[c + L * i] : 0.0;
  }
}

}  // namespace

void chol_inv_blocked(Handle& h, const DMat& G, int l, double shift_coef, DMat R, DMat Rinv,
                      int* shift_used) {
  double* A = h.ws.alloc(int64_t(l) * l);
  double* X = h.ws.alloc(int64_t(l) * l);
  int* status = reinterpret_cast<int*>(h.ws.alloc_bytes(16));
  RSVD_CUDA(cudaMemsetAsync(status, 0, 16, h.stream));
  const int nb = (l + kB - 1) / kB;
  int per_sm = 0;
  RSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_blocked_kernel, kT, 0));
  const int grid = std::max(1, std::min(h.sm_count * std::max(1, per_sm), std::max(nb * (nb + 1) / 2, 1)));
  const double* gp = G.p;
  int64_t ldg = G.ld, ldr = R.ld, ldri = Rinv.ld;
  int lv = l;
  double cf = shift_coef;
  double* rp = R.p;
  double* rip = Rinv.p;
  int* fl = h.d_flags;
  void* args[] = {&gp, &ldg, &lv, &cf, &A, &X, &rp, &ldr, &rip, &ldri, &shift_used, &fl, &status};
  RSVD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(chol_blocked_kernel), dim3(grid),
                                        dim3(kT), args, 0, h.stream));
  RSVD_LAUNCHED(h);
}

}  // namespace rsvdb
