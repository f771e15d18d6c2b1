// Small (l <= 32) Cholesky + inverse on one CTA, shared by small.cu's
// kernels and tools/microbench (header-only device code).
#pragma once
#include <cuda_runtime.h>

namespace rsvdb {

// l <= 32: the Cholesky factor R (G = R^T R) of the (possibly shifted) Gram
// and its inverse, by one 256-thread CTA, as right-looking elimination on the
// augmented rows [G | I] (64 wide):  E G = U with E unit lower triangular,
// U = D Lt^T (G = Lt D Lt^T), so  R = D^-1/2 U  and  R^-1 = E^T D^-1/2.
// Thread t owns row i = t / 8, positions 8 (t % 8) .. +7, in registers (a row's
// eight threads are in one warp).  Step j: the pivot row goes to shared memory
// with r_j = 1/d_j (d_j = U(j,j) = L(j,j)^2, the Cholesky breakdown test
// applies unchanged), one CTA barrier, and every row i > j does
// w_i -= (w_ij r_j) w_j on its 8 positions.  Positions left of the live
// window only touch eliminated entries; E columns right of it are exact zeros
// in the pivot row.  The dependency chain per step is the pivot's rsqrt, a
// shared-memory round trip and one FMA: a single warp doing the same work is
// shared-memory and issue bound (~4x slower, measured).
// Shift policy as chol_inv_kernel.  Returns false (in every thread) on
// breakdown after shifting.  G0 (LD 33, shared) is the Gram; piv is 2 x 136
// doubles of shared scratch (two pivot rows per barrier, double-buffered); outputs R and R^-1 (LD 33, zero outside l x l).
// Must be called by all threads of a 256-thread block.
constexpr int kCholThreads = 256;

// `orig` (optional, shared): the reference diagonal of the breakdown test
// (default: G0's diagonal + shift); `attempts` = 1 disables the shifted retry
// (the blocked factorization of chol_blocked_kernel decides shifts globally);
// `start` = 1 goes straight to the shifted factorization.
// Shared scratch (doubles) cta_chol_inv needs for `piv`: two pivot-row
// buffers of 136 (64 + 8 row-j words, 64 row-(j+1) words) per barrier pair.
constexpr int kCholPivScratch = 2 * 136;

__device__ __forceinline__ bool cta_chol_inv(const double* G0, int l, double shift_coef, double* piv, double* Rs,
                                             double* Rinvs, bool* shifted, long long* pr = nullptr,
                                             const double* orig = nullptr, int attempts = 2,
                                             int start = 0) {
  constexpr int LD = 33;
  constexpr unsigned kFull = 0xffffffffu;
  const int t = threadIdx.x, i = t >> 3, c = t & 7, base = (t & 31) & ~7;
  if (pr && t == 0) pr[0] = clock64();
  const bool row = i < l;
  double tr = 0.0;
  for (int k = 0; k < l; ++k) tr += G0[k + LD * k];  // identical in every thread
  double w[8];
  bool ok = false;
  *shifted = false;
#pragma unroll 1
  for (int attempt = start; attempt < attempts && !ok; ++attempt) {
    const double shift = attempt ? shift_coef * tr : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int p = 8 * c + q;
      double v = 0.0;
      if (row && p < l) v = G0[i + LD * p] + (p == i ? shift : 0.0);
      if (row && p == 32 + i) v = 1.0;
      w[q] = v;
    }
    bool broke = false;
#pragma unroll 1
    for (int jb = 0; jb * 8 < l && !broke; ++jb) {
#pragma unroll
      for (int jj = 0; jj < 8; jj += 2) {
        const int j = 8 * jb + jj;
#ifdef CHOL_STEP_PROBE
        if (pr && t == 0 && j < l) pr[8 + j] = clock64();
#endif
        if (j < l && !broke) {
          // Two pivots (j, j+1) per barrier.  Row j+1 is stored as it stands
          // before step j (pv[72..]); after the barrier every thread applies
          // step j to it itself (its 8 columns and the scalars at columns j,
          // j+1), takes the rsqrt of the updated pivot d1 and applies step
          // j+1: the same operations in the same order as one step per
          // barrier, so the factor is bitwise unchanged.  w_ij, w_i,j+1 (final
          // since step j-1) and the breakdown references are fetched before
          // the barrier.
          const bool two = j + 1 < l;  // uniform
          double* pv = piv + ((j >> 1) & 1) * 136;
          const double wij = __shfl_sync(kFull, w[jj], base + jb);
          const double wij1 = __shfl_sync(kFull, w[jj + 1], base + jb);
          const double oj = orig ? orig[j] : G0[j + LD * j] + shift;
          const double oj1 = two ? (orig ? orig[j + 1] : G0[(j + 1) + LD * (j + 1)] + shift) : 1.0;
          // pivot-row column 8c+q lives at pv[8q+c]: the 8 lane groups of a
          // warp touch 8 consecutive words (at pv[8c+q], 4-way bank conflicts)
          if (i == j) {
#pragma unroll
            for (int q = 0; q < 8; ++q) pv[8 * q + c] = w[q];
            if (c == jb) {
              const double d = w[jj];
              const double rs = rsqrt(d);
              pv[64] = rs * rs;
              pv[65] = d;
            }
          }
          if (two && i == j + 1) {
#pragma unroll
            for (int q = 0; q < 8; ++q) pv[72 + 8 * q + c] = w[q];
          }
          __syncthreads();
          const double d = pv[65], ivd = pv[64];
          const double f = wij * ivd;
          bool bad = !(d > 1e-12 * oj) || !(d > 0.0);
          if (two) {
            const double fj = pv[72 + 8 * jj + jb] * ivd;  // f_{j+1,j}
            const double d1 = fma(-fj, pv[8 * (jj + 1) + jb], pv[72 + 8 * (jj + 1) + jb]);
            if (i > j + 1) {
              const double wi1 = fma(-f, pv[8 * (jj + 1) + jb], wij1);  // w_i,j+1 after step j
              const double rs1 = rsqrt(d1);
              const double f2 = wi1 * (rs1 * rs1);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const double wq = fma(-f, pv[8 * q + c], w[q]);
                w[q] = fma(-f2, fma(-fj, pv[8 * q + c], pv[72 + 8 * q + c]), wq);
              }
            } else if (i == j + 1) {
#pragma unroll
              for (int q = 0; q < 8; ++q) w[q] = fma(-f, pv[8 * q + c], w[q]);
            }
            bad = bad || !(d1 > 1e-12 * oj1) || !(d1 > 0.0);
          } else if (i > j) {
#pragma unroll
            for (int q = 0; q < 8; ++q) w[q] = fma(-f, pv[8 * q + c], w[q]);
          }
          if (bad) broke = true;  // identical in every thread
        }
      }
    }
    ok = !broke;
    if (ok && attempt == 1) *shifted = true;
    __syncthreads();  // piv reuse across attempts
  }
  if (!ok) return false;
  if (pr && t == 0) pr[1] = clock64();
  // s_i = U(i,i)^-1/2 from the diagonal owner (thread i*8 + i/8, slot i%8)
  double dg = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (8 * c + q == i) dg = w[q];
  dg = __shfl_sync(kFull, dg, base + (i >> 3));
  const double si = row ? rsqrt(dg) : 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int p = 8 * c + q;
    if (p < 32)
      Rs[i + LD * p] = (row && p >= i && p < l) ? w[q] * si : 0.0;
    else
      Rinvs[(p - 32) + LD * i] = (row && p - 32 <= i) ? w[q] * si : 0.0;
  }
  __syncthreads();
  if (pr && t == 0) pr[2] = clock64();
  return true;
}

}  // namespace rsvdb
