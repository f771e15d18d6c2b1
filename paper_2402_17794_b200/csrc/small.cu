// Small dense kernels: orthonormalization, l x l Jacobi SVD / EVD, sign rule.
//
// Reference counterparts (core.hpp): orthonormalize :96-105 (Eigen
// HouseholderQR), svd_small :111-124 (Eigen BDCSVD + sign rule), evd_symmetric
// :130-162 (SelfAdjointEigenSolver + |lambda| sort).
//
// B200 design:
//  * Householder TSQR for l <= 64: every CTA factors a 128/256-row block in
//    shared memory (warp-per-column reflector updates), the R factors are
//    stacked and factored again until one block remains, and Q is formed
//    top-down by applying each level's reflectors to the parent's Q rows.
//    Householder keeps the reference's numerics (any conditioning, exact rank
//    deficiency padded to full width) with only l x l data between blocks.
//  * CholeskyQR2 for l > 64 (well-conditioned sketches, BASELINE C3-C5): Gram
//    X^T X on the DMMA pass engine, Cholesky + triangular inverse of the l x l
//    factor on chip, Q = X R^-1 on the pass engine, repeated twice; a shifted
//    first pass (shifted CholeskyQR3) when the Gram is not numerically SPD.
//  * One-sided Jacobi (Hestenes) on the l x l R factor for svd_small: round-
//    robin parallel ordering, one warp per column pair, whole matrix resident
//    in shared memory for l <= 112, L2-resident otherwise.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "dist.cuh"
#include "pass.cuh"
#include "small.cuh"
#include "diag.cuh"
#include "cholsmall.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace rsvdb {

namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ Householder
// Factor one block of `rows_blk` rows (zero padded to b) of X in shared
// memory.  Writes Householder vectors (unit diagonal implied) to V (ld b, one
// b x l panel per block), tau (l per block) and the l x l R into Rstack rows
// [blk*l, blk*l + l) (ld ldr).
__global__ void hh_factor_kernel(const double* __restrict__ X, int64_t rows, int l, int64_t ldx,
                                 int b, double* __restrict__ V, double* __restrict__ tau,
                                 double* __restrict__ Rs, int64_t ldr, int* flags) {
  RSVD_PDL_ENTRY();
  extern __shared__ double sm[];
  double* A = sm;                  // b x l, ld = b
  double* red = sm + int64_t(b) * l;  // scratch: tau/beta broadcast
  const int blk = blockIdx.x;
  const int64_t r0 = int64_t(blk) * b;
  const int nthr = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = nthr >> 5;
  bool bad = false;
  for (int64_t e = tid; e < int64_t(b) * l; e += nthr) {
    const int i = int(e % b), j = int(e / b);
    double v = 0.0;
    if (r0 + i < rows) {
      v = X[j * ldx + r0 + i];
      if (!isfinite(v)) bad = true;
    }
    A[e] = v;
  }
  if (bad) atomicOr(flags, kFlagNonFinite);
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    if (warp == 0) {
      double s = 0.0;
      for (int i = j + 1 + lane; i < b; i += 32) {
        const double v = A[j * b + i];
        s += v * v;
      }
      s = warp_sum(s);
      if (lane == 0) {
        const double alpha = A[j * b + j];
        double t = 0.0, beta = alpha, scal = 0.0;
        if (s > 0.0) {
          const double nrm = sqrt(alpha * alpha + s);
          beta = alpha >= 0.0 ? -nrm : nrm;
          t = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        red[0] = t;
        red[1] = beta;
        red[2] = scal;
      }
    }
    __syncthreads();
    const double t = red[0], beta = red[1], scal = red[2];
    if (t != 0.0)
      for (int i = j + 1 + tid; i < b; i += nthr) A[j * b + i] *= scal;
    __syncthreads();
    if (tid == 0) A[j * b + j] = beta;
    if (t != 0.0) {
      for (int c = j + 1 + warp; c < l; c += nwarps) {
        double w = (lane == 0) ? A[c * b + j] : 0.0;
        for (int i = j + 1 + lane; i < b; i += 32) w += A[j * b + i] * A[c * b + i];
        w = warp_sum(w) * t;
        if (lane == 0) A[c * b + j] -= w;
        for (int i = j + 1 + lane; i < b; i += 32) A[c * b + i] -= w * A[j * b + i];
      }
    }
    if (tid == 0) tau[int64_t(blk) * l + j] = t;
    __syncthreads();
  }
  // outputs
  double* Vb = V + int64_t(blk) * b * l;
  for (int64_t e = tid; e < int64_t(b) * l; e += nthr) Vb[e] = A[e];
  for (int64_t e = tid; e < int64_t(l) * l; e += nthr) {
    const int i = int(e % l), j = int(e / l);
    Rs[j * ldr + int64_t(blk) * l + i] = (i <= j) ? A[j * b + i] : 0.0;
  }
}

// Q_blk = H_1 ... H_l [C_blk; 0], C_blk = rows [blk*l, blk*l+l) of the parent
// Q (ld ldc) or the identity when C == nullptr.  Writes the real rows of the
// block into Q (ld ldq).
__global__ void hh_apply_kernel(const double* __restrict__ V, const double* __restrict__ tau,
                                int64_t rows, int l, int b, const double* __restrict__ C,
                                int64_t ldc, double* __restrict__ Q, int64_t ldq) {
  RSVD_PDL_ENTRY();
  extern __shared__ double sm[];
  double* M = sm;                  // b x l
  double* Vs = sm + int64_t(b) * l;  // b x l
  const int blk = blockIdx.x;
  const int64_t r0 = int64_t(blk) * b;
  const int nthr = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = nthr >> 5;
  const double* Vb = V + int64_t(blk) * b * l;
  for (int64_t e = tid; e < int64_t(b) * l; e += nthr) {
    const int i = int(e % b), j = int(e / b);
    Vs[e] = Vb[e];
    double v = 0.0;
    if (i < l) v = C ? C[j * ldc + int64_t(blk) * l + i] : (i == j ? 1.0 : 0.0);
    M[e] = v;
  }
  __syncthreads();
  for (int j = l - 1; j >= 0; --j) {
    const double t = tau[int64_t(blk) * l + j];
    if (t != 0.0) {
      for (int c = warp; c < l; c += nwarps) {
        double w = (lane == 0) ? M[c * b + j] : 0.0;
        for (int i = j + 1 + lane; i < b; i += 32) w += Vs[j * b + i] * M[c * b + i];
        w = warp_sum(w) * t;
        if (lane == 0) M[c * b + j] -= w;
        for (int i = j + 1 + lane; i < b; i += 32) M[c * b + i] -= w * Vs[j * b + i];
      }
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < int64_t(b) * l; e += nthr) {
    const int i = int(e % b), j = int(e / b);
    if (r0 + i < rows) Q[j * ldq + r0 + i] = M[e];
  }
}

int tsqr_block_rows(int l) { return l <= 32 ? 256 : 128; }

// ---------------------------------------------------------- one-sided Jacobi
// Rm J = W diag(sigma) for square l x l Rm.  Single CTA; X, J in smem when
// `in_smem`, otherwise in the global scratch buffers gX / gJ (L2 resident).
template <int GS>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = GS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// GS lanes per column pair: 32 (one warp) for large l, 8 for l <= 64 (fewer
// shuffle levels and 4 pairs per warp: the round latency is the bottleneck).
// Rotation threshold of the one-sided Jacobi sweeps (|g| > tol sqrt(a b)):
// the rounding noise of an l-term dot product is ~sqrt(l) u, so a fixed 1e-15
// would never report convergence for large l.  (Measured: l u instead of
// 2 sqrt(l) u changes neither the sweep count nor the time on C1/C2.)
__device__ __forceinline__ double jacobi_tol(int l) {
  return fmax(1e-15, 2.0 * sqrt(double(l)) * 1.1102230246251565e-16);
}

template <int GS>
__global__ void jacobi_svd_kernel(const double* __restrict__ Rm, int64_t ldr, int l,
                                  double* __restrict__ Jout, int64_t ldj,
                                  double* __restrict__ Wout, int64_t ldw,
                                  double* __restrict__ sigma, double* gX, double* gJ,
                                  int in_smem, int* flags, double* dbg = nullptr) {
  RSVD_PDL_ENTRY();
  extern __shared__ double sm[];
  __shared__ double wmax_s[32];  // per warp: largest g^2/(a b) met this sweep
  double m_prev = 1.0;           // previous sweep's maximum (identical in all threads)
  double* X = in_smem ? sm : gX;
  double* J = in_smem ? sm + int64_t(l) * l : gJ;
  __shared__ int changed;  // any rotation this sweep
  __shared__ int order[1024];
  __shared__ double nrm[1024];
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = nthr >> 5;
  for (int64_t e = tid; e < int64_t(l) * l; e += nthr) {
    const int i = int(e % l), j = int(e / l);
    X[e] = Rm[j * ldr + i];
    J[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int lp = l + (l & 1);  // even number of slots (one dummy if odd)
  // rotation threshold: the rounding noise of an l-term dot product is ~sqrt(l) eps,
  // so a fixed 1e-15 would never report convergence for large l
  const double tol = jacobi_tol(l);
  int sweep = 0;
  // l <= 32 with one warp per pair: lane i holds row i of both columns in
  // registers; the three inner products are warp-shuffle trees computed side
  // by side, so a round costs one shared-memory round trip, ~5 shuffle
  // latencies and the rotation (~4-5x fewer cycles than groups of 8 lanes
  // looping over rows).
  const bool warp_path = (l <= 32) && (nwarps >= lp / 2);
  for (; warp_path && sweep < 60; ++sweep) {
    if (tid == 0) changed = 0;
    // running max of g^2/(a b) as a fraction num/den (no division per round)
    double mnum = 0.0, mden = 1.0;
    __syncthreads();
    for (int round = 0; round < lp - 1; ++round) {
      const int pr = warp;
      int pcol = 0, qcol = l;
      if (pr < lp / 2) {
        int ia = pr - 1 + round;
        if (ia >= lp - 1) ia -= lp - 1;
        int ib = lp - 2 - pr + round;
        if (ib >= lp - 1) ib -= lp - 1;
        const int a = (pr == 0) ? 0 : 1 + ia;
        const int bq = 1 + ib;
        pcol = min(a, bq);
        qcol = max(a, bq);
      }
      const bool act = qcol < l;  // warp-uniform
      // probe: clock stamps of warp 0, sweep 0, rounds 0..7 (dbg[32 + 8 r + k])
      const bool stamp = dbg && sweep == 0 && round < 8 && warp == 0 && lane == 0;
      if (stamp) dbg[32 + 8 * round] = double(clock64());
      if (act) {
        const bool row = lane < l;
        double xp = row ? X[pcol * l + lane] : 0.0, xq = row ? X[qcol * l + lane] : 0.0;
        // J rows loaded with X (X and J share the shared buffer: the compiler
        // cannot move these loads above the X stores below)
        const double jp = row ? J[pcol * l + lane] : 0.0, jq = row ? J[qcol * l + lane] : 0.0;
        if (stamp) dbg[33 + 8 * round] = double(clock64()) + 0.0 * (xp + xq);
        // (a, b, g) = sums of xp^2, xq^2, xp xq over the warp.  The round is
        // bound by the warp shuffles of the 13 warps (one SHFL.32 per clock
        // per SM: measured 93 cycles per butterfly level for 3 values), so a
        // reduce-scatter halves the traffic: at offset 16 lanes with bit 4
        // clear keep (a, b) and the others keep g, at offset 8 the (a, b)
        // lanes split a / b, then three levels on one value each and three
        // broadcasts: 9 64-bit shuffles instead of 15.
        double al, be, ga;
        {
          const bool hi4 = (lane & 16) != 0, hi3 = (lane & 8) != 0;
          const double a0 = xp * xp, b0 = xq * xq, g0 = xp * xq;
          const double s1 = __shfl_xor_sync(0xffffffffu, hi4 ? a0 : g0, 16);
          const double s2 = __shfl_xor_sync(0xffffffffu, hi4 ? b0 : 0.0, 16);
          const double k1 = hi4 ? g0 + s1 : a0 + s1;  // hi4: g, else: a
          const double k2 = b0 + s2;                  // !hi4: b
          const double send = hi4 ? k1 : (hi3 ? k1 : k2);
          const double r = __shfl_xor_sync(0xffffffffu, send, 8);
          double v = hi4 ? k1 + r : (hi3 ? k2 + r : k1 + r);  // lane quantity: g | b | a
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          al = __shfl_sync(0xffffffffu, v, 0);
          be = __shfl_sync(0xffffffffu, v, 8);
          ga = __shfl_sync(0xffffffffu, v, 16);
        }
        if (stamp) dbg[34 + 8 * round] = double(clock64()) + 0.0 * (al + be + ga);
        // rotation from two reciprocal square roots (no sqrt/div on the chain):
        // ir = 1/r, r = |(d, 2g)|; cos 2th = |d|/r; c = sqrt(h), h = (1+cos 2th)/2;
        // s = sgn(d) sin 2th / (2c) = sgn(d) g ir / sqrt(h)  (c^2 + s^2 = 1)
        if (ga * ga * mden > mnum * (al * be)) {
          mnum = ga * ga;
          mden = al * be;
        }
        if (ga * ga > tol * tol * (al * be) && ga != 0.0) {
          const double d = be - al, g2 = 2.0 * ga;
          const double ir = rsqrt(fma(d, d, g2 * g2));
          const double hh = fma(0.5 * fabs(d), ir, 0.5);
          const double ih = rsqrt(hh);
          const double c = hh * ih, sn = copysign(1.0, d) * (ga * ir) * ih;
          if (stamp) dbg[35 + 8 * round] = double(clock64()) + 0.0 * (c + sn);
          if (row) {
            X[pcol * l + lane] = c * xp - sn * xq;
            X[qcol * l + lane] = sn * xp + c * xq;
            J[pcol * l + lane] = c * jp - sn * jq;
            J[qcol * l + lane] = sn * jp + c * jq;
          }
          if (lane == 0) changed = 1;
          if (stamp) dbg[36 + 8 * round] = double(clock64());
        }
      }
      __syncthreads();
      if (stamp) dbg[37 + 8 * round] = double(clock64());
    }
    if (lane == 0) wmax_s[warp] = mden > 0.0 ? mnum / mden : 0.0;
    __syncthreads();
    double m_k = 0.0;
    for (int w = 0; w < nwarps; ++w) m_k = fmax(m_k, wmax_s[w]);
    if (dbg && tid == 0 && sweep < 30) dbg[1 + sweep] = sqrt(m_k);
    if (dbg && tid == 0) dbg[0] = sweep + 1;
    if (!changed || (sweep > 0 && jacobi_quad_stop(m_k, m_prev))) break;
    m_prev = m_k;
    __syncthreads();
  }
  for (; !warp_path && sweep < 60; ++sweep) {
    if (tid == 0) changed = 0;
    double mnum = 0.0, mden = 1.0;
    __syncthreads();
    for (int round = 0; round < lp - 1; ++round) {
      // circle method: slot 0 fixed, others rotate
      const int ngroups = nthr / GS, grp = tid / GS, gl = tid % GS;
      for (int pr0 = 0; pr0 < lp / 2; pr0 += ngroups) {
        const int pr = pr0 + grp;
        int pcol = 0, qcol = l;  // inactive group -> dummy
        if (pr < lp / 2) {
          // circle method without runtime modulo: slot (pr - 1 + round) wraps once
          int ia = pr - 1 + round;
          if (ia >= lp - 1) ia -= lp - 1;
          int ib = lp - 2 - pr + round;
          if (ib >= lp - 1) ib -= lp - 1;
          const int a = (pr == 0) ? 0 : 1 + ia;
          const int bq = 1 + ib;
          pcol = min(a, bq);
          qcol = max(a, bq);
        }
        const bool act = qcol < l;
        double al = 0, be = 0, ga = 0;
        if (act)
          for (int i = gl; i < l; i += GS) {
            const double xp = X[pcol * l + i], xq = X[qcol * l + i];
            al += xp * xp;
            be += xq * xq;
            ga += xp * xq;
          }
        al = group_sum<GS>(al);  // all lanes participate (full-mask shuffles)
        be = group_sum<GS>(be);
        ga = group_sum<GS>(ga);
        if (act && ga * ga * mden > mnum * (al * be)) {
          mnum = ga * ga;
          mden = al * be;
        }
        if (act && fabs(ga) > tol * sqrt(al * be) && ga != 0.0) {
          // t = tan(theta) = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
          // rewritten with one division and one square root
          const double d = be - al, g2 = 2.0 * ga;
          const double t = copysign(1.0, d) * g2 / (fabs(d) + sqrt(d * d + g2 * g2));
          const double c = rsqrt(1.0 + t * t), s = c * t;
          for (int i = gl; i < l; i += GS) {
            const double xp = X[pcol * l + i], xq = X[qcol * l + i];
            X[pcol * l + i] = c * xp - s * xq;
            X[qcol * l + i] = s * xp + c * xq;
            const double jp = J[pcol * l + i], jq = J[qcol * l + i];
            J[pcol * l + i] = c * jp - s * jq;
            J[qcol * l + i] = s * jp + c * jq;
          }
          if (gl == 0) changed = 1;
        }
      }
      __syncthreads();
    }
    {
      double mw = mden > 0.0 ? mnum / mden : 0.0;
      for (int o = 16; o > 0; o >>= 1) mw = fmax(mw, __shfl_xor_sync(0xffffffffu, mw, o));
      if (lane == 0) wmax_s[warp] = mw;
    }
    __syncthreads();
    double m_k = 0.0;
    for (int w = 0; w < nwarps; ++w) m_k = fmax(m_k, wmax_s[w]);
    if (!changed || (sweep > 0 && jacobi_quad_stop(m_k, m_prev))) break;
    m_prev = m_k;
    __syncthreads();
  }
  if (sweep >= 60 && tid == 0) atomicOr(flags, kFlagJacobiNoConv);
  if (tid == 0 && flags) atomicMax(flags + 8, sweep + 1);  // sweep statistics (probe)
  // column norms and stable descending order
  for (int j = warp; j < l; j += nwarps) {
    double s = 0;
    for (int i = lane; i < l; i += 32) s += X[j * l + i] * X[j * l + i];
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < l; j += nthr) {
    int rank = 0;
    const double v = order_key(nrm[j]);
    for (int k = 0; k < l; ++k) {
      const double u = order_key(nrm[k]);
      if (u > v || (u == v && k < j)) ++rank;
    }
    order[rank] = j;
  }
  __syncthreads();
  const double smax = nrm[order[0]];
  for (int64_t e = tid; e < int64_t(l) * l; e += nthr) {
    const int i = int(e % l), jn = int(e / l);
    const int src = order[jn];
    Jout[jn * ldj + i] = J[src * l + i];
    const double s = nrm[src];
    Wout[jn * ldw + i] = (s > 0.0 && s > smax * 1e-300) ? X[src * l + i] / s : 0.0;
  }
  for (int j = tid; j < l; j += nthr) sigma[j] = nrm[order[j]];
  __syncthreads();
  // Complete zero columns of W to an orthonormal set (rank-deficient input).
  if (warp == 0) {
    for (int jn = 0; jn < l; ++jn) {
      const double s = nrm[order[jn]];
      if (s > 0.0 && s > smax * 1e-300) continue;
      double bestn = -1.0;
      int besti = 0;
      for (int cand = 0; cand < l; ++cand) {
        // residual norm of e_cand after projecting out valid columns
        double r2 = 1.0;
        for (int k = 0; k < l; ++k) {
          if (k == jn) continue;
          const double sk = nrm[order[k]];
          const bool valid = (k < jn) || (sk > 0.0 && sk > smax * 1e-300);
          if (!valid) continue;
          const double w = Wout[k * ldw + cand];
          r2 -= w * w;
        }
        if (r2 > bestn + 1e-12) {
          bestn = r2;
          besti = cand;
        }
      }
      for (int i = lane; i < l; i += 32) Wout[jn * ldw + i] = (i == besti) ? 1.0 : 0.0;
      __syncwarp();
      for (int pass = 0; pass < 2; ++pass) {
        for (int k = 0; k < l; ++k) {
          if (k == jn) continue;
          const double sk = nrm[order[k]];
          const bool valid = (k < jn) || (sk > 0.0 && sk > smax * 1e-300);
          if (!valid) continue;
          double d = 0;
          for (int i = lane; i < l; i += 32) d += Wout[k * ldw + i] * Wout[jn * ldw + i];
          d = warp_sum(d);
          for (int i = lane; i < l; i += 32) Wout[jn * ldw + i] -= d * Wout[k * ldw + i];
          __syncwarp();
        }
        double nn = 0;
        for (int i = lane; i < l; i += 32) nn += Wout[jn * ldw + i] * Wout[jn * ldw + i];
        nn = sqrt(warp_sum(nn));
        for (int i = lane; i < l; i += 32) Wout[jn * ldw + i] /= nn;
        __syncwarp();
      }
    }
  }
}

// ------------------------------------------------------ symmetric Jacobi EVD
// Two-sided cyclic Jacobi with round-robin ordering; single CTA.
__global__ void jacobi_evd_kernel(const double* __restrict__ Cin, int64_t ldc, int l,
                                  double* __restrict__ Uout, int64_t ldu,
                                  double* __restrict__ lam, double* gA, double* gV, int in_smem,
                                  double* rot, int* flags) {
  RSVD_PDL_ENTRY();
  extern __shared__ double sm[];
  double* A = in_smem ? sm : gA;
  double* V = in_smem ? sm + int64_t(l) * l : gV;
  __shared__ int changed;
  __shared__ int order[1024];
  __shared__ int pp[512], qq[512];
  __shared__ double cs[512], sn[512];
  const int tid = threadIdx.x, nthr = blockDim.x;
  __shared__ double wsum[32];
  double part = 0.0;
  for (int64_t e = tid; e < int64_t(l) * l; e += nthr) {
    const int i = int(e % l), j = int(e / l);
    const double v = Cin[j * ldc + i];
    A[e] = v;
    part += v * v;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  part = warp_sum(part);
  if ((tid & 31) == 0) wsum[tid >> 5] = part;
  __syncthreads();
  double fro2 = 0.0;
  for (int w = 0; w < (nthr >> 5); ++w) fro2 += wsum[w];
  // rotations below this magnitude are backward-stable no-ops (eps * ||C||_F)
  const double abs_tol = 1e-17 * sqrt(fro2);
  const int lp = l + (l & 1);
  const int npairs = lp / 2;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (tid == 0) changed = 0;
    __syncthreads();
    for (int round = 0; round < lp - 1; ++round) {
      for (int pr = tid; pr < npairs; pr += nthr) {
        int a = (pr == 0) ? 0 : 1 + (pr - 1 + round) % (lp - 1);
        int b = 1 + (lp - 2 - pr + round) % (lp - 1);
        int p = min(a, b), q = max(a, b);
        double c = 1.0, s = 0.0;
        if (q < l) {
          const double apq = A[q * l + p];
          const double app = A[p * l + p], aqq = A[q * l + q];
          if (fabs(apq) > abs_tol && fabs(apq) > 1e-300 &&
              fabs(apq) > 1e-16 * sqrt(fabs(app)) * sqrt(fabs(aqq)) * 0.5) {
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = (fabs(theta) > 1e150)
                                 ? 0.5 / theta
                                 : copysign(1.0, theta) / (fabs(theta) + sqrt(1.0 + theta * theta));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            changed = 1;
          }
        } else {
          q = -1;
        }
        pp[pr] = p;
        qq[pr] = q;
        cs[pr] = c;
        sn[pr] = s;
      }
      __syncthreads();
      // A <- A J (columns), V <- V J
      for (int64_t e = tid; e < int64_t(npairs) * l; e += nthr) {
        const int pr = int(e / l), i = int(e % l);
        const int p = pp[pr], q = qq[pr];
        if (q < 0 || sn[pr] == 0.0) continue;
        const double c = cs[pr], s = sn[pr];
        const double ap = A[p * l + i], aq = A[q * l + i];
        A[p * l + i] = c * ap - s * aq;
        A[q * l + i] = s * ap + c * aq;
        const double vp = V[p * l + i], vq = V[q * l + i];
        V[p * l + i] = c * vp - s * vq;
        V[q * l + i] = s * vp + c * vq;
      }
      __syncthreads();
      // A <- J^T A (rows)
      for (int64_t e = tid; e < int64_t(npairs) * l; e += nthr) {
        const int pr = int(e / l), j = int(e % l);
        const int p = pp[pr], q = qq[pr];
        if (q < 0 || sn[pr] == 0.0) continue;
        const double c = cs[pr], s = sn[pr];
        const double ap = A[j * l + p], aq = A[j * l + q];
        A[j * l + p] = c * ap - s * aq;
        A[j * l + q] = s * ap + c * aq;
      }
      __syncthreads();
    }
    if (!changed) break;
    __syncthreads();
  }
  if (sweep >= 60 && tid == 0) atomicOr(flags, kFlagJacobiNoConv);
  (void)rot;
  // order by |lambda| descending, ties by ascending lambda value then index
  // (reference: stable sort of an ascending eigenvalue list).
  for (int j = tid; j < l; j += nthr) {
    const double v0 = A[j * l + j], v = (v0 != v0) ? 0.0 : v0;
    const double av = order_key(fabs(v0));
    int rank = 0;
    for (int k = 0; k < l; ++k) {
      const double u0 = A[k * l + k], u = (u0 != u0) ? 0.0 : u0;
      const double au = order_key(fabs(u0));
      // |lambda| descending; exact ties: positive first, then index (the
      // reference's Eigen solver returns (-1+d, 1) for [[0,1],[1,0]], so its
      // stable |lambda| sort yields (1, -1); test_core.cpp:148-162)
      const bool before = (au > av) || (au == av && (u > v || (u == v && k < j)));
      if (before) ++rank;
    }
    order[rank] = j;
  }
  __syncthreads();
  for (int64_t e = tid; e < int64_t(l) * l; e += nthr) {
    const int i = int(e % l), jn = int(e / l);
    Uout[jn * ldu + i] = V[order[jn] * l + i];
  }
  for (int j = tid; j < l; j += nthr) lam[j] = A[order[j] * l + order[j]];
}

// -------------------------------------------------------------- sign rule
__global__ void sign_rule_kernel(double* U, int64_t rows, int64_t ldu, double* V, int64_t vrows,
                                 int64_t ldv) {
  RSVD_PDL_ENTRY();
  const int j = blockIdx.x;
  __shared__ double bv[32];
  __shared__ long long bi[32];
  double best = -1.0;
  long long bidx = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double a = fabs(U[j * ldu + i]);
    if (a > best) {
      best = a;
      bidx = i;
    }
  }
  // warp argmax, lowest index on ties
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) {
      best = ob;
      bidx = oi;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    bv[warp] = best;
    bi[warp] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w)
      if (bv[w] > best || (bv[w] == best && bi[w] < bidx)) {
        best = bv[w];
        bidx = bi[w];
      }
    bi[0] = bidx;
  }
  __syncthreads();
  const bool flip = U[j * ldu + bi[0]] < 0.0;
  __syncthreads();
  if (!flip) return;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) U[j * ldu + i] = -U[j * ldu + i];
  if (V)
    for (int64_t i = threadIdx.x; i < vrows; i += blockDim.x) V[j * ldv + i] = -V[j * ldv + i];
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols,
                                 int64_t ldi, double* __restrict__ out, int64_t ldo) {
  RSVD_PDL_ENTRY();
  __shared__ double t[32][33];
  const int64_t i0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + k;
    if (i < rows && j < cols) t[k][threadIdx.x] = in[j * ldi + i];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + k;  // out(j, i) = in(i, j)
    if (i < rows && j < cols) out[i * ldo + j] = t[threadIdx.x][k];
  }
}

__global__ void scale_cols_kernel(double* X, int64_t rows, int64_t cols, int64_t ld,
                                  const double* s, int inv) {
  RSVD_PDL_ENTRY();
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    X[j * ld + i] = inv ? X[j * ld + i] / s[j] : X[j * ld + i] * s[j];
  }
}

__global__ void sym_part_kernel(const double* A, int64_t n, int64_t lda, double* C, int64_t ldc) {
  RSVD_PDL_ENTRY();
  const int64_t tot = n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    C[j * ldc + i] = 0.5 * (A[j * lda + i] + A[i * lda + j]);
  }
}

__global__ void finite_kernel(const double* X, int64_t rows, int64_t cols, int64_t ld, int* flags,
                              int bit) {
  RSVD_PDL_ENTRY();
  const int64_t n = rows * cols;
  bool bad = false;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    if (!isfinite(X[j * ld + i])) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, bit);
}

// ---------------------------------------------------------- Cholesky (l x l)
// Right-looking, single CTA, in place on a copy of G (ld l) in shared or global
// memory.  Produces upper R (G + s I = R^T R) and Rinv = R^-1.
// Shift policy (shifted CholeskyQR, Fukaya et al.): the factorization is first
// tried with s = 0; when a pivot has lost all precision (Schur pivot
// <= 1e-12 of its original diagonal, or not positive) it restarts with
// s = shift_coef * trace(G), shift_coef = 11 (m l + l (l+1)) u, and records it
// in *shift_used.  The decision is made on the device: no host round trip.
__global__ void chol_inv_kernel(const double* __restrict__ G, int64_t ldg, int l,
                                double shift_coef, double* __restrict__ R, int64_t ldr,
                                double* __restrict__ Rinv, int64_t ldri, double* gA, int in_smem,
                                int* shift_used, int* flags) {
  RSVD_PDL_ENTRY();
  extern __shared__ double sm[];
  double* A = in_smem ? sm : gA;  // lower-triangular working copy (col-major, ld l)
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = nthr >> 5;
  __shared__ int broke;
  __shared__ double trace;
  __shared__ double diag0[1024];  // original diagonal (pivot-loss test), kept on chip
  for (int j = tid; j < l; j += nthr) diag0[j] = G[j * ldg + j];
  __syncthreads();
  for (int attempt = 0; attempt < 2; ++attempt) {
    double shift = 0.0;
    if (attempt == 1) {
      if (tid == 0) {
        double t = 0;
        for (int j = 0; j < l; ++j) t += diag0[j];
        trace = t;
      }
      __syncthreads();
      shift = shift_coef * trace;
    }
    if (tid == 0) broke = 0;
    for (int64_t e = tid; e < int64_t(l) * l; e += nthr) {
      const int i = int(e % l), j = int(e / l);
      double v = G[j * ldg + i];
      if (i == j) v += shift;
      A[e] = v;
    }
    __syncthreads();
    for (int j = 0; j < l; ++j) {
      const double d = A[j * l + j];
      const double orig = diag0[j] + shift;
      if (!(d > 1e-12 * orig) || !(d > 0.0)) {
        if (tid == 0) broke = 1;
        __syncthreads();
        break;
      }
      const double rd = sqrt(d);
      __syncthreads();
      for (int i = j + 1 + tid; i < l; i += nthr) A[j * l + i] /= rd;
      if (tid == 0) A[j * l + j] = rd;
      __syncthreads();
      // trailing update: A(i,k) -= L(i,j) L(k,j), k in (j, l), i >= k
      for (int k = j + 1 + warp; k < l; k += nwarps) {
        const double lkj = A[j * l + k];
        for (int i = k + lane; i < l; i += 32) A[k * l + i] -= A[j * l + i] * lkj;
      }
      __syncthreads();
    }
    if (!broke) {
      if (attempt == 1 && tid == 0 && shift_used) *shift_used = 1;
      break;
    }
    if (attempt == 1) {
      if (tid == 0) atomicOr(flags, kFlagCholBreakdown);
      return;
    }
    __syncthreads();
  }
  // R = L^T
  for (int64_t e = tid; e < int64_t(l) * l; e += nthr) {
    const int i = int(e % l), j = int(e / l);
    R[j * ldr + i] = (i <= j) ? A[i * l + j] : 0.0;
  }
  // Rinv: solve R x = e_c for each column c by back substitution; R(i,k) = L(k,i)
  for (int c = warp; c < l; c += nwarps) {
    for (int i = lane; i < l; i += 32) Rinv[c * ldri + i] = 0.0;
    __syncwarp();
    for (int i = c; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1 + lane; k <= c; k += 32) s += A[i * l + k] * Rinv[c * ldri + k];
      s = warp_sum(s);
      if (lane == 0) Rinv[c * ldri + i] = ((i == c ? 1.0 : 0.0) - s) / A[i * l + i];
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kCholThreads) chol_inv_small_kernel(
    const double* __restrict__ G, int64_t ldg, int l, double shift_coef, double* __restrict__ R, int64_t ldr,
    double* __restrict__ Rinv, int64_t ldri, int* shift_used, int* flags) {
  RSVD_PDL_ENTRY();
  constexpr int LD = 33;
  __shared__ double G0[32 * LD], piv[kCholPivScratch], Rs[32 * LD], Ri[32 * LD];
  for (int e = threadIdx.x; e < l * l; e += kCholThreads)
    G0[(e % l) + LD * (e / l)] = G[int64_t(e / l) * ldg + (e % l)];
  __syncthreads();
  bool shifted;
  if (!cta_chol_inv(G0, l, shift_coef, piv, Rs, Ri, &shifted)) {
    if (threadIdx.x == 0) atomicOr(flags, kFlagCholBreakdown);
    return;
  }
  if (shifted && threadIdx.x == 0 && shift_used) *shift_used = 1;
  for (int e = threadIdx.x; e < l * l; e += kCholThreads) {
    const int i = e % l, c = e / l;
    R[int64_t(c) * ldr + i] = Rs[i + LD * c];
    Rinv[int64_t(c) * ldri + i] = Ri[i + LD * c];
  }
}

// Whole CholeskyQR orthonormalization of a tall m x l (l <= 32) matrix in ONE
// cooperative launch.  Each CTA keeps its row block in shared memory for all
// passes; per pass: register-blocked partial Gram -> grid barrier -> every CTA
// sums the partials in CTA order (identical in every CTA) and factors the
// Gram with one warp (warp_chol_inv) -> rows <- rows * R^-1 in place.  The
// partial buffers alternate between passes so one barrier per pass suffices.
constexpr int kFqThreads = 256;
static_assert(kFqThreads == kCholThreads, "cta_chol_inv runs on the whole CTA");

__global__ void __launch_bounds__(kFqThreads, 1) cholqr_fused_kernel(
    const double* __restrict__ Y, int64_t ldy, int64_t m, int l, int64_t rows_per,
    double* __restrict__ Qo, int64_t ldq, double* __restrict__ part, double* __restrict__ Rout,
    int64_t ldr, double shift_coef, int passes, int* __restrict__ flags, long long* probe) {
  RSVD_PDL_ENTRY();
  constexpr int LD = 33;
  cg::grid_group grid = cg::this_grid();
  int np_ = 0;
  auto mark = [&]() {
    if (probe && blockIdx.x == 0 && threadIdx.x == 0 && np_ < 64) probe[np_++] = clock64();
    if (np_ >= 44) np_ = 43;
  };
  mark();
  // dynamic shared memory: red[8][32*33] | Gs | Rs | Ri | Rt (32*33 each) | Ys
  extern __shared__ double fsm[];
  double (*red)[32 * LD] = reinterpret_cast<double (*)[32 * LD]>(fsm);
  double* Gs = fsm + 8 * 32 * LD;
  double* Rs = Gs + 32 * LD;
  double* Ri = Rs + 32 * LD;
  double* Rt = Ri + 32 * LD;
  double* Ys = Rt + 32 * LD;  // rows_per x 33 (row-major, padded)
  __shared__ int okf, prev_shift;
  __shared__ double devw[kFqThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int RP = int(rows_per);
  if (tid == 0) prev_shift = 0;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per;
  const int nr = int(m - r0 < rows_per ? m - r0 : rows_per);
  const int G = gridDim.x;
  bool bad = false;
#pragma unroll 4
  for (int e = tid; e < RP * 32; e += kFqThreads) {
    const int r = e % RP, a = e / RP;
    double v = 0.0;
    if (r < nr && a < l) {
      v = Y[int64_t(a) * ldy + r0 + r];
      if (!isfinite(v)) bad = true;
    }
    Ys[r * LD + a] = v;
  }
  if (bad) atomicOr(flags, kFlagNonFinite);
  for (int e = tid; e < 32 * LD; e += kFqThreads) Rt[e] = ((e % LD) == (e / LD)) ? 1.0 : 0.0;
  __syncthreads();
  mark();
  for (int pass = 0; pass < passes; ++pass) {
    // ---- partial Gram Ys^T Ys on DMMA: warp w reduces rows [w*RP/8, (w+1)*RP/8)
    // into a full 32 x 32 tile (16 m8n8 accumulators); warp tiles summed in order.
    {
      const int lane = tid & 31, r8 = lane >> 2, c4 = lane & 3;
      const int wrows = RP / 8, rw0 = warp * wrows;
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int k0 = rw0; k0 < rw0 + wrows; k0 += 4) {
        const double* yr = Ys + (k0 + c4) * LD;  // row k0 + c4
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          af[i] = yr[i * 8 + r8];  // A(m = a, k = r): Ys[r][a]
          bf[i] = af[i];           // B(k = r, n = b): Ys[r][b], same fragment shape
        }
        // the Gram is symmetric: upper tiles only (10 of 16), mirrored below
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = i; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i; j < 4; ++j) {
          const int a0 = i * 8 + r8, b0 = j * 8 + 2 * c4;
          red[warp][a0 + LD * b0] = acc[i][j][0];
          red[warp][a0 + LD * (b0 + 1)] = acc[i][j][1];
          if (j > i) {
            red[warp][b0 + LD * a0] = acc[i][j][0];
            red[warp][(b0 + 1) + LD * a0] = acc[i][j][1];
          }
        }
    }
    __syncthreads();
    double* pp = part + (int64_t(pass & 1) * G + blockIdx.x) * 1024;
    {
      // the thread's four entries interleaved (four independent add chains)
      constexpr int EPT = 1024 / kFqThreads;
      double v[EPT];
#pragma unroll
      for (int x = 0; x < EPT; ++x) v[x] = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w)
#pragma unroll
        for (int x = 0; x < EPT; ++x) {
          const int e = tid + kFqThreads * x;
          v[x] += red[w][(e & 31) + LD * (e >> 5)];
        }
#pragma unroll
      for (int x = 0; x < EPT; ++x) pp[tid + kFqThreads * x] = v[x];
    }
    __threadfence();
    mark();
    grid.sync();
    mark();
    // ---- total Gram, identical in every CTA (fixed CTA order)
    const double* pb0 = part + int64_t(pass & 1) * G * 1024;
    {
      // the thread's four entries together: 32 loads in flight per round
      // trip instead of 8 (same CTA order per entry: bitwise unchanged)
      constexpr int EPT = 1024 / kFqThreads;
      double v[EPT];
#pragma unroll
      for (int x = 0; x < EPT; ++x) v[x] = 0.0;
      int c = 0;
      for (; c + 8 <= G; c += 8) {
        double t[EPT][8];
#pragma unroll
        for (int x = 0; x < EPT; ++x)
#pragma unroll
          for (int q = 0; q < 8; ++q) t[x][q] = __ldcg(pb0 + int64_t(c + q) * 1024 + tid + kFqThreads * x);
#pragma unroll
        for (int x = 0; x < EPT; ++x)
#pragma unroll
          for (int q = 0; q < 8; ++q) v[x] += t[x][q];
      }
      for (; c < G; ++c)
#pragma unroll
        for (int x = 0; x < EPT; ++x) v[x] += __ldcg(pb0 + int64_t(c) * 1024 + tid + kFqThreads * x);
#pragma unroll
      for (int x = 0; x < EPT; ++x) {
        const int e = tid + kFqThreads * x;
        Gs[(e & 31) + LD * (e >> 5)] = v[x];
      }
    }
    __syncthreads();
    mark();
    // Converged: the Gram of the current rows is the identity to rounding
    // (|G - I| <= 4 l u): the remaining passes would multiply by R^-1 = I.
    // Nearly converged (|G - I| <= 1e-8): R from its series, no elimination:
    // with E = G - I and Phi(M) = upper triangle of M with halved diagonal,
    // R = I + Phi(E) - Phi(Phi(E)^T Phi(E)) + O(E^3) and
    // R^-1 = I - Phi(E) + Phi(E)^2 + O(E^2), i.e. orthogonality to O(E^2) <= 1e-16.
    bool series = false;
    if (pass > 0) {
      double dev = 0.0;
      for (int e = tid; e < l * l; e += kFqThreads) {
        const int i = e % l, j = e / l;
        dev = fmax(dev, fabs(Gs[i + LD * j] - (i == j ? 1.0 : 0.0)));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
      if ((tid & 31) == 0) devw[warp] = dev;
      __syncthreads();
      dev = 0.0;
#pragma unroll
      for (int w = 0; w < kFqThreads / 32; ++w) dev = fmax(dev, devw[w]);  // identical in every CTA
      __syncthreads();
      if (dev <= 4.0 * l * 1.1102230246251565e-16) break;
      series = dev <= 1e-8;
    }
    {
      long long* pr = (probe && blockIdx.x == 0 && pass < 5) ? probe + 44 + 4 * pass : nullptr;
      bool ok = true;
      if (series) {
        auto phi = [&](int a, int b) -> double {
          return (a < b) ? Gs[a + LD * b] : (a == b ? 0.5 * (Gs[a + LD * a] - 1.0) : 0.0);
        };
        for (int e = tid; e < 32 * 32; e += kFqThreads) {
          const int i = e & 31, j = e >> 5;
          double v = 0.0;
          if (i < l && j < l && i <= j) {
            double s2 = 0.0;
            for (int k = i; k <= j; ++k) s2 = fma(phi(i, k), phi(k, j), s2);
            v = (i == j ? 1.0 : 0.0) - phi(i, j) + s2;
          }
          Ri[i + LD * j] = v;
        }
        if (Rout && blockIdx.x == 0) {
          double* Mt = &red[0][0];  // Phi^T Phi (the Gram partials are consumed)
          for (int e = tid; e < 32 * 32; e += kFqThreads) {
            const int i = e & 31, j = e >> 5;
            double v = 0.0;
            for (int k = 0; k <= min(i, j); ++k) v = fma(phi(k, i), phi(k, j), v);
            Mt[i + LD * j] = v;
          }
          __syncthreads();
          for (int e = tid; e < 32 * 32; e += kFqThreads) {
            const int i = e & 31, j = e >> 5;
            double v = 0.0;
            if (i < l && j < l && i <= j) {
              const double pm = (i < j) ? Mt[i + LD * j] : 0.5 * Mt[i + LD * i];
              v = (i == j ? 1.0 : 0.0) + phi(i, j) - pm;
            }
            Rs[i + LD * j] = v;
          }
        }
        __syncthreads();
        if (tid == 0) okf = 1;
      } else {
        bool shifted;
        // the Gram partials in red[] are consumed: red[] is the pivot scratch.
        // When the first pass needed the shift, the second goes straight to
        // the shifted factorization (measured on the C2 sketch: its unshifted
        // attempt breaks down too); later passes stay unshifted first, as an
        // orthonormal Q requires.
        ok = cta_chol_inv(Gs, l, shift_coef, &red[0][0], Rs, Ri, &shifted, pr, nullptr, 2,
                          (pass == 1 && prev_shift) ? 1 : 0);
        if (tid == 0) okf = ok ? 1 : 0;
        if (!ok && blockIdx.x == 0 && tid == 0) atomicOr(flags, kFlagCholBreakdown);
        __syncthreads();
        if (tid == 0) prev_shift = shifted ? 1 : 0;
      }
      // R_total <- R * R_total (both upper triangular), warp 0 of CTA 0
      if (ok && Rout && blockIdx.x == 0 && warp == 0) {
        // lane c: column c of R_total in registers; rows of R are broadcast loads
        const int c = threadIdx.x & 31;
        double t[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) t[k] = Rt[k + LD * c];
#pragma unroll 1
        for (int i = 0; i < l; ++i) {
          double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k & 3] = fma(Rs[i + LD * k], t[k], v[k & 3]);
          Rt[i + LD * c] = (v[0] + v[1]) + (v[2] + v[3]);
        }
        __syncwarp();
      }
      if (pr && tid == 0) pr[3] = clock64();
    }
    __syncthreads();
    mark();
    if (!okf) return;  // identical decision in every CTA
    // ---- rows <- rows * R^-1 on DMMA, in place: warp w owns rows
    // [w*RP/8, (w+1)*RP/8) in chunks of 32 (4 m8 tiles x 4 n8 tiles, K = 32)
    {
      const int lane = tid & 31, r8 = lane >> 2, c4 = lane & 3;
      const int wrows = RP / 8, rw0 = warp * wrows;
      for (int m0 = rw0; m0 < rw0 + wrows; m0 += 32) {
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        // R^-1 is upper triangular: column tile j only meets rows k < 8 (j + 1)
        // (80 of 128 DMMAs per 32-row chunk)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const int kk = ks * 4 + c4;
          double af[4], bf[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = Ys[(m0 + i * 8 + r8) * LD + kk];  // A(r, k)
#pragma unroll
          for (int j = ks / 2; j < 4; ++j) bf[j] = Ri[kk + LD * (j * 8 + r8)];  // B(k, c)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = ks / 2; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = m0 + i * 8 + r8, c = j * 8 + 2 * c4;
            Ys[r * LD + c] = (c < l) ? acc[i][j][0] : 0.0;
            Ys[r * LD + c + 1] = (c + 1 < l) ? acc[i][j][1] : 0.0;
          }
        __syncwarp();
      }
    }
    __syncthreads();
    mark();
  }
  for (int e = tid; e < RP * l; e += kFqThreads) {
    const int r = e % RP, a = e / RP;
    if (r < nr) Qo[int64_t(a) * ldq + r0 + r] = Ys[r * LD + a];
  }
  if (Rout && blockIdx.x == 0)
    for (int e = tid; e < l * l; e += kFqThreads) {
      const int i = e % l, c = e / l;
      Rout[int64_t(c) * ldr + i] = Rt[i + LD * c];
    }
}

}  // namespace

// =================================================================== host
// Opt a kernel into `bytes` of dynamic shared memory (idempotent, grows only).
template <class K>
static void ensure_smem(K kernel, size_t bytes) {
  smem_attr(kernel, bytes);
}

void check_flags(Handle& h, const char* what) {
  RSVD_CUDA(cudaMemcpyAsync(h.h_flags, h.d_flags, sizeof(int), cudaMemcpyDeviceToHost, h.stream));
  stream_sync(h);
  const int f = *h.h_flags;
  if (f & kFlagRetryRobust) {  // a speculated branch was wrong: re-run robustly
    clear_flags(h);
    throw RetryRobust{};
  }
  if (f) {
    clear_flags(h);
    std::string m = std::string(what) + ": ";
    if (f & kFlagNonFinite) throw_numeric(m + "input has non-finite entries");
    if (f & kFlagAsymmetric) throw_numeric(m + "input is not symmetric");
    if (f & kFlagJacobiNoConv) throw_numeric(m + "Jacobi iteration did not converge");
    if (f & kFlagCholBreakdown) throw_numeric(m + "Cholesky breakdown");
    if (f & kFlagPowerCap) throw_numeric(m + "power iteration hit the 5000-step cap");
    if (f & kFlagRngExhausted) throw Error(RSVD_ERR_INTERNAL, m + "rng attempt budget exhausted");
    if (f & kFlagRngPatchOverflow) throw Error(RSVD_ERR_INTERNAL, m + "rng exact-log patch list overflow");
    if (f & kFlagLaunchShape) throw Error(RSVD_ERR_CUDA, m + "a cluster kernel was launched without its cluster shape");
    throw Error(RSVD_ERR_INTERNAL, m + "device flag set");
  }
}

void clear_flags(Handle& h) {
  RSVD_CUDA(cudaMemsetAsync(h.d_flags, 0, sizeof(int), h.stream));
}

void check_finite(Handle& h, const DMat& X, int bit) {
  if (X.rows * X.cols == 0) return;
  const int64_t n = X.rows * X.cols;
  const int blocks = int(std::min<int64_t>(ceil_div(n, 256), 4 * h.sm_count));
  launch_k(h, finite_kernel, blocks, 256, 0, X.p, X.rows, X.cols, X.ld, h.d_flags, bit);
  RSVD_LAUNCHED(h);
}

void transpose(Handle& h, const DMat& in, DMat out) {
  if (in.rows * in.cols == 0) return;
  dim3 grid(unsigned(ceil_div(in.rows, 32)), unsigned(ceil_div(in.cols, 32)));
  launch_k(h, transpose_kernel, grid, dim3(32, 8), 0, in.p, in.rows, in.cols, in.ld, out.p,
                                                       out.ld);
  RSVD_LAUNCHED(h);
}

void copy(Handle& h, const DMat& X, DMat Y) {
  if (X.rows * X.cols == 0 || X.p == Y.p) return;
  RSVD_CUDA(cudaMemcpy2DAsync(Y.p, Y.ld * 8, X.p, X.ld * 8, X.rows * 8, X.cols,
                              cudaMemcpyDeviceToDevice, h.stream));
}

void scale_cols(Handle& h, DMat X, const double* s, bool inv) {
  const int64_t n = X.rows * X.cols;
  if (!n) return;
  const int blocks = int(std::min<int64_t>(ceil_div(n, 256), 4 * h.sm_count));
  launch_k(h, scale_cols_kernel, blocks, 256, 0, X.p, X.rows, X.cols, X.ld, s, inv ? 1 : 0);
  RSVD_LAUNCHED(h);
}

void sym_part(Handle& h, const DMat& A, DMat C) {
  const int64_t n = A.rows;
  if (!n) return;
  const int blocks = int(std::min<int64_t>(ceil_div(n * n, 256), 4 * h.sm_count));
  launch_k(h, sym_part_kernel, blocks, 256, 0, A.p, n, A.ld, C.p, C.ld);
  RSVD_LAUNCHED(h);
}

void sign_rule(Handle& h, DMat U, DMat* V) {
  if (U.cols == 0) return;
  launch_k(h, sign_rule_kernel, unsigned(U.cols), 256, 0, 
      U.p, U.rows, U.ld, V ? V->p : nullptr, V ? V->rows : 0, V ? V->ld : 0);
  RSVD_LAUNCHED(h);
}

namespace {
struct TsqrLevel {
  int64_t rows;
  int nblk;
  double* V;
  double* tau;
};

// Factor levels until one block remains; returns the l x l R (view into ws).
DMat tsqr_factor(Handle& h, const DMat& X, std::vector<TsqrLevel>& lv) {
  const int l = int(X.cols);
  const int b = tsqr_block_rows(l);
  const size_t smem_f = (size_t(b) * l + 4) * 8;
  ensure_smem(hh_factor_kernel, smem_f);
  DMat cur = X;
  while (true) {
    TsqrLevel L;
    L.rows = cur.rows;
    L.nblk = int(ceil_div(cur.rows, b));
    L.V = h.ws.alloc(int64_t(L.nblk) * b * l);
    L.tau = h.ws.alloc(int64_t(L.nblk) * l);
    DMat Rs = h.ws.mat(int64_t(L.nblk) * l, l);
    launch_k(h, hh_factor_kernel, L.nblk, 256, smem_f, cur.p, cur.rows, l, cur.ld, b, L.V, L.tau,
                                                        Rs.p, Rs.ld, h.d_flags);
    RSVD_LAUNCHED(h);
    lv.push_back(L);
    if (L.nblk == 1) return DMat(Rs.p, l, l, Rs.ld);
    cur = Rs;
  }
}

// Form Q top-down; the top level applies its reflectors to C_top (l x l, the
// identity when null).
void tsqr_form(Handle& h, const std::vector<TsqrLevel>& lv, int l, const double* c_top,
               int64_t ld_top, DMat Q) {
  const int b = tsqr_block_rows(l);
  const size_t smem_a = size_t(2) * b * l * 8;
  ensure_smem(hh_apply_kernel, smem_a);
  const double* parent = c_top;
  int64_t ldp = ld_top;
  for (int t = int(lv.size()) - 1; t >= 0; --t) {
    const TsqrLevel& L = lv[t];
    DMat out = (t == 0) ? Q : h.ws.mat(L.rows, l);
    launch_k(h, hh_apply_kernel, L.nblk, 256, smem_a, L.V, L.tau, L.rows, l, b, parent, ldp,
                                                       out.p, out.ld);
    RSVD_LAUNCHED(h);
    parent = out.p;
    ldp = out.ld;
  }
}
}  // namespace

void tsqr(Handle& h, const DMat& X, DMat Q, DMat* R, bool dist) {
  const int l = int(X.cols);
  std::vector<TsqrLevel> lv;
  DMat Rloc = tsqr_factor(h, X, lv);
  if (!dist || !h.dist()) {
    if (R) copy(h, Rloc, *R);
    tsqr_form(h, lv, l, nullptr, 0, Q);
    return;
  }
  // Row-sharded: gather every rank's l x l R, factor the stack redundantly,
  // and seed this rank's tree with its l rows of the stacked Q.
  const int P = h.nranks;
  double* packed = h.ws.alloc(int64_t(l) * l);
  DMat Rp(packed, l, l, l);
  copy(h, Rloc, Rp);
  double* gath = h.ws.alloc(int64_t(P) * l * l);
  allgather(h, packed, gath, int64_t(l) * l);
  // gath holds P column-major l x l blocks; restack as (P l) x l
  DMat S = h.ws.mat(int64_t(P) * l, l);
  for (int r = 0; r < P; ++r)
    RSVD_CUDA(cudaMemcpy2DAsync(S.p + int64_t(r) * l, S.ld * 8, gath + int64_t(r) * l * l, l * 8,
                                l * 8, l, cudaMemcpyDeviceToDevice, h.stream));
  std::vector<TsqrLevel> lv2;
  DMat Rtop = tsqr_factor(h, S, lv2);
  if (R) copy(h, Rtop, *R);
  DMat Qs = h.ws.mat(int64_t(P) * l, l);
  tsqr_form(h, lv2, l, nullptr, 0, Qs);
  tsqr_form(h, lv, l, Qs.p + int64_t(h.rank) * l, Qs.ld, Q);
}

namespace {
size_t small_smem_limit() { return 200 * 1024; }
}  // namespace


// CholeskyQR with device-side shifting (see chol_inv_kernel): 2 passes when
// the first Gram factors without a shift (CholeskyQR2), 4 when it needed one
// (shifted CholeskyQR3 + 1: covers kappa(X) up to ~1/u and exact rank
// deficiency, whose null directions come out as orthonormal round-off noise,
// i.e. the basis is padded to full width as core.hpp:93-95 requires).  For
// l <= 64 the 4 passes are always run (no host round trip); for larger l one
// flag read after pass 1 picks 2 or 4.
// One cooperative launch for l <= 32 on one GPU (see cholqr_fused_kernel).
static bool cholqr_fused(Handle& h, const DMat& X, DMat Q, DMat* Rout) {
  const int l = int(X.cols);
  const int64_t m = X.rows;
  if (l > 32) return false;
  // rows per CTA: a multiple of 256 (8 warps x 32-row DMMA chunks), <= 512
  int64_t G = std::max<int64_t>(1, std::min<int64_t>(h.sm_count, ceil_div(m, 256)));
  const int64_t rp = round_up(ceil_div(m, G), 256);
  const size_t smem = (size_t(rp) * 33 + 12 * 32 * 33) * 8;
  if (rp > 512 || smem > 220 * 1024) return false;
  G = ceil_div(m, rp);
  smem_attr(cholqr_fused_kernel, smem);
  double* part = h.ws.alloc(2 * G * 1024);
  const double coef = 11.0 * (double(m) * l + double(l) * (l + 1)) * 1.1102230246251565e-16;
  // the kernel stops as soon as Q^T Q = I to 4 l u; numerically rank-deficient
  // inputs need up to ~6 shifted passes to lift their null directions
  int passes = 8;
  const double* yp = X.p;
  int64_t ldy = X.ld;
  double* qp = Q.p;
  int64_t ldq = Q.ld;
  int64_t mm = m, rpp = rp;
  int lv = l;
  double* rp_out = Rout ? Rout->p : nullptr;
  int64_t ldr = Rout ? Rout->ld : 0;
  double cf = coef;
  int* fl = h.d_flags;
  static const bool probe_on = std::getenv("RSVD_PROBE_FQ") != nullptr;
  long long* probe = nullptr;
  if (probe_on) {
    probe = reinterpret_cast<long long*>(h.ws.alloc_bytes(64 * 8));
    RSVD_CUDA(cudaMemsetAsync(probe, 0, 64 * 8, h.stream));
  }
  void* args[] = {&yp, &ldy, &mm, &lv, &rpp, &qp, &ldq, &part, &rp_out, &ldr, &cf, &passes, &fl, &probe};
  RSVD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cholqr_fused_kernel), dim3(unsigned(G)),
                                        dim3(kFqThreads), args, smem, h.stream));
  RSVD_LAUNCHED(h);
  if (probe) {
    long long hp[64];
    RSVD_CUDA(cudaMemcpyAsync(hp, probe, sizeof hp, cudaMemcpyDeviceToHost, h.stream));
    stream_sync(h);
    std::fprintf(stderr, "cholqr_fused m=%lld l=%d G=%lld:", (long long)m, l, (long long)G);
    for (int i = 1; i < 44 && hp[i]; ++i) std::fprintf(stderr, " %lld", hp[i] - hp[i - 1]);
    std::fprintf(stderr, "\n  chol/inv/rtotal:");
    for (int i = 44; i < 64 && hp[i]; i += 4)
      std::fprintf(stderr, " [%lld %lld %lld]", hp[i + 1] - hp[i], hp[i + 2] - hp[i + 1], hp[i + 3] - hp[i + 2]);
    std::fprintf(stderr, "\n");
  }
  return true;
}

// Speculative CholeskyQR check (see cholqr): retry if a shift was used and
// (l <= 64) the final Gram deviates from I by more than tol.
__global__ void retry_flag_kernel(const int* shift_used, const double* dev, double tol, int* flags) {
  RSVD_PDL_ENTRY();
  if (threadIdx.x == 0 && *shift_used && (dev == nullptr || !(*dev <= tol)))
    atomicOr(flags, kFlagRetryRobust);
}

static void cholqr(Handle& h, const DMat& X, DMat Q, DMat* Rout, bool dist) {
  const int l = int(X.cols);
  if (!dist && cholqr_fused(h, X, Q, Rout)) return;
  DMat G = h.ws.mat(l, l), R1 = h.ws.mat(l, l), Ri = h.ws.mat(l, l);
  const bool in_smem = size_t(l) * l * 8 <= small_smem_limit();
  double* gA = in_smem ? nullptr : h.ws.alloc(int64_t(l) * l);
  int* shift_used = reinterpret_cast<int*>(h.ws.alloc_bytes(16));
  RSVD_CUDA(cudaMemsetAsync(shift_used, 0, 16, h.stream));
  ensure_smem(chol_inv_kernel, in_smem ? size_t(l) * l * 8 : 0);
  int64_t m_global = X.rows, row_off = 0;
  if (dist) shard_rows(h, X.rows, &m_global, &row_off);
  const double coef = 11.0 * (double(m_global) * l + double(l) * (l + 1)) * 1.1102230246251565e-16;
  // l > 32: blocked multi-CTA Cholesky (cholblk.cu); RSVD_CHOL_BLOCKED=0 keeps
  // the one-CTA kernel (comparison)
  static const bool use_blocked = [] {
    const char* e = std::getenv("RSVD_CHOL_BLOCKED");
    return !(e && e[0] == '0');
  }();
  auto pass = [&](const DMat& Y, DMat Qo, bool have_gram = false) {
    if (!have_gram) {
      gemm_tn(h, Y, Y, G);
      if (dist) allreduce_mat(h, G);
    }
    if (l <= 32)
      launch_k(h, chol_inv_small_kernel, 1, kCholThreads, 0, G.p, G.ld, l, coef, R1.p, R1.ld, Ri.p, Ri.ld,
                                                   shift_used, h.d_flags);
    else if (use_blocked)
      chol_inv_blocked(h, G, l, coef, R1, Ri, shift_used);
    else
      launch_k(h, chol_inv_kernel, 1, 1024, in_smem ? size_t(l) * l * 8 : 0, 
          G.p, G.ld, l, coef, R1.p, R1.ld, Ri.p, Ri.ld, gA, in_smem ? 1 : 0, shift_used,
          h.d_flags);
    if (l <= 32 || !use_blocked) RSVD_LAUNCHED(h);
    if (Y.p == Qo.p) {
      DMat Qt = h.ws.mat(Qo.rows, l);
      gemm_nn(h, Y, Ri, Qt);
      copy(h, Qt, Qo);
    } else {
      gemm_nn(h, Y, Ri, Qo);
    }
  };
  check_finite(h, X, kFlagNonFinite);
  DMat X0 = X;
  if (Rout && X.p == Q.p) {  // keep X for R = Q^T X
    X0 = h.ws.mat(X.rows, l);
    copy(h, X, X0);
  }
  pass(X0, Q);
  int passes = 4;
  if (l > 64) {
    if (h.robust) {
      int used = 0;
      RSVD_CUDA(cudaMemcpyAsync(&used, shift_used, sizeof(int), cudaMemcpyDeviceToHost, h.stream));
      stream_sync(h);
      passes = used ? 4 : 2;
    } else {
      passes = 2;  // speculated: no shift (checked below, on the device)
    }
  }
  for (int i = 1; i < passes; ++i) pass(Q, Q);
  if (!h.robust) {
    // Speculative form (no host round trip): the robust form takes more
    // passes exactly when a Cholesky needed the shift (l > 64), or when, after
    // a shifted pass, Q^T Q is not the identity to working accuracy (l <= 64).
    // Either case sets the retry flag, and the call re-runs in robust mode;
    // otherwise both forms executed the same operations (bitwise the same Q).
    double* dev = nullptr;
    if (l <= 64) {
      gemm_tn(h, Q, Q, G);
      if (dist) allreduce_mat(h, G);
      dev = h.ws.alloc(1);
      RSVD_CUDA(cudaMemsetAsync(dev, 0, sizeof(double), h.stream));
      gram_deviation_dev(h, G, dev);
    }
    launch_k(h, retry_flag_kernel, 1, 32, 0, static_cast<const int*>(shift_used),
             static_cast<const double*>(dev), 8.0 * l * 1.1102230246251565e-16, h.d_flags);
    RSVD_LAUNCHED(h);
    if (Rout) {
      gemm_tn(h, Q, X0, *Rout);
      if (dist) allreduce_mat(h, *Rout);
    }
    return;
  }
  // Numerically rank-deficient input (the shift was needed): each shifted
  // pass lifts the null-space directions by ~1/sqrt(shift) until they are
  // unit vectors, which can take more than the fixed passes.  Continue until
  // Q^T Q = I to working accuracy (the padded basis of core.hpp:93-95); the
  // check's Gram is the next pass's Gram.
  int used = 0;
  RSVD_CUDA(cudaMemcpyAsync(&used, shift_used, sizeof(int), cudaMemcpyDeviceToHost, h.stream));
  stream_sync(h);
  if (used) {
    const double tol = 8.0 * l * 1.1102230246251565e-16;
    for (int extra = 0; extra < 8; ++extra) {
      gemm_tn(h, Q, Q, G);
      if (dist) allreduce_mat(h, G);
      if (gram_deviation(h, G) <= tol) break;
      pass(Q, Q, true);
    }
  }
  if (Rout) {
    // X = Q R with R = Q^T X (exact relation once Q spans X; R need not be
    // triangular for its consumers: the Jacobi SVD of the l x l factor).
    gemm_tn(h, Q, X0, *Rout);
    if (dist) allreduce_mat(h, *Rout);
  }
}

void orthonormalize(Handle& h, const DMat& X, DMat Q, DMat* R, bool dist) {
  if (X.cols > X.rows && !dist)
    throw_dim("orthonormalize: more columns than rows (" + std::to_string(X.cols) + " > " +
              std::to_string(X.rows) + ")");
  if (X.cols == 0) return;
  // Small problems (one 128/256-row block, the reference's unit-test sizes):
  // Householder in one CTA, numerically the reference's algorithm.  Otherwise
  // CholeskyQR on the DMMA pass engine (see cholqr).
  if (!dist && X.cols <= 64 && X.rows <= tsqr_block_rows(int(X.cols)))
    tsqr(h, X, Q, R, dist);
  else
    cholqr(h, X, Q, R, dist);
}

void jacobi_svd_square(Handle& h, const DMat& Rm, DMat J, DMat W, double* sigma) {
  const int l = int(Rm.rows);
  if (l > 64) {
    block_jacobi_svd(h, Rm, J, W, sigma);
    return;
  }
  if (l > 1024) throw_dim("jacobi_svd: l > 1024 not supported");
  const bool in_smem = size_t(2) * l * l * 8 <= small_smem_limit();
  double* gX = nullptr;
  double* gJ = nullptr;
  if (!in_smem) {
    gX = h.ws.alloc(int64_t(l) * l);
    gJ = h.ws.alloc(int64_t(l) * l);
  }
  const size_t dyn = in_smem ? size_t(2) * l * l * 8 : 0;
  const int pairs = (l + 1) / 2;
  if (l <= 64) {
    ensure_smem(jacobi_svd_kernel<8>, dyn);
    // l <= 32: one warp per column pair (the kernel's register path)
    const int thr = (l <= 32) ? 32 * pairs : std::max(32, int(round_up(8 * pairs, 32)));
    static const bool probe_on = std::getenv("RSVD_PROBE_FQ") != nullptr;
    double* dbg = nullptr;
    if (probe_on) {
      dbg = h.ws.alloc(128);
      RSVD_CUDA(cudaMemsetAsync(dbg, 0, 128 * 8, h.stream));
    }
    launch_k(h, jacobi_svd_kernel<8>, 1, thr, dyn, Rm.p, Rm.ld, l, J.p, J.ld, W.p, W.ld, sigma,
                                                    gX, gJ, in_smem ? 1 : 0, h.d_flags, dbg);
    if (probe_on) {
      double hd[128];
      RSVD_CUDA(cudaMemcpyAsync(hd, dbg, sizeof hd, cudaMemcpyDeviceToHost, h.stream));
      stream_sync(h);
      std::fprintf(stderr, "jacobi_svd l=%d sweeps=%d max rel g per sweep:", l, int(hd[0]));
      for (int i = 1; i <= int(hd[0]) && i < 31; ++i) std::fprintf(stderr, " %.1e", hd[i]);
      std::fprintf(stderr, "\n  round phases (cycles: load, reduce, rotation, store, barrier; round total):");
      for (int r = 0; r < 7; ++r) {
        const double* q = hd + 32 + 8 * r;
        std::fprintf(stderr, " [%.0f %.0f %.0f %.0f %.0f; %.0f]", q[1] - q[0], q[2] - q[1], q[3] - q[2],
                     q[4] - q[3], q[5] - q[4], q[8] - q[0]);
      }
      std::fprintf(stderr, "\n");
    }
  } else {
    ensure_smem(jacobi_svd_kernel<32>, dyn);
    // one warp per column pair of a round (no idle warps in the per-round barrier)
    const int thr = 32 * std::max(1, std::min(32, pairs));
    launch_k(h, jacobi_svd_kernel<32>, 1, thr, dyn, Rm.p, Rm.ld, l, J.p, J.ld, W.p, W.ld, sigma,
                                                     gX, gJ, in_smem ? 1 : 0, h.d_flags, nullptr);
  }
  RSVD_LAUNCHED(h);

}

void jacobi_evd_sym(Handle& h, const DMat& C, DMat U, double* lambda) {
  const int l = int(C.rows);
  if (l > 64) {
    evd_shifted(h, C, U, lambda);
    return;
  }
  if (l > 1024) throw_dim("jacobi_evd: l > 1024 not supported");
  const bool in_smem = size_t(2) * l * l * 8 <= small_smem_limit();
  double* gA = nullptr;
  double* gV = nullptr;
  if (!in_smem) {
    gA = h.ws.alloc(int64_t(l) * l);
    gV = h.ws.alloc(int64_t(l) * l);
  }
  ensure_smem(jacobi_evd_kernel, in_smem ? size_t(2) * l * l * 8 : 0);
  launch_k(h, jacobi_evd_kernel, 1, 1024, in_smem ? size_t(2) * l * l * 8 : 0, 
      C.p, C.ld, l, U.p, U.ld, lambda, gA, gV, in_smem ? 1 : 0, nullptr, h.d_flags);
  RSVD_LAUNCHED(h);

}

}  // namespace rsvdb
