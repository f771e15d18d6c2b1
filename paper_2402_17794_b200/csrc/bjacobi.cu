// Block one-sided Jacobi SVD for l x l factors with l > 64 (BASELINE C3-C5:
// l = 110, 220, 550), replacing the single-CTA kernel whose l - 1 rounds per
// sweep each cost a full block barrier over one SM.
//
//   M J = W diag(sigma):  columns of M are grouped in blocks of kBJ; a sweep is
//   a round-robin over block pairs (nb/2 pairs per round, all in parallel).
//   A block pair is visited by a CLUSTER of CS CTAs (CS = 1..8, chosen so the
//   visits of a round fill the SMs): CTA r of the cluster owns rows
//   [r*rp, (r+1)*rp) of the pair's two block-columns (l x 2kBJ), loads them
//   into shared memory, forms its partial 2kBJ x 2kBJ Gram with DMMA; the
//   partials are summed over distributed shared memory in rank order (every
//   CTA gets the same Gram), every CTA runs the same inner two-sided sweep on
//   it accumulating the rotation V, and applies V to its own rows of the
//   block-columns of M and J.  The l-long work of a visit is split CS ways;
//   only the 32 x 32 inner sweep is replicated.  Rounds are separated by a
//   grid-wide barrier (cooperative launch); a sweep with no rotation above
//   the threshold ends the iteration.  Deterministic: the pair schedule and
//   every reduction are fixed, no atomics on data.  The panel held per CTA is
//   rp x 2kBJ, so l is bounded only by 8 x (shared memory / 256 B).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "pass.cuh"
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

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

constexpr int kGL = 33;  // ld of the 32 x 32 Gram in shared memory
constexpr int kVL = 36;  // ld of V: 36 % 16 == 4 keeps DMMA B-fragment loads conflict-free

// Block pair visit = Gram-based inner step (Hari-Veselic block Jacobi):
//   G = Xb^T Xb (DMMA), cyclic two-sided Jacobi on the 32 x 32 G accumulating
//   the rotation V (same rotation rule and threshold as one-sided Jacobi on
//   the columns), then X(:, pair) <- Xb V and J(:, pair) <- J(:, pair) V (DMMA).
// The l-long column work is three small GEMMs instead of 31 inner rounds of
// l-long dot products; the inner rounds touch only the 32 x 32 G.  Outer
// convergence is measured on the freshly computed G of every visit, so the
// final orthogonality is that of one-sided Jacobi.
// Up to two independent problems of the same size share one launch (the
// two joint-core SVDs of Alg 6): CTAs walk the (problem, pair) items of a
// round; a converged problem's visits are skipped until both are done.
struct BJProblem {
  double* X;
  double* Jm;
  int* changed;  // kBJMaxSweeps + 3 ints: per sweep, no-convergence, zero-column count, launch shape
  unsigned long long* smax;  // per sweep: largest g^2/(a b) of the fresh Grams (bits)
};
struct BJBatch {
  BJProblem p[2];
  int nprob;
};

__global__ void __launch_bounds__(kBJThreads) bjacobi_kernel(BJBatch batch, int l, int ldp,
                                                            int rows_per, int nb, int inner_max,
                                                            double graded_ratio,
                                                            long long* __restrict__ probe) {
  RSVD_PDL_ENTRY();
  long long pt[6] = {0, 0, 0, 0, 0, 0}, tlast = clock64();
  auto mark = [&](int ph) {
    if (probe && blockIdx.x == 0 && threadIdx.x == 0) {
      const long long t = clock64();
      pt[ph] += t - tlast;
      tlast = t;
    }
  };
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = int(cluster.num_blocks()), crank = int(cluster.block_rank());
  if (cs * rows_per < l) {
    // launched without its cluster shape (seen under an ncu kernel replay):
    // the visits would miss rows -- fail loudly instead of not converging
    if (threadIdx.x == 0 && blockIdx.x == 0) batch.p[0].changed[kBJMaxSweeps + 2] = 1;
    return;
  }
  const int cid = int(blockIdx.x) / cs, ncl = int(gridDim.x) / cs;
  const int r_lo = crank * rows_per, r_hi = min(l, r_lo + rows_per), nr = max(0, r_hi - r_lo);
  extern __shared__ double sm[];
  double* Xb = sm;                           // kBJW columns x ldp local rows (rows >= nr are zero)
  double* G = Xb + size_t(kBJW) * ldp;       // kBJW x kBJW, ld kGL (the cluster's sum)
  double* V = G + kBJW * kGL;                // kBJW x kBJW, ld kVL (column-major: V[c * kVL + r])
  double* Gp = V + kBJW * kVL;               // this CTA's partial Gram, ld kGL
  double* Dp = Gp + kBJW * kGL;              // graded route: partial (a, b, g) of 16 pairs
  __shared__ int colmap[kBJW];
  __shared__ double rc[kBJW / 2], rs[kBJW / 2];
  __shared__ int rp[kBJW / 2], rq[kBJW / 2];
  __shared__ int any_first, any_inner, any_visit, graded;
  __shared__ double vmaxw[32];  // per warp: largest g^2/(a b) of this visit's Gram
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r8 = lane >> 2, c4 = lane & 3;
  const int nbp = nb + (nb & 1);
  const double tol = fmax(1e-15, 2.0 * sqrt(double(l)) * 1.1102230246251565e-16);
  const double tol2 = tol * tol;
  const int npairs = nbp / 2;
  bool done0 = false, done1 = batch.nprob < 2;  // identical in every thread
  for (int sweep = 0; sweep < kBJMaxSweeps; ++sweep) {
    for (int round = 0; round < nbp - 1; ++round) {
      for (int item = cid; item < batch.nprob * npairs; item += ncl) {
        const int prob = item / npairs, pr = item % npairs;
        if (prob == 0 ? done0 : done1) continue;
        double* __restrict__ X = batch.p[prob].X;
        double* __restrict__ Jm = batch.p[prob].Jm;
        int* __restrict__ changed = batch.p[prob].changed;
        int a, b;
        circle(pr, round, nbp, a, b);
        const int I = min(a, b), K = max(a, b);
        if (K >= nb) continue;  // dummy block
        const int wI = min(kBJ, l - I * kBJ), wK = min(kBJ, l - K * kBJ);
        const int w = wI + wK;
        if (tid < kBJW) colmap[tid] = (tid < wI) ? I * kBJ + tid : (tid < w ? K * kBJ + (tid - wI) : -1);
        if (tid == 0) any_first = any_visit = 0;
        __syncthreads();
        // ---- panel load (zero padded to kBJW columns x ldp rows)
        // warp w: columns w and w + 16, lanes along rows, 4 loads in flight
        for (int c = warp; c < kBJW; c += 16) {
          const int gc = colmap[c];
          const double* src = X + int64_t(gc < 0 ? 0 : gc) * l + r_lo;
          double* dst = Xb + c * ldp;
#pragma unroll 4
          for (int r = lane; r < ldp; r += 32) dst[r] = (gc >= 0 && r < nr) ? src[r] : 0.0;
        }
        for (int e = tid; e < kBJW * kVL; e += blockDim.x) V[e] = ((e % kVL) == (e / kVL)) ? 1.0 : 0.0;
        __syncthreads();
        mark(0);
        // ---- G = Xb^T Xb: warp -> 8 x 8 tile (ti, tj) of the 4 x 4 tile grid, K = ldp
        {
          const int ti = warp >> 2, tj = warp & 3;
          // four independent accumulator chains, K = ldp (multiple of 4)
          double g[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          const double* pa = Xb + (ti * 8 + r8) * ldp + c4;  // A(m = col, k = row)
          const double* pb = Xb + (tj * 8 + r8) * ldp + c4;  // B(k = row, n = col)
          int k0 = 0;
          for (; k0 + 16 <= ldp; k0 += 16) {
#pragma unroll
            for (int u = 0; u < 4; ++u) dmma884(g[u][0], g[u][1], pa[k0 + 4 * u], pb[k0 + 4 * u]);
          }
#pragma unroll
          for (int u = 0; u < 3; ++u)
            if (k0 + 4 * u < ldp) dmma884(g[u][0], g[u][1], pa[k0 + 4 * u], pb[k0 + 4 * u]);
          const int gi = ti * 8 + r8, gj = tj * 8 + 2 * c4;
          Gp[gi + kGL * gj] = (g[0][0] + g[1][0]) + (g[2][0] + g[3][0]);
          Gp[gi + kGL * (gj + 1)] = (g[0][1] + g[1][1]) + (g[2][1] + g[3][1]);
        }
        // the cluster's Gram: partials summed in rank order over distributed
        // shared memory (bitwise the same G in every CTA of the cluster)
        cluster.sync();
        for (int e = tid; e < kBJW * kBJW; e += blockDim.x) {
          const int o = (e % kBJW) + kGL * (e / kBJW);
          double v = 0.0;
          for (int r = 0; r < cs; ++r) v += cluster.map_shared_rank(Gp, r)[o];
          G[o] = v;
        }
        __syncthreads();
        mark(1);
        // ---- graded panel?  The Gram route below updates G by rotations, which
        // inject absolute errors ~u * max G_cc into every entry: columns whose
        // norm is below ~1e-6 of the panel's largest can then never be
        // orthogonalized (the next visit's fresh Gram shows it, and the sweep
        // never ends: rank-deficient or strongly graded factors).  Such panels
        // take the one-sided inner sweep instead: rotations from fresh dot
        // products of the panel columns themselves (relative accuracy).
        if (tid == 0) {
          double gmax = 0.0, gmin = 1e308;
          for (int c = 0; c < w; ++c) {
            const double d = G[c + kGL * c];
            gmax = fmax(gmax, d);
            if (d > 0.0) gmin = fmin(gmin, d);
          }
          graded = (gmin < graded_ratio * gmax) ? 1 : 0;
        }
        // largest relative off-diagonal of the fresh Gram (sweep stopping rule)
        {
          double vm = 0.0;
          for (int e = tid; e < kBJW * kBJW; e += blockDim.x) {
            const int i = e % kBJW, j = e / kBJW;
            if (i < j && j < w) {
              const double gij = G[i + kGL * j], dd = G[i + kGL * i] * G[j + kGL * j];
              if (dd > 0.0) vm = fmax(vm, (gij * gij) / dd);
            }
          }
          for (int o = 16; o > 0; o >>= 1) vm = fmax(vm, __shfl_xor_sync(0xffffffffu, vm, o));
          if (lane == 0) vmaxw[warp] = vm;
        }
        __syncthreads();
        const int wp = w + (w & 1), np2 = wp / 2;
        if (graded) {
          for (int it = 0; it < inner_max; ++it) {
            if (tid == 0) any_inner = 0;
            __syncthreads();
            for (int r2 = 0; r2 < wp - 1; ++r2) {
              // partial dot products of this CTA's rows, summed over the
              // cluster in rank order (distributed shared memory)
              if (warp < np2) {
                int pa, pb;
                circle(warp, r2, wp, pa, pb);
                const int p0 = min(pa, pb), q0 = max(pa, pb);
                double al = 0.0, be = 0.0, ga = 0.0;
                if (q0 < w) {
                  const double* xp = Xb + p0 * ldp;
                  const double* xq = Xb + q0 * ldp;
                  for (int r = lane; r < ldp; r += 32) {
                    const double a = xp[r], b = xq[r];
                    al = fma(a, a, al);
                    be = fma(b, b, be);
                    ga = fma(a, b, ga);
                  }
                }
                al = wsum(al);
                be = wsum(be);
                ga = wsum(ga);
                if (lane == 0) {
                  Dp[3 * warp] = al;
                  Dp[3 * warp + 1] = be;
                  Dp[3 * warp + 2] = ga;
                }
              }
              cluster.sync();
              if (warp < np2) {  // warp = pair: rotation, update of the local rows
                int pa, pb;
                circle(warp, r2, wp, pa, pb);
                const int p0 = min(pa, pb), q0 = max(pa, pb);
                if (q0 < w) {
                  double* xp = Xb + p0 * ldp;
                  double* xq = Xb + q0 * ldp;
                  double al = 0.0, be = 0.0, ga = 0.0;
                  for (int r = 0; r < cs; ++r) {
                    const double* d = cluster.map_shared_rank(Dp, r);
                    al += d[3 * warp];
                    be += d[3 * warp + 1];
                    ga += d[3 * warp + 2];
                  }
                  if (ga * ga > tol2 * (al * be) && ga != 0.0) {
                    const double d = be - al, g2 = 2.0 * ga;
                    const double ir = rsqrt(fma(d, d, g2 * g2));
                    const double hh = fma(0.5 * fabs(d), ir, 0.5);
                    const double ih = rsqrt(hh);
                    const double c = hh * ih, sn = copysign(1.0, d) * (ga * ir) * ih;
                    for (int r = lane; r < ldp; r += 32) {
                      const double a = xp[r], b = xq[r];
                      xp[r] = c * a - sn * b;
                      xq[r] = sn * a + c * b;
                    }
                    const double vp = V[lane + kVL * p0], vq = V[lane + kVL * q0];
                    V[lane + kVL * p0] = c * vp - sn * vq;
                    V[lane + kVL * q0] = sn * vp + c * vq;
                    if (lane == 0) any_inner = 1;
                  }
                }
              }
              cluster.sync();  // every CTA read the partials before they are rewritten
            }
            const int rot = any_inner;
            if (tid == 0) {
              if (it == 0) any_first = rot;
              any_visit |= rot;
            }
            __syncthreads();
            if (!rot) break;
          }
        }
        // ---- cyclic two-sided Jacobi on G (w active columns), accumulating V.
        // Per round: the wp/2 rotations (one thread each), then G <- R^T G R as
        // independent 2 x 2 blocks (pair i rows x pair j columns) and V <- V R:
        // two barriers per round.  Measured alternatives: a warp-per-pair
        // variant with rows in registers and shuffled column rotations (2x
        // slower); every thread computing its own rotations with G double
        // buffered, one barrier per round (~1300 vs ~1060 cycles per round:
        // the two dependent DP reciprocal square roots of a rotation dominate).
        double vmax_visit = 0.0;
        for (int wi = 0; wi < int(blockDim.x >> 5); ++wi) vmax_visit = fmax(vmax_visit, vmaxw[wi]);
        // a visit whose fresh Gram is diagonal to the rotation threshold makes
        // no rotation: skip its inner sweep (the clean visits of the last sweeps)
        const bool clean = !graded && !(vmax_visit > tol2);
        for (int it = 0; !graded && !clean && it < inner_max; ++it) {
          if (tid == 0) any_inner = 0;
          for (int r2 = 0; r2 < wp - 1; ++r2) {
            if (tid < np2) {
              int pa, pb;
              circle(tid, r2, wp, pa, pb);
              const int p0 = min(pa, pb), q0 = max(pa, pb);
              double c = 1.0, sn = 0.0;
              const double al = G[p0 + kGL * p0], be = G[q0 + kGL * q0], ga = G[p0 + kGL * q0];
              if (q0 < w && ga * ga > tol2 * (al * be) && ga != 0.0) {
                // rotation zeroing the (p, q) inner product (X' = X R, R = [[c, s], [-s, c]]),
                // tan(theta) = sgn(d) 2g / (|d| + r), r = |(d, 2g)|, d = G_qq - G_pp,
                // from two reciprocal square roots: c = sqrt(h), h = (1 + |d|/r) / 2,
                // s = sgn(d) g / (r c).  (A single-precision angle made orthogonal
                // to double precision by a series was measured slower: ~1300
                // vs ~1060 cycles per inner round.)
                const double d = be - al, g2 = 2.0 * ga;
                const double ir = rsqrt(fma(d, d, g2 * g2));
                const double hh = fma(0.5 * fabs(d), ir, 0.5);
                const double ih = rsqrt(hh);
                c = hh * ih;
                sn = copysign(1.0, d) * (ga * ir) * ih;
                any_inner = 1;
              }
              rc[tid] = c;
              rs[tid] = sn;
              rp[tid] = p0;
              rq[tid] = q0;
            }
            __syncthreads();
            if (tid < 256) {
              const int bi = tid >> 4, bj = tid & 15;
              if (bi < np2 && bj < np2 && (rs[bi] != 0.0 || rs[bj] != 0.0)) {
                const int pi = rp[bi], qi = rq[bi], pj = rp[bj], qj = rq[bj];
                const double ci = rc[bi], si = rs[bi], cj = rc[bj], sj = rs[bj];
                const double b00 = G[pi + kGL * pj], b01 = G[pi + kGL * qj];
                const double b10 = G[qi + kGL * pj], b11 = G[qi + kGL * qj];
                // rows: R_i^T B
                const double m00 = ci * b00 - si * b10, m01 = ci * b01 - si * b11;
                const double m10 = si * b00 + ci * b10, m11 = si * b01 + ci * b11;
                // columns: (R_i^T B) R_j
                G[pi + kGL * pj] = cj * m00 - sj * m01;
                G[pi + kGL * qj] = sj * m00 + cj * m01;
                G[qi + kGL * pj] = cj * m10 - sj * m11;
                G[qi + kGL * qj] = sj * m10 + cj * m11;
              }
            } else {
              const int k = (tid - 256) >> 4, i0 = (tid - 256) & 15;
              if (k < np2 && rs[k] != 0.0) {
                const int p0 = rp[k], q0 = rq[k];
                const double c = rc[k], sn = rs[k];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                  const int i = i0 + 16 * h2;
                  const double vp = V[i + kVL * p0], vq = V[i + kVL * q0];
                  V[i + kVL * p0] = c * vp - sn * vq;
                  V[i + kVL * q0] = sn * vp + c * vq;
                }
              }
            }
            __syncthreads();
          }
          const int rot = any_inner;
          if (tid == 0) {
            if (it == 0) any_first = rot;
            any_visit |= rot;
          }
          __syncthreads();
          if (!rot) break;
        }
        mark(2);
        if (any_visit) {
          // ---- X(:, pair) <- Xb V and J(:, pair) <- J(:, pair) V: warp -> 8-row tiles
          double vb[4][8];  // B fragments of V: [n tile][k step]
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) vb[nt][ks] = V[(nt * 8 + r8) * kVL + ks * 4 + c4];
          const int ntiles = (nr + 7) / 8;
#pragma unroll 2
          for (int mt = warp; mt < 2 * ntiles; mt += 16) {
            const bool isJ = mt >= ntiles;
            const int m0 = (isJ ? mt - ntiles : mt) * 8;  // local row tile
            if (graded && !isJ) {  // one-sided route: Xb holds the rotated columns
              const int row = m0 + r8;
              if (row < nr)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    const int cc = nt * 8 + 2 * c4 + e, gc = colmap[cc];
                    if (gc >= 0) X[int64_t(gc) * l + r_lo + row] = Xb[cc * ldp + row];
                  }
              continue;
            }
            double af[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const int k = ks * 4 + c4, row = m0 + r8;
              if (!isJ) {
                af[ks] = Xb[k * ldp + row];
              } else {
                const int gc = colmap[k];
                af[ks] = (gc >= 0 && row < nr) ? Jm[int64_t(gc) * l + r_lo + row] : 0.0;
              }
            }
            double acc[4][2];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
              for (int ks = 0; ks < 8; ++ks) dmma884(acc[nt][0], acc[nt][1], af[ks], vb[nt][ks]);
            }
            double* dst = isJ ? Jm : X;
            const int row = m0 + r8;
            if (row < nr) {
#pragma unroll
              for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int gc = colmap[nt * 8 + 2 * c4 + e];
                  if (gc >= 0) dst[int64_t(gc) * l + r_lo + row] = acc[nt][e];
                }
            }
          }
        }
        if (tid == 0 && crank == 0 && any_first) atomicOr(&changed[sweep], 1);
        // graded panels' Gram entries carry absolute rounding: no early stop
        if (tid == 0 && crank == 0) {
          const double vm = graded ? 1.0 : vmax_visit;
          atomicMax(&batch.p[prob].smax[sweep], static_cast<unsigned long long>(__double_as_longlong(vm)));
        }
        __syncthreads();
        mark(3);
      }
      grid.sync();
      mark(4);
    }
    // done: no rotation in this sweep, or the quadratic-regime stop
    auto conv = [&](const BJProblem& P) {
      if (*reinterpret_cast<volatile int*>(&P.changed[sweep]) == 0) return true;
      if (sweep == 0) return false;
      const double mk = __longlong_as_double(static_cast<long long>(
          *reinterpret_cast<volatile unsigned long long*>(&P.smax[sweep])));
      const double mp = __longlong_as_double(static_cast<long long>(
          *reinterpret_cast<volatile unsigned long long*>(&P.smax[sweep - 1])));
      return jacobi_quad_stop(mk, mp);
    };
    if (!done0) done0 = conv(batch.p[0]);
    if (!done1) done1 = conv(batch.p[1]);
    if (done0 && done1) {
      if (probe && blockIdx.x == 0 && threadIdx.x == 0)
        for (int i = 0; i < 6; ++i) probe[i] = pt[i];
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)  // no convergence
    for (int q = 0; q < batch.nprob; ++q)
      if (!(q == 0 ? done0 : done1)) batch.p[q].changed[kBJMaxSweeps] = 1;
}

// column norms (sigma), stable descending order, permuted outputs
__global__ void bj_norms_kernel(const double* __restrict__ X, int l, double* __restrict__ nrm) {
  RSVD_PDL_ENTRY();
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
  RSVD_PDL_ENTRY();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < l; j += gridDim.x * blockDim.x) {
    const double v = order_key(nrm[j]);
    int rank = 0;
    for (int k = 0; k < l; ++k) {
      const double u = order_key(nrm[k]);
      if (u > v || (u == v && k < j)) ++rank;
    }
    order[rank] = j;
    sigma[rank] = nrm[j];
  }
}

__global__ void bj_permute_kernel(const double* __restrict__ X, const double* __restrict__ Jm,
                                  const double* __restrict__ nrm, const int* __restrict__ order,
                                  int l, double* __restrict__ Jout, int64_t ldj,
                                  double* __restrict__ Wout, int64_t ldw, int* __restrict__ nzero) {
  RSVD_PDL_ENTRY();
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
  RSVD_PDL_ENTRY();
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
  RSVD_PDL_ENTRY();
  const int64_t n = int64_t(l) * l;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e % l), j = int(e / l);
    X[e] = Rm[int64_t(j) * ldr + i];
    Jm[e] = (i == j) ? 1.0 : 0.0;
  }
}

__global__ void bj_flag_kernel(const int* changed, int* flags) {
  RSVD_PDL_ENTRY();
  if (changed[kBJMaxSweeps]) atomicOr(flags, kFlagJacobiNoConv);
  if (changed[kBJMaxSweeps + 2]) atomicOr(flags, kFlagLaunchShape);
}

// mu >= max_i sum_j |c_ij| >= |lambda|_max (Gershgorin): C + mu I is PSD.
__global__ void gershgorin_kernel(const double* __restrict__ C, int64_t ldc, int l,
                                  double* __restrict__ mu) {
  RSVD_PDL_ENTRY();
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
  RSVD_PDL_ENTRY();
  const int64_t n = int64_t(l) * l;
  const double m = *mu;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e % l), j = int(e / l);
    T[e] = C[int64_t(j) * ldc + i] + (i == j ? m : 0.0);
  }
}

// Rayleigh quotients lambda_j = u_j^T (C u_j) of the computed eigenvectors (one
// CTA per column).  Second-order accurate in the eigenvector error, unlike
// sigma_j - mu, whose absolute error carries the shift mu and the rounding
// of every accumulated rotation.
__global__ void rayleigh_kernel(const double* __restrict__ Jm, int64_t ldj,
                                const double* __restrict__ CJ, int64_t ldc, int l,
                                double* __restrict__ lam) {
  RSVD_PDL_ENTRY();
  const int c = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < l; i += blockDim.x) s = fma(Jm[int64_t(c) * ldj + i], CJ[int64_t(c) * ldc + i], s);
  __shared__ double red[8];
  s = wsum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    lam[c] = t;
  }
}

// eigenvalues (Rayleigh quotients) reordered by |lambda| descending; exact
// ties: positive first (see evd_symmetric in small.cu / the oracle).
__global__ void evd_order_kernel(const double* __restrict__ lam_in, int l,
                                 double* __restrict__ lambda, int* __restrict__ order) {
  RSVD_PDL_ENTRY();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < l; j += gridDim.x * blockDim.x) {
    const double v0 = lam_in[j], v = (v0 != v0) ? 0.0 : v0, av = order_key(fabs(v0));
    int rank = 0;
    for (int k = 0; k < l; ++k) {
      const double u0 = lam_in[k], u = (u0 != u0) ? 0.0 : u0, au = order_key(fabs(u0));
      if (au > av || (au == av && (u > v || (u == v && k < j)))) ++rank;
    }
    order[rank] = j;
    lambda[rank] = v0;
  }
}

__global__ void evd_permute_kernel(const double* __restrict__ Jm, int64_t ldj, int l,
                                   const int* __restrict__ order, double* __restrict__ U,
                                   int64_t ldu) {
  RSVD_PDL_ENTRY();
  const int jn = blockIdx.x, src = order[jn];
  for (int i = threadIdx.x; i < l; i += blockDim.x) U[int64_t(jn) * ldu + i] = Jm[int64_t(src) * ldj + i];
}

}  // namespace

namespace {
struct BJWork {
  double *X, *Jm, *nrm;
  int *order, *changed, *nzero;
  unsigned long long* smax;
};

BJWork bj_prepare(Handle& h, const DMat& Rm) {
  const int l = int(Rm.rows);
  BJWork w;
  w.X = h.ws.alloc(int64_t(l) * l);
  w.Jm = h.ws.alloc(int64_t(l) * l);
  w.nrm = h.ws.alloc(l);
  w.order = reinterpret_cast<int*>(h.ws.alloc_bytes(size_t(l) * 4 + 16));
  const size_t cb = size_t(kBJMaxSweeps + 4) * 4, mb = size_t(kBJMaxSweeps) * 8;
  w.changed = reinterpret_cast<int*>(h.ws.alloc_bytes(cb + mb));  // 256-byte aligned
  w.nzero = w.changed + kBJMaxSweeps + 1;
  w.smax = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(w.changed) + cb);
  RSVD_CUDA(cudaMemsetAsync(w.changed, 0, cb + mb, h.stream));
  launch_k(h, bj_init_kernel, std::max(1, std::min(4 * h.sm_count, (l * l + 255) / 256)), 256, 0, 
      Rm.p, Rm.ld, l, w.X, w.Jm);
  RSVD_LAUNCHED(h);
  return w;
}

void bj_finish(Handle& h, const BJWork& w, int l, DMat J, DMat W, double* sigma) {
  launch_k(h, bj_flag_kernel, 1, 1, 0, w.changed, h.d_flags);
  RSVD_LAUNCHED(h);
  launch_k(h, bj_norms_kernel, l, 256, 0, w.X, l, w.nrm);
  RSVD_LAUNCHED(h);
  launch_k(h, bj_order_kernel, (l + 255) / 256, 256, 0, w.nrm, l, w.order, sigma);
  RSVD_LAUNCHED(h);
  launch_k(h, bj_permute_kernel, l, 128, 0, w.X, w.Jm, w.nrm, w.order, l, J.p, J.ld, W.p, W.ld,
                                            w.nzero);
  RSVD_LAUNCHED(h);
  launch_k(h, bj_complete_kernel, 1, 32, 0, sigma, l, W.p, W.ld, w.nzero);
  RSVD_LAUNCHED(h);
}

// One cooperative launch over 1 or 2 problems of size l.
void bj_run(Handle& h, int l, const BJWork* work, int nprob) {
  const int nb = (l + kBJ - 1) / kBJ;
  // panel rows padded to ldp = l rounded up to 8 with ldp % 16 in {4, 12}... use the
  // smallest ldp >= l, ldp % 4 == 0, (ldp / 4) odd: conflict-free DMMA fragment loads
  const int nbp = nb + (nb & 1);
  const int items = nprob * (nbp / 2);
  // cluster size: split each visit's rows CS ways (any CS in 1..8: clusters
  // must fit inside a GPC, so e.g. 36 visits fit as clusters of 3 but not of
  // 4) -- the largest CS whose clusters all fit the SMs at once and whose
  // row slices stay >= 16 rows; RSVD_BJ_CLUSTER overrides (1 = unsplit)
  const int cs_env = std::getenv("RSVD_BJ_CLUSTER") ? std::atoi(std::getenv("RSVD_BJ_CLUSTER")) : 0;
  auto panel_ld = [](int rows) {
    int ld = (rows + 3) / 4 * 4;
    if ((ld / 4) % 2 == 0) ld += 4;
    return ld;
  };
  auto smem_of = [&](int c) {
    const int rpc = int(ceil_div(l, c));
    return (size_t(panel_ld(rpc)) * kBJW + 2 * kBJW * kGL + kBJW * kVL + 64) * 8;
  };
  // co-residency (cooperative launch): at most the device's active clusters
  auto max_clusters = [&](int c) {
    smem_attr(bjacobi_kernel, smem_of(c));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(c * std::max(1, h.sm_count / c)));
    cfg.blockDim = dim3(kBJThreads);
    cfg.dynamicSmemBytes = smem_of(c);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(c);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    RSVD_CUDA(cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(bjacobi_kernel), &cfg));
    return n;
  };
  int cs = 1, ncl_max = 0;
  if (cs_env > 0) {
    cs = std::min(8, cs_env);
    ncl_max = max_clusters(cs);
  } else {
    for (int c = 8; c >= 1; --c) {
      const bool fits_smem = smem_of(c) <= 220 * 1024;
      if (!fits_smem) break;  // smaller clusters need even more shared memory
      if (c > 1 && (items * c > h.sm_count || ceil_div(l, c) < 16)) continue;
      const int n = max_clusters(c);
      if (n >= std::min(items, h.sm_count / c) || c == 1) {
        cs = c;
        ncl_max = n;
        break;
      }
    }
    if (ncl_max == 0) {  // large l: the smallest split that fits shared memory
      cs = 1;
      while (cs < 8 && smem_of(cs) > 220 * 1024) ++cs;
      ncl_max = max_clusters(cs);
    }
  }
  if (ncl_max < 1) throw_dim("block_jacobi_svd: no co-resident cluster fits");
  const size_t smem = smem_of(cs);
  if (smem > 227 * 1024) throw_dim("block_jacobi_svd: l too large for a block pair on 8 SMs");
  const int rp = int(ceil_div(l, cs));
  const int ldp = panel_ld(rp);
  smem_attr(bjacobi_kernel, smem);
  BJBatch batch{};
  batch.nprob = nprob;
  for (int q = 0; q < 2; ++q) {
    const BJWork& w = work[q < nprob ? q : 0];
    batch.p[q] = BJProblem{w.X, w.Jm, w.changed, w.smax};
  }
  int nbv = nb, lv = l, ldpv = ldp, rpv = rp;
  // one inner sweep per visit: more inner sweeps do not reduce the outer sweep
  // count measurably (C3-C5 shapes)
  static const int inner_env = std::getenv("RSVD_BJ_INNER") ? std::atoi(std::getenv("RSVD_BJ_INNER")) : 1;
  int inner = inner_env;
  int grid = cs * std::max(1, std::min(std::min(items, h.sm_count / cs), ncl_max));
  static const double graded_env =
      std::getenv("RSVD_BJ_GRADED") ? std::atof(std::getenv("RSVD_BJ_GRADED")) : 1e-12;
  double graded_ratio = graded_env;
  long long* probe = nullptr;
  static const bool probe_on = std::getenv("RSVD_PROBE_FQ") != nullptr;
  if (probe_on) {
    probe = reinterpret_cast<long long*>(h.ws.alloc_bytes(8 * 8));
    RSVD_CUDA(cudaMemsetAsync(probe, 0, 64, h.stream));
  }
  void* args[] = {&batch, &lv, &ldpv, &rpv, &nbv, &inner, &graded_ratio, &probe};
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (probe_on) {
    cudaEventCreate(&pe0);
    cudaEventCreate(&pe1);
    cudaEventRecord(pe0, h.stream);
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBJThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h.stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = unsigned(cs);
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    RSVD_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(bjacobi_kernel), args));
  }
  RSVD_LAUNCHED(h);
  if (probe_on) {
    cudaEventRecord(pe1, h.stream);
    int hc[kBJMaxSweeps + 1];
    double hm[kBJMaxSweeps];
    RSVD_CUDA(cudaMemcpyAsync(hc, work[0].changed, sizeof hc, cudaMemcpyDeviceToHost, h.stream));
    RSVD_CUDA(cudaMemcpyAsync(hm, work[0].smax, sizeof hm, cudaMemcpyDeviceToHost, h.stream));
    stream_sync(h);
    std::fprintf(stderr, "bjacobi max rel g per sweep:");
    for (int i = 0; i < kBJMaxSweeps && hm[i] > 0.0; ++i) std::fprintf(stderr, " %.1e", std::sqrt(hm[i]));
    std::fprintf(stderr, "\n");
    float ms = 0;
    cudaEventElapsedTime(&ms, pe0, pe1);
    int sw = 0;
    while (sw < kBJMaxSweeps && hc[sw]) ++sw;
    long long hp[6];
    RSVD_CUDA(cudaMemcpy(hp, probe, sizeof hp, cudaMemcpyDeviceToHost));
    std::fprintf(stderr,
                 "bjacobi l=%d nb=%d nprob=%d grid=%d cluster=%d sweeps=%d (+1 clean) %.3f ms  cycles load %lld "
                 "gram %lld inner %lld update %lld gridsync %lld\n",
                 l, nb, nprob, grid, cs, sw, ms, hp[0], hp[1], hp[2], hp[3], hp[4]);
    cudaEventDestroy(pe0);
    cudaEventDestroy(pe1);
  }
}
}  // namespace

void block_jacobi_svd(Handle& h, const DMat& Rm, DMat J, DMat W, double* sigma) {
  const int l = int(Rm.rows);
  const BJWork w = bj_prepare(h, Rm);
  bj_run(h, l, &w, 1);
  bj_finish(h, w, l, J, W, sigma);
}

void block_jacobi_svd2(Handle& h, const DMat& R0, DMat J0, DMat W0, double* s0, const DMat& R1,
                       DMat J1, DMat W1, double* s1) {
  const int l = int(R0.rows);
  if (R1.rows != l) throw_dim("block_jacobi_svd2: sizes differ");
  const BJWork w[2] = {bj_prepare(h, R0), bj_prepare(h, R1)};
  bj_run(h, l, w, 2);
  bj_finish(h, w[0], l, J0, W0, s0);
  bj_finish(h, w[1], l, J1, W1, s1);
}

// Symmetric EVD for l > 64: the SVD of the positive semidefinite C + mu I
// (right singular vectors = eigenvectors, sigma = lambda + mu).  Eigenvalues
// carry an absolute error ~eps * ||C||, the accuracy class of the reference's
// tridiagonal-QR eigensolver.
void evd_shifted(Handle& h, const DMat& C, DMat U, double* lambda) {
  const int l = int(C.rows);
  double* mu = h.ws.alloc(1);
  launch_k(h, gershgorin_kernel, 1, 256, 0, C.p, C.ld, l, mu);
  RSVD_LAUNCHED(h);
  DMat T = h.ws.mat(l, l), Jm = h.ws.mat(l, l), W = h.ws.mat(l, l);
  launch_k(h, shift_copy_kernel, std::max(1, std::min(4 * h.sm_count, (l * l + 255) / 256)), 256, 0, 
      C.p, C.ld, l, mu, T.p);
  RSVD_LAUNCHED(h);
  double* sg = h.ws.alloc(l);
  block_jacobi_svd(h, DMat(T.p, l, l, l), Jm, W, sg);
  int* order = reinterpret_cast<int*>(h.ws.alloc_bytes(size_t(l) * 4 + 16));
  DMat CJ = h.ws.mat(l, l);
  gemm_nn(h, C, Jm, CJ);
  double* rq = h.ws.alloc(l);
  launch_k(h, rayleigh_kernel, l, 128, 0, Jm.p, Jm.ld, CJ.p, CJ.ld, l, rq);
  RSVD_LAUNCHED(h);
  launch_k(h, evd_order_kernel, (l + 255) / 256, 256, 0, rq, l, lambda, order);
  RSVD_LAUNCHED(h);
  launch_k(h, evd_permute_kernel, l, 128, 0, Jm.p, Jm.ld, l, order, U.p, U.ld);
  RSVD_LAUNCHED(h);
}

}  // namespace rsvdb
