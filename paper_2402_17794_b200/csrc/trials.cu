// Batched trials: the trial loops of the reference's
// run_bounds / run_angles (drivers.hpp:340-356, 400-431), where trial t
// re-runs Stage 1 (or the whole rsvd) with Rng(seed + t) (sketch.hpp:37-39).
//
// B200 mapping.  The reference repeats every streaming pass over A once per
// trial.  Here the T trials' sketches sit side by side, Omega_all =
// [Omega_1 ... Omega_T] (n x T l), so every pass of the range finder --
// A Omega, the power steps A^T Y / A Z, and Stage 2's A^T Q -- is ONE pass
// over A of width T l: A is read once for all trials and the pass moves from
// the FP64/HBM ridge (l = 25) to the compute-bound regime of the C3-C5
// shapes.  Only the per-trial orthonormalizations, small SVDs and lifts stay
// per trial (they are independent column blocks).  Each trial's result is
// the single-trial result up to rounding (the fused pass sums in a different
// split-K order), and its Omega_t is bit-for-bit the one Rng(seed + t) draws.
#include <algorithm>
#include <random>
#include <sstream>
#include <vector>

#include "common.cuh"
#include "diag.cuh"
#include "engine.cuh"
#include "pass.cuh"
#include "rng.cuh"
#include "small.cuh"
#include "trials.cuh"

namespace rsvdb {

// The reference's Rng(seed) state: std::mt19937_64(seed) (sketch.hpp:36), no
// cached normal.
void seeded_state(uint64_t seed, rsvd_rng_state* st) {
  std::mt19937_64 eng(seed);
  std::stringstream ss;
  ss << eng;
  for (auto& w : st->mt) ss >> w;
  ss >> st->pos;
  st->has_cached = 0;
  st->pad_ = 0;
  st->cached = 0.0;
}

namespace {

DMat block(const DMat& X, int64_t t, int64_t l) { return DMat(X.p + t * l * X.ld, X.rows, l, X.ld); }

// Omega_all columns [t l, (t + 1) l) = gaussian(n, l, Rng(seed_base + t)).
// All T states are staged in one pinned buffer and uploaded with one copy.
void gaussian_trials(Handle& h, int64_t n, int64_t l, uint64_t seed_base, int64_t T, DMat Om) {
  if (T > h.h_rng_batch_cap) {
    if (h.h_rng_batch) {
      stream_sync(h);
      RSVD_CUDA(cudaFreeHost(h.h_rng_batch));
    }
    RSVD_CUDA(cudaMallocHost(&h.h_rng_batch, size_t(T) * sizeof(rsvd_rng_state)));
    h.h_rng_batch_cap = T;
  } else {
    stream_sync(h);  // the staging buffer may still be in flight
  }
  for (int64_t t = 0; t < T; ++t) seeded_state(seed_base + uint64_t(t), h.h_rng_batch + t);
  auto* d = static_cast<rsvd_rng_state*>(h.ws.alloc_bytes(size_t(T) * sizeof(rsvd_rng_state)));
  RSVD_CUDA(cudaMemcpyAsync(d, h.h_rng_batch, size_t(T) * sizeof(rsvd_rng_state),
                            cudaMemcpyHostToDevice, h.stream));
  for (int64_t t = 0; t < T; ++t) {
    DevRng r;
    r.d = d + t;
    r.has_cached = 0;
    gaussian_dev(h, n, l, r, block(Om, t, l));
  }
}

void check_trials(const Problem& P, int64_t k, int64_t p, int q, int mode, int64_t T) {
  if (T < 1) throw_param("trials must be >= 1");
  if (mode < 0 || mode > 2) throw_param("unknown range mode");
  if (k < 1) throw_param("target rank k must be >= 1");
  if (p < 0) throw_param("oversampling p must be >= 0");
  if (q < 0) throw_param("power steps q must be >= 0");
  const int64_t mn = std::min(P.m_global, P.A.cols);
  if (k + p > mn)
    throw_dim("k+p = " + std::to_string(k + p) + " exceeds min(m,n) = " + std::to_string(mn));
}

}  // namespace

// Stage 1 of every trial (rangefinder.hpp:60-105): Qall (m x T l), block t =
// range_basis(A, cfg, Rng(seed_base + t)).
void range_basis_trials_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                             uint64_t seed_base, int64_t T, DMat Qall) {
  if (mode == RSVD_MODE_BASIC) q = 0;  // SketchConfig::normalized (rangefinder.hpp:37-41)
  check_trials(P, k, p, q, mode, T);
  const int64_t n = P.A.cols, ml = P.A.rows, l = k + p, L = T * l;
  // the shared passes are T l columns wide: from ~100 columns up they run on
  // the INT8 tensor cores with A's slices cached for the call (ozaki.cu)
  if (P.oz_passes == 0) P.oz_passes = 2 * q + 1;
  DMat Om = h.ws.mat(n, L);
  gaussian_trials(h, n, l, seed_base, T, Om);
  DMat Y = h.ws.mat(ml, L);
  op_apply(h, P, Om, Y);  // A [Omega_1 ... Omega_T]: one pass for all trials
  auto orth_all = [&](const DMat& X, DMat Qo, bool dist) {
    for (int64_t t = 0; t < T; ++t) orthonormalize(h, block(X, t, l), block(Qo, t, l), nullptr, dist);
  };
  if (mode == RSVD_MODE_POWER) {
    DMat Z = h.ws.mat(n, L);
    for (int j = 0; j < q; ++j) {  // rangefinder.hpp:74-77, every trial in the same pass
      op_adjoint(h, P, Y, Z);
      op_apply(h, P, Z, Y);
    }
    orth_all(Y, Qall, P.dist);
  } else if (mode == RSVD_MODE_POWER_ORTHO) {
    orth_all(Y, Qall, P.dist);
    DMat Z = h.ws.mat(n, L), W = h.ws.mat(n, L);
    for (int j = 0; j < q; ++j) {  // rangefinder.hpp:89-92
      op_adjoint(h, P, Qall, Z);
      orth_all(Z, W, false);
      op_apply(h, P, W, Y);
      orth_all(Y, Qall, P.dist);
    }
  } else {
    orth_all(Y, Qall, P.dist);
  }
}

// rsvd of every trial (factor.hpp:12-24): block t of U (m x T l), sigma (T l),
// V (n x T l) = rsvd(A, cfg, Rng(seed_base + t)).
void rsvd_trials_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                      uint64_t seed_base, int64_t T, DMat U, double* sigma, DMat V) {
  const int64_t n = P.A.cols, ml = P.A.rows, l = k + p, L = T * l;
  DMat Q = h.ws.mat(ml, L);
  P.oz_passes = 2 * (mode == RSVD_MODE_BASIC ? 0 : q) + 2;
  range_basis_trials_impl(h, P, k, p, q, mode, seed_base, T, Q);
  DMat Z = h.ws.mat(n, L);
  op_adjoint(h, P, Q, Z);  // B_t^T = A^T Q_t for every trial: one pass
  for (int64_t t = 0; t < T; ++t)  // as rsvd_impl (engine.cu), per trial
    rsvd_stage2(h, block(Q, t, l), block(Z, t, l), block(U, t, l), sigma + t * l, block(V, t, l));
}

// computed_range_error (bounds.hpp:107-120) of every trial's Stage-1 basis:
// the run_bounds loop (drivers.hpp:343-346).  Host output.
void range_error_trials_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                             uint64_t seed_base, int64_t T, double* errors) {
  const int64_t l = k + p;
  DMat Q = h.ws.mat(P.A.rows, T * l);
  range_basis_trials_impl(h, P, k, p, q, mode, seed_base, T, Q);
  DMat R = h.ws.mat(P.A.rows, P.A.cols);  // one residual buffer, reused by every trial
  for (int64_t t = 0; t < T; ++t) errors[t] = computed_range_error_impl(h, P.A, block(Q, t, l), &R);
}

}  // namespace rsvdb
