// Batched trials (trials.cu): the run_bounds / run_angles trial loops with
// every streaming pass fused across trials.
#pragma once
#include "common.cuh"
#include "engine.cuh"

namespace rsvdb {
// the reference's Rng(seed) state (sketch.hpp:36)
void seeded_state(uint64_t seed, rsvd_rng_state* st);
void range_basis_trials_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                             uint64_t seed_base, int64_t T, DMat Qall);
void rsvd_trials_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                      uint64_t seed_base, int64_t T, DMat U, double* sigma, DMat V);
void range_error_trials_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                             uint64_t seed_base, int64_t T, double* errors);
}  // namespace rsvdb
