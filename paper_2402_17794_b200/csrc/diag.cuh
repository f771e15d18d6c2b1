// Residual and subspace diagnostics (diag.cu): reference core.hpp:180-221,
// bounds.hpp:107-120, angles.hpp:24-60.
#pragma once
#include "common.cuh"

namespace rsvdb {
// singular values of M, descending (core.hpp:180-183); s has min(m, n) entries
void singular_values_impl(Handle& h, const DMat& M, double* s);
// max |G - I| of a Gram (synchronizes)
double gram_deviation(Handle& h, const DMat& G);
// max |G - I| into *d (device, zeroed by the caller; atomic max), no host read
void gram_deviation_dev(Handle& h, const DMat& G, double* d);
// max |X^T X - I| (synchronizes)
double orthonormal_deviation(Handle& h, const DMat& X);
// R = A - Q Z^T  (A m x n, Q m x l, Z n x l)
void residual_lowrank(Handle& h, const DMat& A, const DMat& Q, const DMat& Z, DMat R);
// ||M||_2 (core.hpp:188-221); iterations: power steps taken (0 on the dense route)
double spectral_norm_impl(Handle& h, const DMat& M, int64_t* iterations);
// ||A - Q Q^T A||_2 (bounds.hpp:107-120); resid: optional m x n scratch for the residual
double computed_range_error_impl(Handle& h, const DMat& A, const DMat& Q, DMat* resid = nullptr);
// ascending sines of the principal angles between range(X) and range(Y),
// min(cols X, cols Y) of them, clamped to [0, 1] (angles.hpp:42-60)
void canonical_sines_impl(Handle& h, const DMat& X, const DMat& Y, double* out);
// ||M||_F (deterministic reduction; synchronizes)
double frobenius_impl(Handle& h, const DMat& M);
// run_svd's error report (reference drivers.hpp:145-151) for A ~ U diag(s) V^T:
// relative Frobenius and spectral norms of the residual, on the device
void reconstruction_error_impl(Handle& h, const DMat& A, const DMat& U, const double* s,
                               const DMat& V, double* rel_fro, double* rel_spec);
}  // namespace rsvdb
