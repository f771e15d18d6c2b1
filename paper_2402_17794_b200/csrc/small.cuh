// Small dense kernels of the rsvd hot path (small.cu): orthonormalization
// (Householder TSQR / CholeskyQR2), the l x l one-sided Jacobi SVD, the
// symmetric Jacobi EVD, the sign rule, and helpers.
#pragma once
#include "common.cuh"

namespace rsvdb {

// Q (m x l) with range(Q) >= range(X), always exactly l orthonormal columns
// (reference core.hpp:93-105).  If R != nullptr it receives the l x l factor
// with X = Q R.  X and Q may alias.  dist: X is this rank's row shard of a
// row-sharded matrix (NCCL exchange of l x l factors only).
void orthonormalize(Handle& h, const DMat& X, DMat Q, DMat* R = nullptr, bool dist = false);

// Householder TSQR (any conditioning, rank-deficient inputs padded), l <= 64.
void tsqr(Handle& h, const DMat& X, DMat Q, DMat* R, bool dist);

// One-sided Jacobi on a square l x l matrix Rm:  Rm J = W diag(sigma).
// sigma descending (stable), J orthogonal, W orthonormal (zero-sigma columns
// completed to an orthonormal set).  Device outputs.
void jacobi_svd_square(Handle& h, const DMat& Rm, DMat J, DMat W, double* sigma);
// Cholesky G + s I = R^T R and R^-1 of an l x l Gram on the whole GPU (cholblk.cu).
void chol_inv_blocked(Handle& h, const DMat& G, int l, double shift_coef, DMat R, DMat Rinv,
                      int* shift_used);

// Block one-sided Jacobi (cooperative, multi-CTA) for l > 64 (bjacobi.cu).
void block_jacobi_svd(Handle& h, const DMat& Rm, DMat J, DMat W, double* sigma);
// Two independent l x l problems (l > 64) in one cooperative launch.
void block_jacobi_svd2(Handle& h, const DMat& R0, DMat J0, DMat W0, double* s0, const DMat& R1,
                       DMat J1, DMat W1, double* s1);
// Symmetric EVD for l > 64 via the SVD of C + mu I (bjacobi.cu).
void evd_shifted(Handle& h, const DMat& C, DMat U, double* lambda);

// Symmetric two-sided Jacobi EVD of an l x l symmetric matrix (device), with
// eigenvalues reordered by |lambda| descending, stable (core.hpp:148-152).
void jacobi_evd_sym(Handle& h, const DMat& C, DMat U, double* lambda);

// Reference sign rule (core.hpp:115-122): for each column j of U, the entry of
// largest magnitude (lowest row on ties) is made >= 0; the flip is applied to
// column j of V too (V may be null).
void sign_rule(Handle& h, DMat U, DMat* V);

// out = in^T
void transpose(Handle& h, const DMat& in, DMat out);
// Y = X (copy, shapes equal)
void copy(Handle& h, const DMat& X, DMat Y);
// columns j of X scaled by s[j] (device vector), or by 1/s[j] when inv
void scale_cols(Handle& h, DMat X, const double* s, bool inv);
// C = alpha*(A + B^T) elementwise (square)
void sym_part(Handle& h, const DMat& A, DMat C);
// Set device flag if any entry of X is not finite.
void check_finite(Handle& h, const DMat& X, int flag_bit);

// Quadratic-convergence stop of the cyclic Jacobi sweeps.  e_k = the largest
// relative inner product |g| / sqrt(a b) met in sweep k.  Once the sweeps are
// in the quadratic regime (e_k <= 100 e_{k-1}^2) and e_k <= 1e-7, the next
// sweep would meet terms ~100 e_k^2 <= 1e-12 relative at most (measured on
// the C1 / C2 Stage-2 factors: e = .., 4.3e-4, 1.8e-8, 9.4e-16 and
// .., 2.2e-3, 1.2e-9, 1.1e-15): it is skipped instead of run as a
// (near) rotation-free confirmation sweep.  Compared in squares.
constexpr double kJacobiStop2 = 1e-14;   // (1e-7)^2
constexpr double kJacobiQuadK2 = 1e4;    // 100^2
__host__ __device__ inline bool jacobi_quad_stop(double m_k, double m_prev) {
  return m_k <= kJacobiStop2 && m_k <= kJacobiQuadK2 * m_prev * m_prev;
}

enum FlagBits : int {
  kFlagNonFinite = 1,
  kFlagJacobiNoConv = 2,
  kFlagRngExhausted = 4,
  kFlagAsymmetric = 8,
  kFlagCholBreakdown = 16,
  kFlagPowerCap = 32,
  kFlagRngPatchOverflow = 64,
  kFlagRetryRobust = 128,  // not an error: re-run the call in robust mode
  kFlagLaunchShape = 256,  // a cluster kernel ran without its cluster shape
};
// Raises NumericError if any flag is set (synchronizes the stream).
void check_flags(Handle& h, const char* what);
void clear_flags(Handle& h);

}  // namespace rsvdb
