/*
 * rsvd_b200.h — C ABI of the B200-native randomized-SVD engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (reference proj/include/rsvd/ sketch, rangefinder, factor, singlepass,
 * core .hpp).  The reference has no FFI of its own: its "operator API" is the
 * header-only C++ namespace rsvd.  The headers in include/rsvd/ re-expose it
 * (same names, argument meaning and exceptions) on top of the entry points
 * below; INTEGRATION.md shows how a maintainer binds them.
 *
 * Conventions
 *  - Every matrix is column-major double precision (reference core.hpp:1-4),
 *    given as (pointer, rows, cols, leading dimension).
 *  - Functions named *_dev take DEVICE pointers on the handle's GPU and run on
 *    the handle's stream; A is never modified.  Functions named *_host take
 *    HOST pointers (pageable or pinned) and include the host<->device copies.
 *  - Multi-GPU (row-sharded A): a handle created with rsvd_create_dist holds
 *    rows [row_offset, row_offset + m_local) of A on each rank; per-rank
 *    outputs are the local rows of U / Q, while V, sigma, lambda are
 *    replicated.  Only l x n / n x l / l x l partials cross NVLink (NCCL).
 *  - Errors are returned as rsvd_status; the C++ layer rethrows them as the
 *    reference's DimensionError / ParameterError / NumericError
 *    (core.hpp:23-39).  rsvd_last_error() returns the message (thread-local).
 *  - The RNG is the reference's stream: std::mt19937_64 feeding
 *    std::normal_distribution<double> (sketch.hpp:19-45).  Its full state
 *    (312-word MT vector, position, cached second polar variate) is passed in
 *    and returned advanced by exactly the draws consumed, so a host
 *    rsvd::Rng continues bit-identically after a device call.
 */
#ifndef RSVD_B200_H_
#define RSVD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum rsvd_status {
  RSVD_OK = 0,
  RSVD_ERR_DIMENSION = 1, /* reference DimensionError (std::invalid_argument) */
  RSVD_ERR_PARAMETER = 2, /* reference ParameterError (std::invalid_argument) */
  RSVD_ERR_NUMERIC = 3,   /* reference NumericError (std::runtime_error)      */
  RSVD_ERR_CUDA = 4,
  RSVD_ERR_NCCL = 5,
  RSVD_ERR_INTERNAL = 9
} rsvd_status;

/* RangeMode, reference rangefinder.hpp:13-17. */
typedef enum rsvd_range_mode {
  RSVD_MODE_BASIC = 0,
  RSVD_MODE_POWER = 1,
  RSVD_MODE_POWER_ORTHO = 2
} rsvd_range_mode;

/* Full state of the reference Rng (sketch.hpp:41-44): mt19937_64's 312-word
 * vector and index (libstdc++ _M_x / _M_p), plus normal_distribution's cached
 * second polar variate (_M_saved_available / _M_saved). */
typedef struct rsvd_rng_state {
  uint64_t mt[312];
  uint64_t pos;
  int32_t has_cached;
  int32_t pad_;
  double cached;
} rsvd_rng_state;

/* Block-application counters: the reference CountingOperator contract
 * (singlepass.hpp:15-40) plus the number of physical streaming passes over A
 * (a fused Alg-6 pass counts one apply, one adjoint and ONE physical pass). */
typedef struct rsvd_counters {
  int64_t apply;
  int64_t adjoint;
  int64_t physical_passes;
  int64_t kernel_launches;
  /* calls re-run in robust mode because a speculated, sync-free branch
   * decision (CholeskyQR's pass count) turned out wrong */
  int64_t robust_reruns;
} rsvd_counters;

typedef struct rsvd_handle rsvd_handle;

/* ---------------------------------------------------------------- handle */
rsvd_status rsvd_create(rsvd_handle** h, int device);
/* Multi-GPU: one handle per rank/GPU.  nccl_id is the 128-byte ncclUniqueId
 * produced by rsvd_nccl_unique_id on rank 0 and broadcast by the caller.
 * nranks == 1 with a non-null id builds a one-rank communicator: the
 * row-sharded code path, every NCCL exchange included, on a single GPU. */
rsvd_status rsvd_nccl_unique_id(void* nccl_id_out128);
rsvd_status rsvd_create_dist(rsvd_handle** h, int device, int rank, int nranks,
                             const void* nccl_id128);
void rsvd_destroy(rsvd_handle* h);
const char* rsvd_last_error(void);
const char* rsvd_version(void);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores
 * the handle's own non-blocking stream, on which every call first waits for
 * the work already queued on the legacy default stream (the caller's inputs). */
/* Virtual communicator: nranks ranks of the row-sharded engine in ONE process
 * on ONE device (one host thread per rank, one handle per rank, one shared
 * stream; fixed-order device reductions stand in for NCCL).  Runs the
 * multi-GPU code path -- shard offsets, Psi row selection, distributed
 * CholeskyQR / TSQR, every exchange -- for tests without P GPUs. */
typedef struct rsvd_vcomm rsvd_vcomm;
rsvd_status rsvd_vcomm_create(rsvd_vcomm** vc, int nranks);
void rsvd_vcomm_destroy(rsvd_vcomm* vc);
rsvd_status rsvd_create_virtual(rsvd_handle** h, int device, int rank, rsvd_vcomm* vc);
/* Shard descriptor of a distributed handle: the global row count and this
 * rank's first row (so a call needs no row-count exchange; 0, 0 = exchange). */
rsvd_status rsvd_set_shard(rsvd_handle* h, int64_t m_global, int64_t row_offset);

rsvd_status rsvd_set_stream(rsvd_handle* h, void* cuda_stream);
rsvd_status rsvd_synchronize(rsvd_handle* h);
rsvd_status rsvd_get_counters(rsvd_handle* h, rsvd_counters* out);
rsvd_status rsvd_reset_counters(rsvd_handle* h);
/* Live timing of the streaming-pass kernels: when enabled, every pass launch
 * is bracketed by CUDA events on the handle's stream; totals per kind
 * (0 = apply pass Y = A X, 1 = adjoint pass Z = A^T Y, 2 = other skinny
 * products such as the lift Q U_B) with their algorithmic flops and
 * bytes (2 M N K, 8 (MK + KN + MN)).  Enabling resets the totals. */
rsvd_status rsvd_profile_enable(rsvd_handle* h, int on);
rsvd_status rsvd_profile_read(rsvd_handle* h, int kind, int64_t* launches, double* ms,
                              double* flops, double* bytes);
/* Launch-site trace: when enabled, the device time between consecutive
 * kernel launches (kernel plus any idle gap before it) is accumulated per
 * source launch site; the report is "site count total_ms" lines. */
rsvd_status rsvd_trace_enable(rsvd_handle* h, int on);
rsvd_status rsvd_trace_report(rsvd_handle* h, char* buf, int64_t len);
/* Row-sharding info (1 / 0 for a single-GPU handle). */
rsvd_status rsvd_dist_info(rsvd_handle* h, int* rank, int* nranks);

/* ---------------------------------------------------- sketch.hpp (L1') */
/* gaussian(n, l, rng): n x l i.i.d. N(0,1), column-major fill
 * (reference sketch.hpp:48-59).  ParameterError if n < 1 or l < 1. */
rsvd_status rsvd_gaussian_dev(rsvd_handle* h, int64_t n, int64_t l, rsvd_rng_state* rng,
                              double* out, int64_t ld_out);

/* ------------------------------------------------------ core.hpp (L1) */
/* orthonormalize(M): m x n -> m x n orthonormal Q with range(Q) >= range(M),
 * padded to full width when rank deficient (reference core.hpp:93-105).
 * DimensionError if n > m, NumericError on non-finite input. In == out allowed. */
rsvd_status rsvd_orthonormalize_dev(rsvd_handle* h, int64_t m, int64_t n, const double* in,
                                    int64_t ld_in, double* q, int64_t ld_q);
/* svd_small(M): thin SVD, r = min(m,n) triples, sigma descending, sign rule
 * of reference core.hpp:111-124.  U m x r, s r, V n x r (device). */
rsvd_status rsvd_svd_small_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                               int64_t lda, double* u, int64_t ldu, double* s, double* v,
                               int64_t ldv);
/* evd_symmetric(C): reference core.hpp:130-162 (asymmetry check, |lambda|
 * descending stable order).  U n x n, lambda n (device). */
rsvd_status rsvd_evd_symmetric_dev(rsvd_handle* h, int64_t n, const double* c, int64_t ldc,
                                   double* u, int64_t ldu, double* lambda);
/* solve_ls(G, H): min-norm least squares, cutoff 1e-12 * sigma_max
 * (reference core.hpp:166-177).  G m x n, H m x r, X n x r (device). */
rsvd_status rsvd_solve_ls_dev(rsvd_handle* h, int64_t m, int64_t n, const double* g,
                              int64_t ldg, int64_t r, const double* hm, int64_t ldh, double* x,
                              int64_t ldx);
/* detail::solve_joint_core(g1, h1, g2, h2) (reference singlepass.hpp:84-101),
 * computed by the exactly equivalent Kronecker-diagonalised route. All l x l. */
rsvd_status rsvd_solve_joint_core_dev(rsvd_handle* h, int64_t l, const double* g1,
                                      const double* h1, const double* g2, const double* h2,
                                      double* c);

/* ------------------------------------- diagnostics */
/* singular_values(M): min(m,n) values, descending (reference core.hpp:180-183).
 * NumericError on non-finite input.  s: device. */
rsvd_status rsvd_singular_values_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                     int64_t lda, double* s);
/* spectral_norm(M) (reference core.hpp:188-221): dense SVD when
 * min(m,n) <= 512, else power iteration on M^T M from the reference's LCG
 * start vector (tol 1e-10, NumericError after 5000 steps).  *out: HOST scalar. */
rsvd_status rsvd_spectral_norm_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                   int64_t lda, double* out);
/* computed_range_error(A, Q) = ||A - Q Q^T A||_2 (reference bounds.hpp:107-120):
 * DimensionError if Q has a different row count, NumericError if
 * max|Q^T Q - I| > 1e-8.  A m x n, Q m x l (device); *out: HOST scalar. */
rsvd_status rsvd_computed_range_error_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                          int64_t lda, int64_t l, const double* q, int64_t ldq,
                                          double* out);
/* canonical_sines(X, Y) (reference angles.hpp:42-60): the min(kx, ky)
 * largest singular values of (I - X X^T) Y, ascending, clamped to [0, 1].
 * DimensionError if the row counts differ, NumericError if X or Y is not
 * orthonormal to 1e-8.  X m x kx, Y m x ky, out (device). */
rsvd_status rsvd_canonical_sines_dev(rsvd_handle* h, int64_t m, int64_t kx, const double* x,
                                     int64_t ldx, int64_t ky, const double* y, int64_t ldy,
                                     double* out);
/* run_svd's error report (reference drivers.hpp:145-151) for A ~ U diag(s) V^T
 * (an EVD passes V = U, s = lambda): *rel_fro = ||A - recon||_F / ||A||_F and
 * *rel_spec = ||A - recon||_2 / ||A||_2, the spectral norms by spectral_norm's
 * rules (dense SVD when min(m,n) <= 512, as the reference's
 * singular_values; power iteration above).  A m x n, U m x r, s r, V n x r
 * (device); rel_fro / rel_spec: HOST scalars. */
rsvd_status rsvd_reconstruction_error_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                          int64_t lda, int64_t r, const double* u, int64_t ldu,
                                          const double* s, const double* v, int64_t ldv,
                                          double* rel_fro, double* rel_spec);
rsvd_status rsvd_singular_values_host(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                      int64_t lda, double* s);
rsvd_status rsvd_spectral_norm_host(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                    int64_t lda, double* out);
rsvd_status rsvd_computed_range_error_host(rsvd_handle* h, int64_t m, int64_t n,
                                           const double* a, int64_t lda, int64_t l,
                                           const double* q, int64_t ldq, double* out);
rsvd_status rsvd_canonical_sines_host(rsvd_handle* h, int64_t m, int64_t kx, const double* x,
                                      int64_t ldx, int64_t ky, const double* y, int64_t ldy,
                                      double* out);

/* ----------------------------------- batched trials */
/* The trial loops of the reference's run_bounds / run_angles
 * (drivers.hpp:340-356, 400-431): trial t runs with Rng(seed_base + t)
 * (sketch.hpp:37-39).  Every streaming pass over A is shared by all trials
 * (one pass of width trials * (k + p)); block t of each output is trial t's
 * result.  range_basis_trials: Q m x (trials (k+p)).  rsvd_trials: U m x
 * (trials (k+p)), sigma trials (k+p), V n x (trials (k+p)), each block as
 * rsvd(A, cfg, Rng(seed_base + t)).  range_error_trials: errors[t] =
 * computed_range_error(A, Q_t) (HOST array, single-GPU handle). */
rsvd_status rsvd_range_basis_trials_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                        int64_t lda, int64_t k, int64_t p, int q, int mode,
                                        uint64_t seed_base, int64_t trials, double* q_out,
                                        int64_t ldq);
rsvd_status rsvd_rsvd_trials_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                 int64_t lda, int64_t k, int64_t p, int q, int mode,
                                 uint64_t seed_base, int64_t trials, double* u, int64_t ldu,
                                 double* sigma, double* v, int64_t ldv);
rsvd_status rsvd_range_error_trials_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                        int64_t lda, int64_t k, int64_t p, int q, int mode,
                                        uint64_t seed_base, int64_t trials, double* errors);

/* Host-buffer variants of the kernel-level entry points (the C++ drop-in
 * layer uses these; copies are included). */
rsvd_status rsvd_gaussian_host(rsvd_handle* h, int64_t n, int64_t l, rsvd_rng_state* rng,
                               double* out, int64_t ld_out);
rsvd_status rsvd_orthonormalize_host(rsvd_handle* h, int64_t m, int64_t n, const double* in,
                                     int64_t ld_in, double* q, int64_t ld_q);
rsvd_status rsvd_svd_small_host(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                int64_t lda, double* u, int64_t ldu, double* s, double* v,
                                int64_t ldv);
rsvd_status rsvd_evd_symmetric_host(rsvd_handle* h, int64_t n, const double* c, int64_t ldc,
                                    double* u, int64_t ldu, double* lambda);
rsvd_status rsvd_solve_ls_host(rsvd_handle* h, int64_t m, int64_t n, const double* g,
                               int64_t ldg, int64_t r, const double* hm, int64_t ldh, double* x,
                               int64_t ldx);
rsvd_status rsvd_range_basis_host(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                  int64_t lda, int64_t k, int64_t p, int q, int mode,
                                  rsvd_rng_state* rng, double* q_out, int64_t ldq);

/* -------------------------------------------- streaming passes over A */
/* Y = A X   (A m x n, X n x l, Y m x l): the sketch / power product. */
rsvd_status rsvd_apply_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a, int64_t lda,
                           int64_t l, const double* x, int64_t ldx, double* y, int64_t ldy);
/* Z = A^T Y (A m x n, Y m x l, Z n x l): the adjoint / projection product
 * (B = Q^T A is returned transposed as Z = A^T Q).  Multi-GPU: allreduced. */
rsvd_status rsvd_apply_adjoint_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                   int64_t lda, int64_t l, const double* y, int64_t ldy,
                                   double* z, int64_t ldz);

/* Alg 6's fused pass alone (Y = A Omega_c, W = A^T Psi from one traversal of
 * A; A m x n, Omega_c n x l, Psi m x l): for unit parity tests.
 * panel_rows > 0 issues it in row panels (the streamed launch sequence);
 * macroblock > 0 overrides the macroblock edge (multiple of 64). */
rsvd_status rsvd_debug_dual_pass_dev(rsvd_handle* h, int64_t m, int64_t n, int64_t l,
                                     const double* a, int64_t lda, const double* oc, int64_t ldo,
                                     const double* psi, int64_t ldp, double* y, int64_t ldy,
                                     double* w, int64_t ldw, int64_t panel_rows, int macroblock);

/* The products with A of wide sketches on the INT8 tensor cores (tcgen05
 * kind::i8, Ozaki splitting into `slices` exact 8-bit slices per operand,
 * 8*slices - 2 fractional bits; csrc/ozaki.cu): -1 = the automatic policy,
 * which also follows the RSVD_OZAKI environment variable (default), 0 = off
 * (the FP64 DMMA passes), 3..8 = slices.  7 slices (the automatic choice)
 * are at fp64's own rounding of the product, 8 are below it, 6 are 2^-46 of
 * the row / column maxima. */
rsvd_status rsvd_set_ozaki_slices(rsvd_handle* h, int slices);
/* Which INT8 GEMM kernel runs (process-wide; unit tests): 1 = CTA pair
 * (tcgen05 cta_group::2, the default), 0 = single CTA, -1 = default. */
rsvd_status rsvd_debug_ozaki_kernel(int pair);
/* C = A X (trans = 0: A m x n, X n x l, C m x l) or C = A^T X (trans = 1: X
 * m x l, C n x l) by the sliced INT8 product alone: for unit parity tests. */
rsvd_status rsvd_debug_ozaki_gemm_dev(rsvd_handle* h, int trans, int64_t m, int64_t n,
                                      const double* a, int64_t lda, int64_t l, const double* x,
                                      int64_t ldx, double* c, int64_t ldc, int slices);

/* ------------------------------------------- rangefinder.hpp (L2) */
/* range_basis(A, cfg, rng) (reference rangefinder.hpp:97-105): Q m x (k+p). */
rsvd_status rsvd_range_basis_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a,
                                 int64_t lda, int64_t k, int64_t p, int q, int mode,
                                 rsvd_rng_state* rng, double* q_out, int64_t ldq);

/* --------------------------------------------- factor.hpp (L3) */
/* rsvd(A, cfg, rng) (reference factor.hpp:12-18): full width l = k+p.
 * U m x l, sigma l, V n x l (device pointers). */
rsvd_status rsvd_rsvd_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a, int64_t lda,
                          int64_t k, int64_t p, int q, int mode, rsvd_rng_state* rng, double* u,
                          int64_t ldu, double* sigma, double* v, int64_t ldv);
rsvd_status rsvd_rsvd_host(rsvd_handle* h, int64_t m, int64_t n, const double* a, int64_t lda,
                           int64_t k, int64_t p, int q, int mode, rsvd_rng_state* rng, double* u,
                           int64_t ldu, double* sigma, double* v, int64_t ldv);

/* ----------------------------------------- singlepass.hpp (L3) */
/* spevd_hermitian(A, k, p, rng) (reference singlepass.hpp:45-78): one
 * counted pass over A.  U n x k, lambda k (device).  check_symmetry != 0 runs
 * the reference's uncounted asymmetry precondition (singlepass.hpp:49-53). */
rsvd_status rsvd_spevd_dev(rsvd_handle* h, int64_t n, const double* a, int64_t lda, int64_t k,
                           int64_t p, rsvd_rng_state* rng, int check_symmetry, double* u,
                           int64_t ldu, double* lambda);
/* The same on a row shard of a distributed handle: this rank holds rows
 * [row_offset, row_offset + m_local) of the n x n matrix (m_local == n on a
 * single-GPU handle); U m_local x k.  The asymmetry precondition compares the
 * shards' transposed blocks rank to rank (an uncounted validation pass). */
rsvd_status rsvd_spevd_shard_dev(rsvd_handle* h, int64_t m_local, int64_t n, const double* a,
                                 int64_t lda, int64_t k, int64_t p, rsvd_rng_state* rng,
                                 int check_symmetry, double* u, int64_t ldu, double* lambda);
rsvd_status rsvd_spevd_shard_host(rsvd_handle* h, int64_t m_local, int64_t n, const double* a,
                                  int64_t lda, int64_t k, int64_t p, rsvd_rng_state* rng, double* u,
                                  int64_t ldu, double* lambda);
rsvd_status rsvd_spevd_host(rsvd_handle* h, int64_t n, const double* a, int64_t lda, int64_t k,
                            int64_t p, rsvd_rng_state* rng, double* u, int64_t ldu,
                            double* lambda);
/* spsvd_general(A, k, p, rng) (reference singlepass.hpp:109-137): Y_c = A
 * Omega_c and W = A^T Psi formed in ONE traversal of A (counted as one
 * apply, one adjoint, one physical pass).  U m x k, sigma k, V n x k.  The
 * _host variants (this and spevd) stream A up in row panels and compute on
 * each panel as it lands. */
rsvd_status rsvd_spsvd_dev(rsvd_handle* h, int64_t m, int64_t n, const double* a, int64_t lda,
                           int64_t k, int64_t p, rsvd_rng_state* rng, double* u, int64_t ldu,
                           double* sigma, double* v, int64_t ldv);
rsvd_status rsvd_spsvd_host(rsvd_handle* h, int64_t m, int64_t n, const double* a, int64_t lda,
                            int64_t k, int64_t p, rsvd_rng_state* rng, double* u, int64_t ldu,
                            double* sigma, double* v, int64_t ldv);

#ifdef __cplusplus
}
#endif
#endif /* RSVD_B200_H_ */
