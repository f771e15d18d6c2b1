// Pipelines (engine.cu).
#pragma once
#include <vector>

#include "common.cuh"
#include "ozaki.cuh"
#include "rng.cuh"

namespace rsvdb {

struct Problem {
  DMat A;              // local row shard (m_local x n)
  int64_t m_global = 0;
  int64_t row_off = 0;
  bool dist = false;
  cudaEvent_t ready = nullptr;  // A's upload (host entry points): waited on before first use
  // Row panels of a streamed upload (host entry points of the single-pass
  // algorithms): rows [row0, row1) are resident once `ready` fires.
  struct Panel {
    int64_t row0, row1;
    cudaEvent_t ready;
  };
  std::vector<Panel> panels;
  // Range-finder passes on the INT8 tensor cores (ozaki.cu): A's slices, built
  // by the first pass of a call and reused by the others; `oz_passes` is the
  // number of products with A the calling algorithm will make (0 = unknown).
  mutable OzCache oz;
  mutable int oz_passes = 0;
};

Problem make_problem(Handle& h, const double* a, int64_t m, int64_t n, int64_t lda);
void op_apply(Handle& h, const Problem& P, const DMat& X, DMat Y);
void op_adjoint(Handle& h, const Problem& P, const DMat& Y, DMat Z);
void op_dual(Handle& h, const Problem& P, const DMat& Oc, const DMat& Psi, DMat Yc, DMat W);
void check_symmetric(Handle& h, const DMat& C, bool dist);

// thin SVD without the sign rule (engine.cu)
void svd_core(Handle& h, const DMat& M, DMat U, double* s, DMat V);
void svd_small_impl(Handle& h, const DMat& M, DMat U, double* s, DMat V);
void solve_ls_impl(Handle& h, const DMat& G, const DMat& Hm, DMat X);
void evd_symmetric_impl(Handle& h, const DMat& C, DMat U, double* lambda);
void solve_joint_core_impl(Handle& h, const DMat& G1, const DMat& H1, const DMat& G2,
                           const DMat& H2, DMat C);
void range_basis_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode,
                      DevRng& rng, DMat Q);
// Stage 2 of rsvd given Q and Z = A^T Q (engine.cu)
void rsvd_stage2(Handle& h, const DMat& Q, const DMat& Z, DMat U, double* sigma, DMat V);
void rsvd_impl(Handle& h, const Problem& P, int64_t k, int64_t p, int q, int mode, DevRng& rng,
               DMat U, double* sigma, DMat V);
void spevd_impl(Handle& h, const Problem& P, int64_t k, int64_t p, DevRng& rng, bool check_sym,
                DMat U, double* lambda);
void spsvd_impl(Handle& h, const Problem& P, int64_t k, int64_t p, DevRng& rng, DMat U,
                double* sigma, DMat V);

}  // namespace rsvdb
