// Streaming-pass GEMMs (pass.cu).
#pragma once
#include "common.cuh"

namespace rsvdb {
// C (M x N) = P (M x K) * R (K x N)            [Y = A X]
void gemm_nn(Handle& h, const DMat& P, const DMat& R, DMat C, int force_splits = 0);
// C (M x N) = P^T * R,  P (K x M), R (K x N)   [Z = A^T Y, Gram Q^T Y]
void gemm_tn(Handle& h, const DMat& P, const DMat& R, DMat C, int force_splits = 0);
}  // namespace rsvdb
