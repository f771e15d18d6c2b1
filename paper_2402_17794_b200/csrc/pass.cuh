// Streaming-pass GEMMs (pass.cu).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace rsvdb {
// C (M x N) = P (M x K) * R (K x N)            [Y = A X]
void gemm_nn(Handle& h, const DMat& P, const DMat& R, DMat C, int force_splits = 0);
// C (M x N) = P^T * R,  P (K x M), R (K x N)   [Z = A^T Y, Gram Q^T Y]
void gemm_tn(Handle& h, const DMat& P, const DMat& R, DMat C, int force_splits = 0);
// 2-D column-major fp64 TMA map (dims {rows, cols}, box {box_inner, box_outer},
// 128-byte swizzle) and whether x can be addressed by one (16-byte aligned
// base, even ld).
CUtensorMap make_map(const double* p, int64_t rows, int64_t cols, int64_t ld, int box_inner,
                     int box_outer);
bool tma_ok(const DMat& x);
// x itself when tma_ok, else a copy in an aligned even-ld workspace.
DMat tma_view(Handle& h, const DMat& x);
// Live per-launch timing of a streaming pass (rsvd_profile_enable): CUDA
// events on h.stream around the launch, folded into per-kind totals at the
// call's final synchronization.  Kinds: 0 apply, 1 adjoint, 2 other skinny
// products, 3 the fused Alg-6 pass.
struct ProfScope {
  ProfScope(Handle& h, int kind, double flops, double bytes);
  void end();
  Handle& h;
  Handle::ProfRec rec{};
  unsigned flags = 0;
  bool on = false;
};
}  // namespace rsvdb
