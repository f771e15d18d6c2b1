// Fused single pass of Alg 6: Y = A Omega_c and W = A^T Psi from one
// traversal of A (fused.cu).
#pragma once
#include "common.cuh"

namespace rsvdb {
// Macroblock edge (RSVD_FUSED_MB, default 2048): row panels passed to
// fused_dual_pass must start at multiples of it.
int fused_macroblock(const Handle& h);
// Tile semaphores fused_dual_pass needs for an M x K matrix and L columns.
int64_t fused_semaphores(int64_t M, int64_t K, int64_t L);
// Rows [row0, row_end) of A (M x K): Y rows of the panel = A Omega_c; W +=
// A_panel^T Psi_panel (in panel order).  `first` resets the semaphores and
// starts W; panels must be issued in increasing row order on h.stream.
void fused_dual_pass(Handle& h, const DMat& A, const DMat& Oc, const DMat& Psi, DMat Y, DMat W,
                     int64_t row0, int64_t row_end, int* sem, bool first);
}  // namespace rsvdb
