// FP64 products of the streaming passes on the INT8 tensor cores (tcgen05,
// TMEM accumulators) by the Ozaki splitting: both operands are cut into S
// signed 8-bit slices (balanced base-256 digits) against a per-row /
// per-column power-of-two scale, the S(S+1)/2 slice products that matter are
// exact int32 GEMMs, and the result is reassembled in fp64 (ozaki.cu).
// Default (S = 7) for wide sketches of large matrices (ozaki_slices_auto,
// ozaki_cache_decide).
#pragma once
#include "common.cuh"

namespace rsvdb {
// Slices per operand: rsvd_set_ozaki_slices, else the RSVD_OZAKI environment
// variable (0 = the DMMA passes, 3..8 = slices), else -1 = automatic.
int ozaki_slices(const Handle& h);
// Which GEMM kernel runs: 1 = the CTA-pair kernel (cta_group::2), 0 = the
// single-CTA kernel, -1 = RSVD_OZ_CG2 / default (pair).  Process-wide; tests.
void ozaki_force_pair_kernel(int pair);
// The dual pass's choice for an A of rows x K and l = L sketch columns: the
// explicit setting, else 7 slices for wide sketches of large matrices, else 0.
int ozaki_slices_auto(const Handle& h, int64_t rows, int64_t K, int64_t L);
// Work buffers of one call (device pointers into the handle's workspace),
// reused by every sub-panel: the arena is a bump allocator and the stream
// orders the reuse.  Lives on the caller's stack for the duration of the call.
struct OzakiState {
  bool have = false;
  int64_t cap = 0;            // sub-panel rows the buffers hold
  unsigned char* xs = nullptr;   // the K-long skinny operand's slices (Omega_c), interleaved
  int* e_x = nullptr;
  // A sub-panel slices: plain [s][K][rows] (apply operand) and interleaved
  // [K][rows/32][s][32] (adjoint operand), with the rows' exponents; two sets
  // when the next sub-panel is sliced beside the current one's GEMMs
  int nbuf = 1;
  int64_t count = 0;             // sub-panels sliced so far (buffer = count % nbuf)
  unsigned char* as[2] = {nullptr, nullptr};
  unsigned char* asi[2] = {nullptr, nullptr};
  int* e_a[2] = {nullptr, nullptr};
  unsigned char* ps = nullptr;   // the row-long skinny operand's slices (Psi'), interleaved
  int* e_p = nullptr;
  double* scratch = nullptr;
};
// Rows [row0, row_end) of A (M x K): Y rows of the panel = A Omega_c; W (+)=
// A_panel^T Psi_panel.  Same contract as fused_dual_pass (fused.cuh): `first`
// starts W, panels arrive in increasing row order on h.stream.  `state` is
// filled by the first panel (Omega_c's slices, the panel buffers).
void ozaki_dual_pass(Handle& h, const DMat& A, const DMat& Oc, const DMat& Psi, DMat Y, DMat W,
                     int64_t row0, int64_t row_end, OzakiState* state, bool first, int slices);
// C = A X (trans = 0; A m x n, X n x l) or C = A^T X (trans = 1; X m x l).
void ozaki_gemm(Handle& h, const DMat& A, const DMat& X, DMat C, bool trans, int slices);

// The range finder's passes (Algs 2-4: Y = A X, Z = A^T Y, repeated 2q+2 times
// over the SAME A) on the INT8 tensor cores: A's slices, in both operand
// layouts, are built once per call and cached here (device pointers into the
// handle's workspace; the Problem of the call owns the struct).
struct OzCache {
  bool decided = false, on = false, built = false;
  int S = 0;
  int64_t cap = 0, nsub = 0, Lcap = 0;  // sub-panel rows, count; columns xs / ps hold
  unsigned char* as = nullptr;   // per sub-panel: plain slices
  unsigned char* asi = nullptr;  // per sub-panel: interleaved slices
  int* e_a = nullptr;            // exponents of all rows
  unsigned char* xs = nullptr;
  unsigned char* ps = nullptr;
  int* e_x = nullptr;
  int* e_p = nullptr;
  double* scratch = nullptr;
};
// Decide once per call whether its passes over A (rows x K, sketch width L,
// `passes` products expected) run on the INT8 path: the explicit setting,
// else 7 slices when A has >= 2^26 entries, both layouts of its slices fit in
// device memory and the sketch is wide enough to amortize the slicing pass
// (L >= 96 for passes >= 3, L >= 160 for a single product).
bool ozaki_cache_decide(Handle& h, OzCache& c, const DMat& A, int64_t L, int passes);
void ozaki_cached_gemm(Handle& h, OzCache& c, const DMat& A, const DMat& X, DMat C, bool trans);
}  // namespace rsvdb
