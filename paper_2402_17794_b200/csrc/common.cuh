// Shared plumbing of the B200 rsvd engine: error model, handle, workspace.
//
// Error model mirrors the reference (core.hpp:23-39): internal C++ exceptions
// of three kinds are mapped to rsvd_status at the C-ABI boundary (capi.cu)
// and rethrown as rsvd::DimensionError / ParameterError / NumericError by
// include/rsvd/*.hpp.
#pragma once
#include <cstdlib>
#include <utility>

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "rsvd_b200.h"

namespace rsvdb {

struct Error : std::runtime_error {
  rsvd_status code;
  Error(rsvd_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
// Raised at a call's final check when a speculative (sync-free) branch
// decision turned out to need the robust path: the call is re-run eagerly
// with Handle::robust set (capi.cu).  Never reaches the caller.
struct RetryRobust {};
[[noreturn]] inline void throw_dim(const std::string& m) { throw Error(RSVD_ERR_DIMENSION, m); }
[[noreturn]] inline void throw_param(const std::string& m) { throw Error(RSVD_ERR_PARAMETER, m); }
[[noreturn]] inline void throw_numeric(const std::string& m) { throw Error(RSVD_ERR_NUMERIC, m); }

#define RSVD_CUDA(x)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw ::rsvdb::Error(RSVD_ERR_CUDA, std::string(#x " failed: ") + cudaGetErrorString(e_) + \
                                              " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

#define RSVD_LAUNCH_CHECK() RSVD_CUDA(cudaGetLastError())
// Every kernel launch of the engine goes through this: error check + count
// (rsvd_counters.kernel_launches, reported by bench.py as gpu_launches).
#define RSVD_STR2(x) #x
#define RSVD_STR(x) RSVD_STR2(x)
#define RSVD_LAUNCHED(hh)                                        \
  do {                                                           \
    RSVD_LAUNCH_CHECK();                                         \
    (hh).counters.kernel_launches++;                             \
    if ((hh).trace) ::rsvdb::trace_mark((hh), __FILE__ ":" RSVD_STR(__LINE__)); \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#ifdef __CUDACC__
// Sort key for the rank-by-counting orderings of singular values / |lambda|:
// NaN (a non-finite input that is only reported at the call's end) sorts
// last, so every ordering stays a permutation and no kernel indexes out of
// bounds before the NumericError is raised.
__device__ __forceinline__ double order_key(double x) { return x != x ? -1.0 : x; }
#endif
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Device matrix view (column-major).
struct DMat {
  double* p = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
  DMat() = default;
  DMat(double* ptr, int64_t r, int64_t c, int64_t l) : p(ptr), rows(r), cols(c), ld(l) {}
  double* col(int64_t j) const { return p + j * ld; }
};

// Chunked device arena with a bump allocator.  reset() runs at the start of
// every top-level C-ABI call; every call ends with a stream synchronization, so
// no kernel of the previous call can still be using the memory.  A call that
// outgrows the current chunk gets a new chunk; at the next reset the chunks
// are merged into one allocation of the high-water size.
class Arena {
 public:
  ~Arena();
  void reset();
  void* alloc_bytes(size_t bytes);
  double* alloc(int64_t n) { return static_cast<double*>(alloc_bytes(sizeof(double) * size_t(n))); }
  DMat mat(int64_t r, int64_t c) {
    const int64_t ld = round_up(r < 2 ? 2 : r, 2);  // even ld keeps TMA strides 16B aligned
    return DMat(alloc(ld * c), r, c, ld);
  }
  size_t high_water() const { return high_; }
  // largest request the held chunks can serve without a new cudaMalloc
  size_t remaining() const {
    size_t r = 0;
    for (const auto& c : chunks_) r = c.cap - c.off > r ? c.cap - c.off : r;
    return r;
  }
  // bumped whenever chunk addresses change (captured CUDA graphs hold them)
  uint64_t generation() const { return gen_; }

 private:
  struct Chunk {
    char* p;
    size_t cap, off;
  };
  std::vector<Chunk> chunks_;
  size_t used_total_ = 0, high_ = 0;
  uint64_t gen_ = 0;
};

struct Comm;  // NCCL communicator wrapper (dist.cu)
struct VComm;  // in-process virtual communicator (dist.cu)

// Header of an exact-mode patch list (rng.cu), in pinned mapped memory.
struct PatchHdr {
  uint32_t ready;  // device -> host: count is final
  uint32_t done;   // host -> device: 1 = normals written, 2 = cancelled
  uint64_t count;
  int64_t cap;
};

struct Handle {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // own_stream is non-blocking: a call running on it first waits for the work
  // already queued on the legacy default stream (the caller's inputs, e.g. a
  // framework's default stream), see join_caller_stream()
  cudaEvent_t join_ev = nullptr;
  // host-buffer entry points upload A on copy_stream while the Omega stream is
  // generated on `stream`; the first use of A waits on copy_ev (Problem::ready)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_ev = nullptr, order_ev = nullptr;
  // one event per row panel of a streamed upload (single-pass host entry points)
  std::vector<cudaEvent_t> panel_ev;
  // fused Alg-6 pass macroblock edge override (0 = RSVD_FUSED_MB / default)
  int fused_mb = 0;
  // Ozaki slices of the INT8 tensor-core passes (ozaki.cu): -1 = RSVD_OZAKI
  // environment variable, 0 = off (DMMA passes), 3..8 = slices per operand
  int ozaki_slices = -1;
  // second stream of the INT8 dual pass: the next row panel's exponent scan
  // and slicing (HBM-bound) run beside the current panel's GEMMs (tensor-bound)
  cudaStream_t oz_stream = nullptr;
  cudaEvent_t oz_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // entry, sliced[2], free[2]
  // Robust mode: data-dependent branch decisions (CholeskyQR's pass count
  // after a shifted Cholesky) read the device flag on the host mid-call.
  // Off by default: those decisions are speculated without a host round trip
  // (graph-capturable, no mid-call sync) and a device flag makes the call
  // re-run in robust mode when the speculation was wrong (rare: numerically
  // rank-deficient sketches).
  bool robust = false;
  Arena ws;
  int* d_counters = nullptr;   // split-K tile semaphores (kept zeroed)
  int64_t n_counters = 0;
  int* d_flags = nullptr;      // device status flags (non-finite, breakdown)
  int* h_flags = nullptr;      // pinned mirror
  int sm_count = 148;
  rsvd_counters counters{};
  Comm* comm = nullptr;        // null => single GPU
  // In-process virtual communicator (dist.cu): P ranks = P host threads with
  // P handles on ONE device, sharing one stream; the collectives are
  // fixed-order device reductions (tests of the sharded path without P GPUs)
  VComm* vcomm = nullptr;
  cudaStream_t own_stream_saved = nullptr;  // the handle's own stream while attached
  // Shard descriptor (rsvd_set_shard): global rows and this rank's row offset,
  // so a sharded call needs no row-count exchange (0 = exchange per call)
  int64_t shard_m_global = 0, shard_row_off = 0;
  int rank = 0, nranks = 1;
  // the row-sharded (NCCL) code path: also taken by a one-rank communicator,
  // which runs every exchange of the multi-GPU path on a single device
  bool dist() const { return comm != nullptr || vcomm != nullptr; }
  // Live per-launch timing of the streaming-pass kernels (bench.py roofline):
  // CUDA events recorded on h.stream around every pass launch, folded into
  // per-kind totals at the call's final synchronization.
  bool prof = false;
  struct ProfRec {
    cudaEvent_t a, b;
    int kind;  // 0 = NN (Y = A X), 1 = TN (Z = A^T Y), 2 = other, 3 = Alg-6 dual pass, 4 = INT8 slice GEMM
    double flops, bytes;
    bool graph = false;  // events owned by a captured graph (not pooled)
  };
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> prof_pool;
  double prof_ms[5] = {0, 0, 0, 0, 0}, prof_flops[5] = {0, 0, 0, 0, 0}, prof_bytes[5] = {0, 0, 0, 0, 0};
  int64_t prof_count[5] = {0, 0, 0, 0, 0};
  // Launch-site trace (rsvd_trace_enable): an event after every launch; the
  // time between consecutive events (kernel + any idle gap before it) is
  // charged to the launch site at the call's final synchronization.
  bool trace = false;
  std::vector<std::pair<const char*, cudaEvent_t>> trace_ev;
  std::vector<cudaEvent_t> trace_pool;
  std::vector<std::pair<std::string, std::pair<int64_t, double>>> trace_acc;
  // MT19937-64 jump polynomials on the device (rng.cu / mtjump.cpp)
  uint64_t* d_jump = nullptr;
  uint64_t jump_L = 0;
  int jump_count = 0;
  // pinned staging for the RNG state copy-back (rng.cu)
  void* h_rng = nullptr;
  rsvd_rng_state* rng_user_out = nullptr;
  // pinned staging for the RNG state upload (the graph-captured H2D source)
  rsvd_rng_state* h_rng_in = nullptr;
  // Exact Omega/Psi stream (rng.cu): pinned, device-mapped chunks holding the
  // near-midpoint polar inputs whose log the host evaluates; bump-allocated per
  // top-level call (cursor reset with the workspace), never freed before the
  // handle (captured graphs keep pointers into them).
  std::vector<std::pair<char*, size_t>> patch_chunks;
  size_t patch_chunk = 0, patch_off = 0;
  std::vector<PatchHdr*> patch_pending;  // lists of this call, queue order
  // pinned staging for the per-trial seeded states of batched trials (trials.cu)
  rsvd_rng_state* h_rng_batch = nullptr;
  int64_t h_rng_batch_cap = 0;
  // CUDA-graph replay of repeated top-level device calls (capi.cu): a call
  // is captured on its second occurrence (same shapes, pointers and
  // host-visible RNG state) and replayed as one graph launch afterwards.
  // `generation` is bumped whenever a buffer a graph may hold is reallocated
  // (split-K semaphores, jump polynomials; the arena keeps its own count).
  bool graphs = true;
  // Pass configuration for l > 64: 0 = two 4-warp CTAs per SM (default),
  // 1 = one 8-warp CTA per SM.  Alg 5's single pass keeps the latter: its
  // Ritz values sit at the 1e-10 parity tolerance under u-level rounding
  // changes of the sketch, and that summation order is
  // the one measured inside it on C4.
  int pass_cfg_big = 0;
  uint64_t generation = 0;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    uint64_t gen = 0;
    rsvd_counters delta{};
    std::vector<ProfRec> prof;  // pass-timing events recorded inside the graph
    int seen = 0;
    bool bad = false;  // not capturable (host synchronization inside the call)
    std::vector<DMat> stage;  // output staging the graph writes (copied out per call)
    std::vector<PatchHdr*> patch;  // exact-mode lists the graph waits on (re-armed per launch)
  };
  // output staging of the current graph-cached call (see capi.cu guard_graph)
  std::vector<DMat> stage;
  std::unordered_map<std::string, GraphEntry> graph_cache;
};

// Programmatic dependent launch (PDL).  Every engine kernel starts with
// RSVD_PDL_ENTRY(): griddepcontrol.wait (returns once the previous kernel in
// the stream has completed and its writes are visible -- a no-op for a kernel
// not launched as a dependent), then griddepcontrol.launch_dependents (the
// next kernel's CTAs may now be scheduled and wait at their own entry).  With
// the wait first in every kernel the stream order is unchanged; what overlaps
// is the next kernel's launch and CTA rasterization with this kernel's run --
// the inter-kernel gap of the latency-bound small-matrix chains.
#ifdef __CUDACC__
#define RSVD_PDL_ENTRY()                                   \
  do {                                                     \
    asm volatile("griddepcontrol.wait;" ::: "memory");     \
    asm volatile("griddepcontrol.launch_dependents;" :::); \
  } while (0)
#endif

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RSVD_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

#ifdef __CUDACC__
// Every non-cooperative engine launch: on the handle's stream, as a
// programmatic dependent of the previous kernel (RSVD_PDL=0: plain launch).
template <typename... KArgs, typename... Args>
inline void launch_k(Handle& h, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  RSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}
#endif

// End of a top-level call: synchronize, raise NumericError on device flags,
// copy back a pending RNG state.
void finish_call(Handle& h, const char* what);

void trace_mark(Handle& h, const char* site);
void trace_begin(Handle& h);
void trace_collect(Handle& h);

// Answer / cancel this call's exact-mode lists (rng.cu); stream_sync services
// them and then synchronizes h.stream -- every mid-call host wait goes
// through it (a plain synchronize would wait on a kernel that waits on us).
void patch_service(Handle& h);
void patch_cancel(Handle& h);
void stream_sync(Handle& h);

// Opt `kernel` into `bytes` of dynamic shared memory on the CURRENT device.
// The attribute belongs to the device context, so it is tracked per
// (device, kernel) -- a process with handles on several GPUs sets it on each
// (thread-safe; capi.cu).
void smem_attr_raw(const void* kernel, size_t bytes);
template <class K>
inline void smem_attr(K* kernel, size_t bytes) {
  smem_attr_raw(reinterpret_cast<const void*>(kernel), bytes);
}

// Split-K semaphores, at least n of them.
int* tile_counters(Handle& h, int64_t n);

}  // namespace rsvdb
