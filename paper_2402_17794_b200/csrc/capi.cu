// extern "C" boundary (include/rsvd_b200.h).  Every entry point: select the
// handle's device, reset the per-call workspace, run the device pipeline on the
// handle's stream, synchronize once, map internal errors to rsvd_status.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include "diag.cuh"
#include "trials.cuh"
#include "dist.cuh"
#include "engine.cuh"
#include "fused.cuh"
#include "ozaki.cuh"
#include "pass.cuh"
#include "rng.cuh"
#include "small.cuh"

struct rsvd_handle {
  rsvdb::Handle h;
};

namespace rsvdb {
void smem_attr_raw(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set;
  int dev = 0;
  RSVD_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set[{dev, kernel}];
  // (static shared memory counts toward the 48 KB default too: always opt in)
  if (bytes > cur || cur == 0) {
    RSVD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    cur = std::max<size_t>(bytes, 1);
  }
}
}  // namespace rsvdb

namespace {
thread_local std::string g_err;

// A call on the handle's own (non-blocking) stream must not start before the
// work the caller queued on the legacy default stream -- the kernels that
// produced its inputs (a framework's default stream) -- has finished: the
// non-blocking stream does not synchronize with it implicitly.  Measured
// without this: the inputs of a call issued right after a framework's
// asynchronous input construction were read before they were complete.
void join_caller_stream(rsvdb::Handle& h) {
  if (h.stream != h.own_stream) return;  // caller's stream: ordered already
  RSVD_CUDA(cudaEventRecord(h.join_ev, cudaStreamLegacy));
  RSVD_CUDA(cudaStreamWaitEvent(h.own_stream, h.join_ev, 0));
}

// One eager run of a call's pipeline: f, then the final check.  A wrong
// speculation (RetryRobust from the final check) re-runs f once in robust
// mode -- from the caller's unchanged inputs and RNG state, the counters of
// the first attempt rolled back; every rank of a distributed handle sees the
// same (replicated) flag, so all ranks retry together.
template <class F>
void run_eager(rsvdb::Handle& h, const char* what, F&& f) {
  const rsvd_counters before = h.counters;
  for (int attempt = 0;; ++attempt) {
    h.ws.reset();
    h.patch_chunk = h.patch_off = 0;
    join_caller_stream(h);
    h.rng_user_out = nullptr;
    rsvdb::trace_begin(h);
    try {
      try {
        f(h);
      } catch (const rsvdb::RetryRobust&) {
        throw;
      } catch (...) {
        // a rank failing inside the pipeline releases peers blocked in a
        // virtual collective; errors of the final check (finish_call) are
        // raised by every rank alike and leave the communicator usable
        rsvdb::vcomm_fail(h);
        throw;
      }
      rsvdb::finish_call(h, what);
      h.robust = false;
      return;
    } catch (const rsvdb::RetryRobust&) {
      rsvdb::patch_cancel(h);
      RSVD_CUDA(cudaStreamSynchronize(h.stream));
      h.counters = before;
      h.counters.robust_reruns++;
      if (attempt > 0 || h.robust) {
        h.robust = false;
        throw rsvdb::Error(RSVD_ERR_INTERNAL, std::string(what) + ": robust re-run asked to retry");
      }
      h.robust = true;
    } catch (...) {
      h.robust = false;
      throw;
    }
  }
}

template <class F>
rsvd_status guard(rsvd_handle* hd, const char* what, F&& f) {
  try {
    if (!hd) throw rsvdb::Error(RSVD_ERR_PARAMETER, "null handle");
    rsvdb::Handle& h = hd->h;
    RSVD_CUDA(cudaSetDevice(h.device));
    run_eager(h, what, f);
    return RSVD_OK;
  } catch (const rsvdb::Error& e) {
    g_err = e.what();
    cudaGetLastError();  // clear a non-sticky runtime error so the next call starts clean
    if (hd) {
      hd->h.rng_user_out = nullptr;
      rsvdb::patch_cancel(hd->h);
      cudaStreamSynchronize(hd->h.stream);
      if (hd->h.copy_stream) cudaStreamSynchronize(hd->h.copy_stream);
      cudaMemsetAsync(hd->h.d_flags, 0, sizeof(int), hd->h.stream);
    }
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    if (hd) {
      rsvdb::patch_cancel(hd->h);
      cudaStreamSynchronize(hd->h.stream);
    }
    return RSVD_ERR_INTERNAL;
  }
}

// Graph-replayed variant of guard() for the top-level device pipelines.
// `key` identifies everything the host side of the call depends on (entry
// point, shapes, pointers, the RNG's cached-normal flag); `rng` is the caller's
// state, re-staged before every launch.  First occurrence: eager (warms the
// workspace, jump tables, kernel attributes).  Second: captured on the
// handle's stream, instantiated and launched.  Later: one cudaGraphLaunch plus
// the counter deltas recorded at capture.  Calls that synchronize with the
// host mid-way (large-l shift decisions) fail to capture and stay eager.
// Disabled with RSVD_GRAPHS=0, under profiling/tracing, and with NCCL.
// A device output of a graph-cached call: the graph writes a staging buffer
// in the workspace (stable across replays), copied to the caller's pointer
// after every launch -- so the cache key does not depend on where the caller
// put this call's outputs (fresh output tensors every call would otherwise
// miss the cache and re-capture).
struct OutBuf {
  double* user;
  int64_t rows, cols, ld;
};

// (rows x cols) view of a staging buffer allocated with >= 1 row / column
rsvdb::DMat sub_view(const rsvdb::DMat& st, int64_t rows, int64_t cols) {
  return rsvdb::DMat(st.p, rows, cols, st.ld);
}

void stage_alloc(rsvdb::Handle& h, const std::vector<OutBuf>& outs) {
  h.stage.clear();
  for (const OutBuf& o : outs) h.stage.push_back(h.ws.mat(std::max<int64_t>(o.rows, 1), std::max<int64_t>(o.cols, 1)));
}

void stage_copy_out(rsvdb::Handle& h, const std::vector<rsvdb::DMat>& st, const std::vector<OutBuf>& outs) {
  for (size_t i = 0; i < outs.size(); ++i) {
    const OutBuf& o = outs[i];
    if (o.rows <= 0 || o.cols <= 0 || !o.user) continue;
    RSVD_CUDA(cudaMemcpy2DAsync(o.user, size_t(o.ld) * 8, st[i].p, size_t(st[i].ld) * 8, size_t(o.rows) * 8,
                                size_t(o.cols), cudaMemcpyDeviceToDevice, h.stream));
  }
}

template <class F>
rsvd_status guard_graph(rsvd_handle* hd, const char* what, const std::string& key,
                        rsvd_rng_state* rng, F&& f, const std::vector<OutBuf>& outs = {}) {
  // eager form: outputs through the same staging as the graph
  auto check_outs = [&] {
    for (const OutBuf& o : outs)
      if (o.rows > 0 && o.cols > 0 && o.ld < o.rows)
        throw rsvdb::Error(RSVD_ERR_DIMENSION, "leading dimension < rows");
  };
  auto eager = [&](rsvdb::Handle& h) {
    check_outs();
    stage_alloc(h, outs);
    f(h);
    stage_copy_out(h, h.stage, outs);
  };
  static const bool env_on = [] {
    const char* e = std::getenv("RSVD_GRAPHS");
    return !(e && e[0] == '0');
  }();
  // (NCCL-sharded handles are captured too -- NCCL collectives are
  // graph-capturable; the virtual communicator's host barriers are not)
  if (!hd || !env_on || !hd->h.graphs || hd->h.trace || hd->h.vcomm) return guard(hd, what, eager);
  rsvdb::Handle& h = hd->h;
  auto add = [](rsvd_counters& a, const rsvd_counters& d, int sgn) {
    a.apply += sgn * d.apply;
    a.adjoint += sgn * d.adjoint;
    a.physical_passes += sgn * d.physical_passes;
    a.kernel_launches += sgn * d.kernel_launches;
    a.robust_reruns += sgn * d.robust_reruns;
  };
  try {
    RSVD_CUDA(cudaSetDevice(h.device));
    check_outs();
    join_caller_stream(h);  // before any replay or capture on the stream
    auto gen_now = [&] { return h.generation + h.ws.generation(); };
    if (h.graph_cache.size() > 256 && !h.graph_cache.count(key)) {  // bound the cache
      for (auto& kv : h.graph_cache) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        for (auto& r : kv.second.prof) {
          cudaEventDestroy(r.a);
          cudaEventDestroy(r.b);
        }
      }
      h.graph_cache.clear();
    }
    rsvdb::Handle::GraphEntry& e = h.graph_cache[h.prof ? key + "|prof" : key];
    // a replay (or the capturing run) whose speculation was wrong: undo its
    // counters and re-run the call eagerly in robust mode
    auto robust_rerun = [&](const rsvd_counters& before) {
      rsvdb::patch_cancel(h);
      RSVD_CUDA(cudaStreamSynchronize(h.stream));
      h.counters = before;
      h.counters.robust_reruns++;
      h.rng_user_out = nullptr;
      h.prof_pending.clear();
      h.robust = true;
      return guard(hd, what, eager);
    };
    if (e.exec && e.gen == gen_now()) {
      if (rng) std::memcpy(h.h_rng_in, rng, sizeof(rsvd_rng_state));
      for (rsvdb::PatchHdr* ph : e.patch) {  // re-arm the exact-mode lists
        ph->ready = 0;
        ph->done = 0;
      }
      h.patch_pending = e.patch;
      const rsvd_counters before = h.counters;
      RSVD_CUDA(cudaGraphLaunch(e.exec, h.stream));
      stage_copy_out(h, e.stage, outs);
      add(h.counters, e.delta, 1);
      h.prof_pending = e.prof;
      h.rng_user_out = rng;
      try {
        rsvdb::finish_call(h, what);
      } catch (const rsvdb::RetryRobust&) {
        return robust_rerun(before);
      }
      return RSVD_OK;
    }
    if (e.exec) {  // stale: a buffer it references was reallocated
      cudaGraphExecDestroy(e.exec);
      e.exec = nullptr;
      for (auto& r : e.prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
      }
      e.prof.clear();
    }
    if (++e.seen >= 2 && !e.bad) {
      h.ws.reset();
      h.patch_chunk = h.patch_off = 0;
      h.patch_pending.clear();
      h.rng_user_out = nullptr;
      const rsvd_counters before = h.counters;
      const uint64_t g0 = gen_now();
      cudaGraph_t graph = nullptr;
      bool ok = cudaStreamBeginCapture(h.stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      if (ok) {
        try {
          stage_alloc(h, outs);
          f(h);
        } catch (...) {
          ok = false;
        }
        const cudaError_t ce = cudaStreamEndCapture(h.stream, &graph);
        ok = ok && ce == cudaSuccess && graph != nullptr;
      }
      const cudaError_t last = cudaGetLastError();
      const bool same_gen = gen_now() == g0;
      static const bool dbg = std::getenv("RSVD_GRAPH_DEBUG") != nullptr;
      if (dbg)
        std::fprintf(stderr, "graph capture %s: ok=%d same_gen=%d err=%s key=%s\n", what, int(ok),
                     int(same_gen), cudaGetErrorString(last), key.c_str());
      if (ok && same_gen) {
        cudaGraphExec_t exec = nullptr;
        if (cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
          cudaGraphDestroy(graph);
          e.exec = exec;
          e.gen = g0;
          e.delta = h.counters;
          add(e.delta, before, -1);
          for (auto& r : h.prof_pending) r.graph = true;  // the graph keeps these events
          e.prof = h.prof_pending;
          e.stage = h.stage;
          e.patch = h.patch_pending;  // armed at capture, serviced by finish_call
          RSVD_CUDA(cudaGraphLaunch(e.exec, h.stream));
          stage_copy_out(h, e.stage, outs);
          h.rng_user_out = rng;
          try {
            rsvdb::finish_call(h, what);
          } catch (const rsvdb::RetryRobust&) {
            return robust_rerun(before);
          }
          return RSVD_OK;
        }
        cudaGetLastError();
      }
      if (graph) cudaGraphDestroy(graph);
      h.patch_pending.clear();  // nothing of the failed capture ran
      h.counters = before;
      for (auto& r : h.prof_pending) {  // events of the failed capture back to the pool
        h.prof_pool.push_back(r.a);
        h.prof_pool.push_back(r.b);
      }
      h.prof_pending.clear();
      if (same_gen) e.bad = true;  // genuinely not capturable; a reallocation retries later
    }
  } catch (const rsvdb::Error& err) {
    g_err = err.what();
    cudaGetLastError();
    h.rng_user_out = nullptr;
    rsvdb::patch_cancel(h);
    cudaStreamSynchronize(h.stream);
    cudaMemsetAsync(h.d_flags, 0, sizeof(int), h.stream);
    return err.code;
  }
  return guard(hd, what, eager);
}

std::string graph_key(const char* fn, std::initializer_list<int64_t> v) {
  std::string k(fn);
  char buf[24];
  for (int64_t x : v) {
    std::snprintf(buf, sizeof buf, "|%llx", static_cast<unsigned long long>(x));
    k += buf;
  }
  return k;
}
int64_t pv(const void* p) { return static_cast<int64_t>(reinterpret_cast<uintptr_t>(p)); }

rsvdb::DMat dm(const double* p, int64_t r, int64_t c, int64_t ld) {
  if (r < 0 || c < 0) throw rsvdb::Error(RSVD_ERR_DIMENSION, "negative dimension");
  if (r > 0 && c > 0 && ld < r) throw rsvdb::Error(RSVD_ERR_DIMENSION, "leading dimension < rows");
  return rsvdb::DMat(const_cast<double*>(p), r, c, ld);
}

rsvd_status create_impl(rsvd_handle** out, int device, int rank, int nranks, const void* id) {
  try {
    if (!out) throw rsvdb::Error(RSVD_ERR_PARAMETER, "null output handle");
    auto* hd = new rsvd_handle;
    rsvdb::Handle& h = hd->h;
    h.device = device;
    RSVD_CUDA(cudaSetDevice(device));
    RSVD_CUDA(cudaStreamCreateWithFlags(&h.own_stream, cudaStreamNonBlocking));
    h.stream = h.own_stream;
    RSVD_CUDA(cudaEventCreateWithFlags(&h.join_ev, cudaEventDisableTiming));
    RSVD_CUDA(cudaStreamCreateWithFlags(&h.copy_stream, cudaStreamNonBlocking));
    RSVD_CUDA(cudaEventCreateWithFlags(&h.copy_ev, cudaEventDisableTiming));
    RSVD_CUDA(cudaEventCreateWithFlags(&h.order_ev, cudaEventDisableTiming));
    RSVD_CUDA(cudaMalloc(&h.d_flags, 64));
    RSVD_CUDA(cudaMemset(h.d_flags, 0, 64));
    RSVD_CUDA(cudaMallocHost(&h.h_flags, 64));
    RSVD_CUDA(cudaMallocHost(&h.h_rng, sizeof(rsvd_rng_state)));
    RSVD_CUDA(cudaMallocHost(&h.h_rng_in, sizeof(rsvd_rng_state)));
    RSVD_CUDA(cudaDeviceGetAttribute(&h.sm_count, cudaDevAttrMultiProcessorCount, device));
    rsvdb::rng_init_device(h);
    rsvdb::comm_create(h, rank, nranks, id);
    *out = hd;
    return RSVD_OK;
  } catch (const rsvdb::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RSVD_ERR_INTERNAL;
  }
}

// Host-buffer wrapper: upload A, run, download outputs (the e2e path).
struct HostIO {
  rsvdb::Handle& h;
  rsvdb::DMat up(const double* a, int64_t r, int64_t c, int64_t ld) {
    rsvdb::DMat d = h.ws.mat(r, c);
    if (r * c > 0)
      RSVD_CUDA(cudaMemcpy2DAsync(d.p, d.ld * 8, a, ld * 8, r * 8, c, cudaMemcpyHostToDevice,
                                  h.stream));
    return d;
  }
  // A's upload on the copy stream, overlapping the call's first kernels (the
  // Omega stream): the returned event is waited on before A is first read
  rsvdb::DMat up_overlapped(const double* a, int64_t r, int64_t c, int64_t ld, cudaEvent_t* ready) {
    rsvdb::DMat d = h.ws.mat(r, c);
    *ready = nullptr;
    if (r * c > 0) {
      RSVD_CUDA(cudaEventRecord(h.order_ev, h.stream));  // after this call's earlier work
      RSVD_CUDA(cudaStreamWaitEvent(h.copy_stream, h.order_ev, 0));
      RSVD_CUDA(cudaMemcpy2DAsync(d.p, d.ld * 8, a, ld * 8, r * 8, c, cudaMemcpyHostToDevice,
                                  h.copy_stream));
      RSVD_CUDA(cudaEventRecord(h.copy_ev, h.copy_stream));
      *ready = h.copy_ev;
    }
    return d;
  }
  // A's upload in row panels on the copy stream, one event per panel, so the
  // single-pass algorithms compute on panel i while panel i+1 is in flight
  // (the panels' starts are multiples of the fused pass's macroblock edge).
  rsvdb::DMat up_panels(const double* a, int64_t r, int64_t c, int64_t ld,
                        std::vector<rsvdb::Problem::Panel>* panels) {
    rsvdb::DMat d = h.ws.mat(r, c);
    panels->clear();
    if (r * c == 0) return d;
    const int64_t mb = rsvdb::fused_macroblock(h);
    // ~24 panels (the last panel's compute is the exposed tail), >= 64 MB each
    int64_t rows = std::max<int64_t>(rsvdb::ceil_div(r, 24), (int64_t(64) << 20) / (8 * c));
    rows = std::max<int64_t>(mb, rsvdb::ceil_div(rows, mb) * mb);
    const int64_t np = rsvdb::ceil_div(r, rows);
    while (int64_t(h.panel_ev.size()) < np) {
      cudaEvent_t e;
      RSVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h.panel_ev.push_back(e);
    }
    RSVD_CUDA(cudaEventRecord(h.order_ev, h.stream));  // after this call's earlier work
    RSVD_CUDA(cudaStreamWaitEvent(h.copy_stream, h.order_ev, 0));
    for (int64_t i = 0; i < np; ++i) {
      const int64_t r0 = i * rows, r1 = std::min(r, r0 + rows);
      RSVD_CUDA(cudaMemcpy2DAsync(d.p + r0, d.ld * 8, a + r0, ld * 8, (r1 - r0) * 8, c,
                                  cudaMemcpyHostToDevice, h.copy_stream));
      RSVD_CUDA(cudaEventRecord(h.panel_ev[i], h.copy_stream));
      panels->push_back({r0, r1, h.panel_ev[i]});
    }
    return d;
  }
  void down(const rsvdb::DMat& d, double* a, int64_t ld) {
    if (d.rows * d.cols > 0)
      RSVD_CUDA(cudaMemcpy2DAsync(a, ld * 8, d.p, d.ld * 8, d.rows * 8, d.cols,
                                  cudaMemcpyDeviceToHost, h.stream));
  }
  void down_vec(const double* d, double* a, int64_t n) {
    if (n > 0) RSVD_CUDA(cudaMemcpyAsync(a, d, size_t(n) * 8, cudaMemcpyDeviceToHost, h.stream));
  }
};

}  // namespace

extern "C" {

const char* rsvd_last_error(void) { return g_err.c_str(); }
const char* rsvd_version(void) { return "rsvd-b200 0.1.0 (reference rsvd 0.1.0 API)"; }

rsvd_status rsvd_create(rsvd_handle** h, int device) {
  return create_impl(h, device, 0, 1, nullptr);
}

rsvd_status rsvd_nccl_unique_id(void* out128) {
  try {
    rsvdb::nccl_unique_id(out128);
    return RSVD_OK;
  } catch (const rsvdb::Error& e) {
    g_err = e.what();
    return e.code;
  }
}

struct rsvd_vcomm {
  rsvdb::VComm* v;
};

rsvd_status rsvd_vcomm_create(rsvd_vcomm** out, int nranks) {
  try {
    if (!out) throw rsvdb::Error(RSVD_ERR_PARAMETER, "null output");
    *out = new rsvd_vcomm{rsvdb::vcomm_create(nranks)};
    return RSVD_OK;
  } catch (const rsvdb::Error& e) {
    g_err = e.what();
    return e.code;
  }
}

void rsvd_vcomm_destroy(rsvd_vcomm* vc) {
  if (!vc) return;
  rsvdb::vcomm_destroy(vc->v);
  delete vc;
}

rsvd_status rsvd_create_virtual(rsvd_handle** h, int device, int rank, rsvd_vcomm* vc) {
  if (!vc) {
    g_err = "rsvd_create_virtual: null communicator";
    return RSVD_ERR_PARAMETER;
  }
  const rsvd_status st = create_impl(h, device, 0, 1, nullptr);
  if (st != RSVD_OK) return st;
  try {
    rsvdb::vcomm_attach((*h)->h, vc->v, rank);
    return RSVD_OK;
  } catch (const rsvdb::Error& e) {
    g_err = e.what();
    rsvd_destroy(*h);
    *h = nullptr;
    return e.code;
  }
}

rsvd_status rsvd_set_shard(rsvd_handle* hd, int64_t m_global, int64_t row_offset) {
  if (!hd || m_global < 0 || row_offset < 0) return RSVD_ERR_PARAMETER;
  hd->h.shard_m_global = m_global;
  hd->h.shard_row_off = row_offset;
  return RSVD_OK;
}

rsvd_status rsvd_create_dist(rsvd_handle** h, int device, int rank, int nranks,
                             const void* nccl_id128) {
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    g_err = "rsvd_create_dist: bad rank/nranks";
    return RSVD_ERR_PARAMETER;
  }
  if (nranks > 1 && !nccl_id128) {
    g_err = "rsvd_create_dist: null NCCL id";
    return RSVD_ERR_PARAMETER;
  }
  return create_impl(h, device, rank, nranks, nccl_id128);
}

void rsvd_destroy(rsvd_handle* hd) {
  if (!hd) return;
  rsvdb::Handle& h = hd->h;
  cudaSetDevice(h.device);
  rsvdb::patch_cancel(h);
  if (h.vcomm) h.own_stream = h.own_stream_saved;  // the shared stream belongs to the communicator
  cudaStreamSynchronize(h.stream);
  rsvdb::comm_destroy(h);
  if (h.d_counters) cudaFree(h.d_counters);
  if (h.d_jump) cudaFree(h.d_jump);
  if (h.d_flags) cudaFree(h.d_flags);
  if (h.h_flags) cudaFreeHost(h.h_flags);
  if (h.h_rng) cudaFreeHost(h.h_rng);
  if (h.h_rng_in) cudaFreeHost(h.h_rng_in);
  if (h.h_rng_batch) cudaFreeHost(h.h_rng_batch);
  for (auto& c : h.patch_chunks) cudaFreeHost(c.first);
  for (auto& kv : h.graph_cache) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto& r : kv.second.prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  }
  for (auto e : h.prof_pool) cudaEventDestroy(e);
  for (auto e : h.trace_pool) cudaEventDestroy(e);
  if (h.join_ev) cudaEventDestroy(h.join_ev);
  if (h.copy_stream) {
    cudaStreamSynchronize(h.copy_stream);
    cudaStreamDestroy(h.copy_stream);
  }
  if (h.copy_ev) cudaEventDestroy(h.copy_ev);
  if (h.oz_stream) {
    cudaStreamSynchronize(h.oz_stream);
    cudaStreamDestroy(h.oz_stream);
  }
  for (cudaEvent_t e : h.oz_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h.panel_ev) cudaEventDestroy(e);
  if (h.order_ev) cudaEventDestroy(h.order_ev);
  if (h.own_stream) cudaStreamDestroy(h.own_stream);
  delete hd;
}

rsvd_status rsvd_set_stream(rsvd_handle* hd, void* s) {
  if (!hd) return RSVD_ERR_PARAMETER;
  if (hd->h.vcomm) return RSVD_OK;  // virtual ranks share the communicator's stream
  hd->h.stream = s ? static_cast<cudaStream_t>(s) : hd->h.own_stream;
  return RSVD_OK;
}

rsvd_status rsvd_synchronize(rsvd_handle* hd) {
  if (!hd) return RSVD_ERR_PARAMETER;
  return cudaStreamSynchronize(hd->h.stream) == cudaSuccess ? RSVD_OK : RSVD_ERR_CUDA;
}

rsvd_status rsvd_get_counters(rsvd_handle* hd, rsvd_counters* out) {
  if (!hd || !out) return RSVD_ERR_PARAMETER;
  *out = hd->h.counters;
  return RSVD_OK;
}

rsvd_status rsvd_reset_counters(rsvd_handle* hd) {
  if (!hd) return RSVD_ERR_PARAMETER;
  hd->h.counters = rsvd_counters{};
  return RSVD_OK;
}

rsvd_status rsvd_profile_enable(rsvd_handle* hd, int on) {
  if (!hd) return RSVD_ERR_PARAMETER;
  rsvdb::Handle& h = hd->h;
  h.prof = on != 0;
  for (int k = 0; k < 5; ++k) {
    h.prof_ms[k] = h.prof_flops[k] = h.prof_bytes[k] = 0;
    h.prof_count[k] = 0;
  }
  return RSVD_OK;
}

rsvd_status rsvd_profile_read(rsvd_handle* hd, int kind, int64_t* launches, double* ms,
                              double* flops, double* bytes) {
  if (!hd || kind < 0 || kind > 4) return RSVD_ERR_PARAMETER;
  rsvdb::Handle& h = hd->h;
  if (launches) *launches = h.prof_count[kind];
  if (ms) *ms = h.prof_ms[kind];
  if (flops) *flops = h.prof_flops[kind];
  if (bytes) *bytes = h.prof_bytes[kind];
  return RSVD_OK;
}

rsvd_status rsvd_trace_enable(rsvd_handle* hd, int on) {
  if (!hd) return RSVD_ERR_PARAMETER;
  hd->h.trace = on != 0;
  hd->h.trace_acc.clear();
  return RSVD_OK;
}

rsvd_status rsvd_trace_report(rsvd_handle* hd, char* buf, int64_t len) {
  if (!hd || !buf || len < 1) return RSVD_ERR_PARAMETER;
  std::string out;
  for (auto& kv : hd->h.trace_acc) {
    const char* site = kv.first.c_str();
    const char* slash = std::strrchr(site, '/');
    out += std::string(slash ? slash + 1 : site) + " " + std::to_string(kv.second.first) + " " +
           std::to_string(kv.second.second) + "\n";
  }
  std::strncpy(buf, out.c_str(), size_t(len - 1));
  buf[len - 1] = 0;
  return RSVD_OK;
}

rsvd_status rsvd_dist_info(rsvd_handle* hd, int* rank, int* nranks) {
  if (!hd) return RSVD_ERR_PARAMETER;
  if (rank) *rank = hd->h.rank;
  if (nranks) *nranks = hd->h.nranks;
  return RSVD_OK;
}

rsvd_status rsvd_gaussian_dev(rsvd_handle* hd, int64_t n, int64_t l, rsvd_rng_state* rng,
                              double* out, int64_t ld) {
  return guard(hd, "gaussian", [&](rsvdb::Handle& h) {
    if (n < 1 || l < 1) rsvdb::throw_param("gaussian: dimensions must be positive");
    if (!rng) rsvdb::throw_param("gaussian: null rng");
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::gaussian_dev(h, n, l, r, dm(out, n, l, ld));
    rsvdb::rng_download(h, r, rng);
  });
}

rsvd_status rsvd_orthonormalize_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* in,
                                    int64_t ld_in, double* q, int64_t ld_q) {
  return guard(hd, "orthonormalize", [&](rsvdb::Handle& h) {
    rsvdb::orthonormalize(h, dm(in, m, n, ld_in), dm(q, m, n, ld_q));
  });
}

rsvd_status rsvd_svd_small_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                               int64_t lda, double* u, int64_t ldu, double* s, double* v,
                               int64_t ldv) {
  return guard(hd, "svd_small", [&](rsvdb::Handle& h) {
    const int64_t r = std::min(m, n);
    if (r == 0) return;
    rsvdb::svd_small_impl(h, dm(a, m, n, lda), dm(u, m, r, ldu), s, dm(v, n, r, ldv));
  });
}

rsvd_status rsvd_evd_symmetric_dev(rsvd_handle* hd, int64_t n, const double* c, int64_t ldc,
                                   double* u, int64_t ldu, double* lambda) {
  return guard(hd, "evd_symmetric", [&](rsvdb::Handle& h) {
    if (n == 0) return;
    rsvdb::evd_symmetric_impl(h, dm(c, n, n, ldc), dm(u, n, n, ldu), lambda);
  });
}

rsvd_status rsvd_solve_ls_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* g,
                              int64_t ldg, int64_t r, const double* hm, int64_t ldh, double* x,
                              int64_t ldx) {
  return guard(hd, "solve_ls", [&](rsvdb::Handle& h) {
    if (n == 0 || r == 0) return;
    rsvdb::solve_ls_impl(h, dm(g, m, n, ldg), dm(hm, m, r, ldh), dm(x, n, r, ldx));
  });
}

rsvd_status rsvd_solve_joint_core_dev(rsvd_handle* hd, int64_t l, const double* g1,
                                      const double* h1, const double* g2, const double* h2,
                                      double* c) {
  return guard(hd, "solve_joint_core", [&](rsvdb::Handle& h) {
    if (l < 1) rsvdb::throw_dim("solve_joint_core: l must be >= 1");
    rsvdb::solve_joint_core_impl(h, dm(g1, l, l, l), dm(h1, l, l, l), dm(g2, l, l, l),
                                 dm(h2, l, l, l), dm(c, l, l, l));
  });
}

rsvd_status rsvd_apply_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a, int64_t lda,
                           int64_t l, const double* x, int64_t ldx, double* y, int64_t ldy) {
  return guard(hd, "apply", [&](rsvdb::Handle& h) {
    rsvdb::Problem P;
    P.A = dm(a, m, n, lda);
    rsvdb::op_apply(h, P, dm(x, n, l, ldx), dm(y, m, l, ldy));
  });
}

rsvd_status rsvd_apply_adjoint_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                   int64_t lda, int64_t l, const double* y, int64_t ldy,
                                   double* z, int64_t ldz) {
  return guard(hd, "apply_adjoint", [&](rsvdb::Handle& h) {
    rsvdb::Problem P;
    P.A = dm(a, m, n, lda);
    P.dist = h.dist();
    rsvdb::op_adjoint(h, P, dm(y, m, l, ldy), dm(z, n, l, ldz));
  });
}

rsvd_status rsvd_range_basis_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                 int64_t lda, int64_t k, int64_t p, int q, int mode,
                                 rsvd_rng_state* rng, double* q_out, int64_t ldq) {
  const int64_t lq = std::max<int64_t>(k + p, 0);
  const std::string key = graph_key("range_basis", {m, n, pv(a), lda, k, p, q, mode,
                                                    rng ? rng->has_cached : -1});
  return guard_graph(hd, "range_basis", key, rng, [&](rsvdb::Handle& h) {
    rsvdb::Problem P = rsvdb::make_problem(h, a, m, n, lda);
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::range_basis_impl(h, P, k, p, q, mode, r, sub_view(h.stage[0], m, lq));
    rsvdb::rng_download(h, r, rng);
  }, {{q_out, m, lq, ldq}});
}

rsvd_status rsvd_rsvd_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a, int64_t lda,
                          int64_t k, int64_t p, int q, int mode, rsvd_rng_state* rng, double* u,
                          int64_t ldu, double* sigma, double* v, int64_t ldv) {
  const int64_t l = std::max<int64_t>(k + p, 0);
  const std::string key = graph_key("rsvd", {m, n, pv(a), lda, k, p, q, mode, rng ? rng->has_cached : -1});
  return guard_graph(hd, "rsvd", key, rng, [&](rsvdb::Handle& h) {
    rsvdb::Problem P = rsvdb::make_problem(h, a, m, n, lda);
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::rsvd_impl(h, P, k, p, q, mode, r, sub_view(h.stage[0], m, l), h.stage[1].p,
                     sub_view(h.stage[2], n, l));
    rsvdb::rng_download(h, r, rng);
  }, {{u, m, l, ldu}, {sigma, l, 1, std::max<int64_t>(l, 1)}, {v, n, l, ldv}});
}

rsvd_status rsvd_rsvd_host(rsvd_handle* hd, int64_t m, int64_t n, const double* a, int64_t lda,
                           int64_t k, int64_t p, int q, int mode, rsvd_rng_state* rng, double* u,
                           int64_t ldu, double* sigma, double* v, int64_t ldv) {
  return guard(hd, "rsvd", [&](rsvdb::Handle& h) {
    HostIO io{h};
    cudaEvent_t a_up = nullptr;
    rsvdb::DMat A = io.up_overlapped(a, m, n, lda, &a_up);
    rsvdb::Problem P = rsvdb::make_problem(h, A.p, m, n, A.ld);
    P.ready = a_up;
    const int64_t l = std::max<int64_t>(k + p, 0);
    rsvdb::DMat U = h.ws.mat(m, l), V = h.ws.mat(n, l);
    double* s = h.ws.alloc(std::max<int64_t>(l, 1));
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::rsvd_impl(h, P, k, p, q, mode, r, U, s, V);
    rsvdb::rng_download(h, r, rng);
    io.down(U, u, ldu);
    io.down_vec(s, sigma, l);
    io.down(V, v, ldv);
  });
}

rsvd_status rsvd_spevd_shard_dev(rsvd_handle* hd, int64_t m_local, int64_t n, const double* a,
                                 int64_t lda, int64_t k, int64_t p, rsvd_rng_state* rng,
                                 int check_symmetry, double* u, int64_t ldu, double* lambda) {
  const int64_t kk = std::max<int64_t>(k, 0);
  const std::string key = graph_key("spevd", {m_local, n, pv(a), lda, k, p, check_symmetry,
                                              rng ? rng->has_cached : -1});
  return guard_graph(hd, "spevd_hermitian", key, rng, [&](rsvdb::Handle& h) {
    if (!h.dist() && m_local != n) rsvdb::throw_dim("spevd_hermitian: matrix is not square");
    // squareness of a row shard: m_global == n (checked in spevd_impl)
    rsvdb::Problem P = rsvdb::make_problem(h, a, m_local, n, lda);
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::spevd_impl(h, P, k, p, r, check_symmetry != 0, sub_view(h.stage[0], m_local, kk),
                      h.stage[1].p);
    rsvdb::rng_download(h, r, rng);
  }, {{u, m_local, kk, ldu}, {lambda, kk, 1, std::max<int64_t>(kk, 1)}});
}

rsvd_status rsvd_spevd_dev(rsvd_handle* hd, int64_t n, const double* a, int64_t lda, int64_t k,
                           int64_t p, rsvd_rng_state* rng, int check_symmetry, double* u,
                           int64_t ldu, double* lambda) {
  return rsvd_spevd_shard_dev(hd, n, n, a, lda, k, p, rng, check_symmetry, u, ldu, lambda);
}

rsvd_status rsvd_spevd_shard_host(rsvd_handle* hd, int64_t m_local, int64_t n, const double* a,
                                  int64_t lda, int64_t k, int64_t p, rsvd_rng_state* rng, double* u,
                                  int64_t ldu, double* lambda) {
  return guard(hd, "spevd_hermitian", [&](rsvdb::Handle& h) {
    if (!h.dist() && m_local != n) rsvdb::throw_dim("spevd_hermitian: matrix is not square");
    HostIO io{h};
    std::vector<rsvdb::Problem::Panel> panels;
    rsvdb::DMat A = io.up_panels(a, m_local, n, lda, &panels);
    rsvdb::Problem P = rsvdb::make_problem(h, A.p, m_local, n, A.ld);
    P.panels = panels;
    const int64_t kk = std::max<int64_t>(k, 0);
    rsvdb::DMat U = h.ws.mat(m_local, kk);
    double* lam = h.ws.alloc(std::max<int64_t>(kk, 1));
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::spevd_impl(h, P, k, p, r, true, U, lam);
    rsvdb::rng_download(h, r, rng);
    io.down(U, u, ldu);
    io.down_vec(lam, lambda, kk);
  });
}

rsvd_status rsvd_spevd_host(rsvd_handle* hd, int64_t n, const double* a, int64_t lda, int64_t k,
                            int64_t p, rsvd_rng_state* rng, double* u, int64_t ldu,
                            double* lambda) {
  return rsvd_spevd_shard_host(hd, n, n, a, lda, k, p, rng, u, ldu, lambda);
}

rsvd_status rsvd_spsvd_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a, int64_t lda,
                           int64_t k, int64_t p, rsvd_rng_state* rng, double* u, int64_t ldu,
                           double* sigma, double* v, int64_t ldv) {
  const int64_t kk = std::max<int64_t>(k, 0);
  const std::string key = graph_key("spsvd", {m, n, pv(a), lda, k, p, rng ? rng->has_cached : -1});
  return guard_graph(hd, "spsvd_general", key, rng, [&](rsvdb::Handle& h) {
    rsvdb::Problem P = rsvdb::make_problem(h, a, m, n, lda);
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::spsvd_impl(h, P, k, p, r, sub_view(h.stage[0], m, kk), h.stage[1].p,
                      sub_view(h.stage[2], n, kk));
    rsvdb::rng_download(h, r, rng);
  }, {{u, m, kk, ldu}, {sigma, kk, 1, std::max<int64_t>(kk, 1)}, {v, n, kk, ldv}});
}

rsvd_status rsvd_spsvd_host(rsvd_handle* hd, int64_t m, int64_t n, const double* a, int64_t lda,
                            int64_t k, int64_t p, rsvd_rng_state* rng, double* u, int64_t ldu,
                            double* sigma, double* v, int64_t ldv) {
  return guard(hd, "spsvd_general", [&](rsvdb::Handle& h) {
    HostIO io{h};
    std::vector<rsvdb::Problem::Panel> panels;
    rsvdb::DMat A = io.up_panels(a, m, n, lda, &panels);
    rsvdb::Problem P = rsvdb::make_problem(h, A.p, m, n, A.ld);
    P.panels = panels;
    const int64_t kk = std::max<int64_t>(k, 0);
    rsvdb::DMat U = h.ws.mat(m, kk), V = h.ws.mat(n, kk);
    double* s = h.ws.alloc(std::max<int64_t>(kk, 1));
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::spsvd_impl(h, P, k, p, r, U, s, V);
    rsvdb::rng_download(h, r, rng);
    io.down(U, u, ldu);
    io.down_vec(s, sigma, kk);
    io.down(V, v, ldv);
  });
}

rsvd_status rsvd_debug_dual_pass_dev(rsvd_handle* hd, int64_t m, int64_t n, int64_t l,
                                     const double* a, int64_t lda, const double* oc, int64_t ldo,
                                     const double* psi, int64_t ldp, double* y, int64_t ldy,
                                     double* w, int64_t ldw, int64_t panel_rows, int macroblock) {
  return guard(hd, "dual_pass", [&](rsvdb::Handle& h) {
    struct Mb {  // restored on exceptions too
      rsvdb::Handle& h;
      int old;
      ~Mb() { h.fused_mb = old; }
    } mb_scope{h, h.fused_mb};
    if (macroblock > 0) h.fused_mb = macroblock;
    rsvdb::Problem P;
    P.A = dm(a, m, n, lda);
    P.dist = h.dist();
    P.m_global = m;
    if (panel_rows > 0) {
      const int64_t mb = rsvdb::fused_macroblock(h);
      const int64_t rows = std::max<int64_t>(mb, rsvdb::ceil_div(panel_rows, mb) * mb);
      for (int64_t r0 = 0; r0 < m; r0 += rows) P.panels.push_back({r0, std::min(m, r0 + rows), nullptr});
    }
    rsvdb::op_dual(h, P, dm(oc, n, l, ldo), dm(psi, m, l, ldp), dm(y, m, l, ldy), dm(w, n, l, ldw));
  });
}

rsvd_status rsvd_set_ozaki_slices(rsvd_handle* hd, int slices) {
  return guard(hd, "set_ozaki_slices", [&](rsvdb::Handle& h) {
    if (slices != -1 && slices != 0 && (slices < 3 || slices > 8))
      rsvdb::throw_param("set_ozaki_slices: slices must be -1 (environment), 0 (off) or 3..8");
    h.ozaki_slices = slices;
    h.generation++;  // captured graphs hold the other pass
  });
}

rsvd_status rsvd_debug_ozaki_kernel(int pair) {
  rsvdb::ozaki_force_pair_kernel(pair);
  return RSVD_OK;
}

rsvd_status rsvd_debug_ozaki_gemm_dev(rsvd_handle* hd, int trans, int64_t m, int64_t n,
                                      const double* a, int64_t lda, int64_t l, const double* x,
                                      int64_t ldx, double* c, int64_t ldc, int slices) {
  return guard(hd, "ozaki_gemm", [&](rsvdb::Handle& h) {
    if (trans)
      rsvdb::ozaki_gemm(h, dm(a, m, n, lda), dm(x, m, l, ldx), dm(c, n, l, ldc), true, slices);
    else
      rsvdb::ozaki_gemm(h, dm(a, m, n, lda), dm(x, n, l, ldx), dm(c, m, l, ldc), false, slices);
  });
}

rsvd_status rsvd_gaussian_host(rsvd_handle* hd, int64_t n, int64_t l, rsvd_rng_state* rng,
                               double* out, int64_t ld) {
  return guard(hd, "gaussian", [&](rsvdb::Handle& h) {
    if (n < 1 || l < 1) rsvdb::throw_param("gaussian: dimensions must be positive");
    if (!rng) rsvdb::throw_param("gaussian: null rng");
    HostIO io{h};
    rsvdb::DMat G = h.ws.mat(n, l);
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::gaussian_dev(h, n, l, r, G);
    rsvdb::rng_download(h, r, rng);
    io.down(G, out, ld);
  });
}

rsvd_status rsvd_orthonormalize_host(rsvd_handle* hd, int64_t m, int64_t n, const double* in,
                                     int64_t ld_in, double* q, int64_t ld_q) {
  return guard(hd, "orthonormalize", [&](rsvdb::Handle& h) {
    if (n > m)
      rsvdb::throw_dim("orthonormalize: more columns than rows (" + std::to_string(n) + " > " +
                       std::to_string(m) + ")");
    HostIO io{h};
    rsvdb::DMat X = io.up(in, m, n, ld_in), Q = h.ws.mat(m, n);
    rsvdb::orthonormalize(h, X, Q);
    io.down(Q, q, ld_q);
  });
}

rsvd_status rsvd_svd_small_host(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                int64_t lda, double* u, int64_t ldu, double* s, double* v,
                                int64_t ldv) {
  return guard(hd, "svd_small", [&](rsvdb::Handle& h) {
    const int64_t r = std::min(m, n);
    if (r == 0) return;
    HostIO io{h};
    rsvdb::DMat A = io.up(a, m, n, lda), U = h.ws.mat(m, r), V = h.ws.mat(n, r);
    double* sd = h.ws.alloc(r);
    rsvdb::svd_small_impl(h, A, U, sd, V);
    io.down(U, u, ldu);
    io.down_vec(sd, s, r);
    io.down(V, v, ldv);
  });
}

rsvd_status rsvd_evd_symmetric_host(rsvd_handle* hd, int64_t n, const double* c, int64_t ldc,
                                    double* u, int64_t ldu, double* lambda) {
  return guard(hd, "evd_symmetric", [&](rsvdb::Handle& h) {
    if (n == 0) return;
    HostIO io{h};
    rsvdb::DMat C = io.up(c, n, n, ldc), U = h.ws.mat(n, n);
    double* lam = h.ws.alloc(n);
    rsvdb::evd_symmetric_impl(h, C, U, lam);
    io.down(U, u, ldu);
    io.down_vec(lam, lambda, n);
  });
}

rsvd_status rsvd_solve_ls_host(rsvd_handle* hd, int64_t m, int64_t n, const double* g,
                               int64_t ldg, int64_t r, const double* hm, int64_t ldh, double* x,
                               int64_t ldx) {
  return guard(hd, "solve_ls", [&](rsvdb::Handle& h) {
    if (n == 0 || r == 0) return;
    HostIO io{h};
    rsvdb::DMat G = io.up(g, m, n, ldg), Hm = io.up(hm, m, r, ldh), X = h.ws.mat(n, r);
    rsvdb::solve_ls_impl(h, G, Hm, X);
    io.down(X, x, ldx);
  });
}

rsvd_status rsvd_range_basis_host(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                  int64_t lda, int64_t k, int64_t p, int q, int mode,
                                  rsvd_rng_state* rng, double* q_out, int64_t ldq) {
  const std::string key = graph_key("range_basis", {m, n, pv(a), lda, k, p, q, mode, pv(q_out), ldq,
                                                    rng ? rng->has_cached : -1});
  return guard_graph(hd, "range_basis", key, rng, [&](rsvdb::Handle& h) {
    HostIO io{h};
    rsvdb::DMat A = io.up(a, m, n, lda);
    rsvdb::Problem P = rsvdb::make_problem(h, A.p, m, n, A.ld);
    const int64_t l = std::max<int64_t>(k + p, 0);
    rsvdb::DMat Q = h.ws.mat(m, l);
    rsvdb::DevRng r = rsvdb::rng_upload(h, rng);
    rsvdb::range_basis_impl(h, P, k, p, q, mode, r, Q);
    rsvdb::rng_download(h, r, rng);
    io.down(Q, q_out, ldq);
  });
}

// ------------------------------------------------------------- diagnostics
namespace {
void single_gpu_only(const rsvdb::Handle& h, const char* what) {
  if (h.dist())
    throw rsvdb::Error(RSVD_ERR_PARAMETER, std::string(what) + ": needs a single-GPU handle");
}
}  // namespace

rsvd_status rsvd_singular_values_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                     int64_t lda, double* s) {
  return guard(hd, "singular_values", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "singular_values");
    rsvdb::singular_values_impl(h, dm(a, m, n, lda), s);
  });
}

rsvd_status rsvd_spectral_norm_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                   int64_t lda, double* out) {
  return guard(hd, "spectral_norm", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "spectral_norm");
    *out = rsvdb::spectral_norm_impl(h, dm(a, m, n, lda), nullptr);
  });
}

rsvd_status rsvd_computed_range_error_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                          int64_t lda, int64_t l, const double* q, int64_t ldq,
                                          double* out) {
  return guard(hd, "computed_range_error", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "computed_range_error");
    *out = rsvdb::computed_range_error_impl(h, dm(a, m, n, lda), dm(q, m, l, ldq));
  });
}

rsvd_status rsvd_canonical_sines_dev(rsvd_handle* hd, int64_t m, int64_t kx, const double* x,
                                     int64_t ldx, int64_t ky, const double* y, int64_t ldy,
                                     double* out) {
  return guard(hd, "canonical_sines", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "canonical_sines");
    rsvdb::canonical_sines_impl(h, dm(x, m, kx, ldx), dm(y, m, ky, ldy), out);
  });
}

rsvd_status rsvd_reconstruction_error_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                          int64_t lda, int64_t r, const double* u, int64_t ldu,
                                          const double* s, const double* v, int64_t ldv,
                                          double* rel_fro, double* rel_spec) {
  return guard(hd, "reconstruction_error", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "reconstruction_error");
    rsvdb::reconstruction_error_impl(h, dm(a, m, n, lda), dm(u, m, r, ldu), s, dm(v, n, r, ldv),
                                     rel_fro, rel_spec);
  });
}

rsvd_status rsvd_singular_values_host(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                      int64_t lda, double* s) {
  return guard(hd, "singular_values", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "singular_values");
    const int64_t r = std::min(m, n);
    if (r <= 0) return;
    HostIO io{h};
    rsvdb::DMat A = io.up(a, m, n, lda);
    double* sd = h.ws.alloc(r);
    rsvdb::singular_values_impl(h, A, sd);
    io.down_vec(sd, s, r);
  });
}

rsvd_status rsvd_spectral_norm_host(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                    int64_t lda, double* out) {
  return guard(hd, "spectral_norm", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "spectral_norm");
    HostIO io{h};
    *out = rsvdb::spectral_norm_impl(h, io.up(a, m, n, lda), nullptr);
  });
}

rsvd_status rsvd_computed_range_error_host(rsvd_handle* hd, int64_t m, int64_t n,
                                           const double* a, int64_t lda, int64_t l,
                                           const double* q, int64_t ldq, double* out) {
  return guard(hd, "computed_range_error", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "computed_range_error");
    HostIO io{h};
    rsvdb::DMat A = io.up(a, m, n, lda), Q = io.up(q, m, l, ldq);
    *out = rsvdb::computed_range_error_impl(h, A, Q);
  });
}

rsvd_status rsvd_canonical_sines_host(rsvd_handle* hd, int64_t m, int64_t kx, const double* x,
                                      int64_t ldx, int64_t ky, const double* y, int64_t ldy,
                                      double* out) {
  return guard(hd, "canonical_sines", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "canonical_sines");
    const int64_t cnt = std::min(kx, ky);
    HostIO io{h};
    rsvdb::DMat X = io.up(x, m, kx, ldx), Y = io.up(y, m, ky, ldy);
    double* o = h.ws.alloc(std::max<int64_t>(cnt, 1));
    rsvdb::canonical_sines_impl(h, X, Y, o);
    io.down_vec(o, out, cnt);
  });
}

// ------------------------------------------------------------ batched trials
rsvd_status rsvd_range_basis_trials_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                        int64_t lda, int64_t k, int64_t p, int q, int mode,
                                        uint64_t seed_base, int64_t trials, double* q_out,
                                        int64_t ldq) {
  return guard(hd, "range_basis_trials", [&](rsvdb::Handle& h) {
    rsvdb::Problem P = rsvdb::make_problem(h, a, m, n, lda);
    const int64_t l = std::max<int64_t>(k + p, 0);
    rsvdb::range_basis_trials_impl(h, P, k, p, q, mode, seed_base, trials,
                                   dm(q_out, m, l * std::max<int64_t>(trials, 0), ldq));
  });
}

rsvd_status rsvd_rsvd_trials_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                 int64_t lda, int64_t k, int64_t p, int q, int mode,
                                 uint64_t seed_base, int64_t trials, double* u, int64_t ldu,
                                 double* sigma, double* v, int64_t ldv) {
  return guard(hd, "rsvd_trials", [&](rsvdb::Handle& h) {
    rsvdb::Problem P = rsvdb::make_problem(h, a, m, n, lda);
    const int64_t L = std::max<int64_t>(k + p, 0) * std::max<int64_t>(trials, 0);
    rsvdb::rsvd_trials_impl(h, P, k, p, q, mode, seed_base, trials, dm(u, m, L, ldu), sigma,
                            dm(v, n, L, ldv));
  });
}

rsvd_status rsvd_range_error_trials_dev(rsvd_handle* hd, int64_t m, int64_t n, const double* a,
                                        int64_t lda, int64_t k, int64_t p, int q, int mode,
                                        uint64_t seed_base, int64_t trials, double* errors) {
  return guard(hd, "range_error_trials", [&](rsvdb::Handle& h) {
    single_gpu_only(h, "range_error_trials");
    rsvdb::Problem P = rsvdb::make_problem(h, a, m, n, lda);
    rsvdb::range_error_trials_impl(h, P, k, p, q, mode, seed_base, trials, errors);
  });
}

}  // extern "C"
