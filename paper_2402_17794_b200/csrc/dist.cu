// Row-sharded multi-GPU plumbing: one process per GPU, NCCL over NVLink /
// NVSwitch.  The reference is single-threaded (README.md:152); the only data
// that crosses GPUs in this engine are the small partial products the
// north_star names: n x l / l x n (A^T Y, Q^T A, A^T Psi), l x l Gram / R /
// inner-product partials, and scalars.  A itself never moves.
//
// Determinism: NCCL_ALGO / NCCL_PROTO can be pinned by the caller (bench.py
// pins Ring/Simple) so reruns are bitwise identical.
//
// Virtual mode (VComm): P ranks in one process on ONE device -- P host threads,
// P handles, one shared stream.  Every collective is a host barrier among the
// rank threads around ONE device kernel issued by rank 0 on the shared stream
// that reads every rank's buffer and writes every rank's result, summing in
// rank order (deterministic).  Because all ranks' work is on one stream, the
// kernel runs after every rank's inputs and before any rank's later work,
// with no events; ranks never run kernels concurrently (no co-residency
// hazards for the cooperative / persistent kernels).  The engine above the
// collectives is the same code the NCCL ranks run.
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "dist.cuh"

namespace rsvdb {

struct Comm {
  ncclComm_t c = nullptr;
};

constexpr int kVMaxRanks = 16;

struct VComm {
  int n = 0;
  int device = -1;
  cudaStream_t stream = nullptr;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const double*> in;
  std::vector<double*> out;
  std::vector<int64_t> val;
  int refs = 0;
  bool failed = false;
  // all ranks arrive; returns false if a rank failed (its thread threw)
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (failed) return false;
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || failed; });
    }
    return !failed;
  }
  void fail() {
    std::lock_guard<std::mutex> lk(m);
    failed = true;
    cv.notify_all();
  }
};

struct VPtrs {
  const double* in[kVMaxRanks];
  double* out[kVMaxRanks];
};

// out_r[i] = sum_{s = 0..n-1} in_s[i] (rank order) for every rank r; op 1: max.
__global__ void vc_reduce_kernel(VPtrs p, int n, int64_t count, int op) {
  RSVD_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    double v = p.in[0][i];
    for (int s = 1; s < n; ++s) v = op ? fmax(v, p.in[s][i]) : v + p.in[s][i];
    for (int r = 0; r < n; ++r) p.out[r][i] = v;
  }
}
// out_r[s * count + i] = in_s[i]
__global__ void vc_gather_kernel(VPtrs p, int n, int64_t count) {
  RSVD_PDL_ENTRY();
  const int64_t tot = count * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int s = int(e / count);
    const double v = p.in[s][e % count];
    for (int r = 0; r < n; ++r) p.out[r][e] = v;
  }
}

namespace {
// One collective: deposit (in, out), barrier, rank 0 launches, barrier.
template <class F>
void vcoll(Handle& h, const double* in, double* out, F&& launch) {
  VComm& v = *h.vcomm;
  v.in[size_t(h.rank)] = in;
  v.out[size_t(h.rank)] = out;
  if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
  if (h.rank == 0) {
    VPtrs p{};
    for (int r = 0; r < v.n; ++r) {
      p.in[r] = v.in[size_t(r)];
      p.out[r] = v.out[size_t(r)];
    }
    launch(p);
  }
  if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
}
int vgrid(const Handle& h, int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 2 * h.sm_count)));
}
}  // namespace

VComm* vcomm_create(int nranks) {
  if (nranks < 1 || nranks > kVMaxRanks) throw_param("virtual communicator: 1..16 ranks");
  auto* v = new VComm;
  v->n = nranks;
  v->in.resize(size_t(nranks));
  v->out.resize(size_t(nranks));
  v->val.resize(size_t(nranks));
  return v;
}

void vcomm_destroy(VComm* v) {
  if (!v) return;
  if (v->stream) cudaStreamDestroy(v->stream);
  delete v;
}

void vcomm_attach(Handle& h, VComm* v, int rank) {
  if (!v || rank < 0 || rank >= v->n) throw_param("virtual communicator: bad rank");
  std::lock_guard<std::mutex> lk(v->m);
  if (v->device < 0) {
    v->device = h.device;
    RSVD_CUDA(cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking));
  } else if (v->device != h.device) {
    throw_param("virtual communicator: every rank must use the same device");
  }
  h.vcomm = v;
  h.rank = rank;
  h.nranks = v->n;
  h.own_stream_saved = h.own_stream;
  h.stream = h.own_stream = v->stream;  // one shared stream for all ranks
}

void vcomm_fail(Handle& h) {
  if (h.vcomm) h.vcomm->fail();
}

#define RSVD_NCCL(x)                                                                      \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      throw ::rsvdb::Error(RSVD_ERR_NCCL, std::string(#x " failed: ") + ncclGetErrorString(r_)); \
  } while (0)

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  RSVD_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
}

void comm_create(Handle& h, int rank, int nranks, const void* id128) {
  h.rank = rank;
  h.nranks = nranks;
  // nranks == 1 with an id: a one-rank communicator (the distributed path,
  // every NCCL call included, on one GPU); without an id: no communicator
  if (nranks < 1 || !id128) return;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  h.comm = new Comm;
  RSVD_NCCL(ncclCommInitRank(&h.comm->c, nranks, id, rank));
}

void comm_destroy(Handle& h) {
  if (h.comm) {
    if (h.comm->c) ncclCommDestroy(h.comm->c);
    delete h.comm;
    h.comm = nullptr;
  }
}

void allreduce_sum(Handle& h, double* p, int64_t count) {
  if (!h.dist() || count == 0) return;
  if (h.vcomm) {
    vcoll(h, p, p, [&](const VPtrs& ptrs) {
      launch_k(h, vc_reduce_kernel, vgrid(h, count), 256, 0, ptrs, h.vcomm->n, count, 0);
    });
    return;
  }
  RSVD_NCCL(ncclAllReduce(p, p, size_t(count), ncclDouble, ncclSum, h.comm->c, h.stream));
}

void allreduce_max(Handle& h, double* p, int64_t count) {
  if (!h.dist() || count == 0) return;
  if (h.vcomm) {
    vcoll(h, p, p, [&](const VPtrs& ptrs) {
      launch_k(h, vc_reduce_kernel, vgrid(h, count), 256, 0, ptrs, h.vcomm->n, count, 1);
    });
    return;
  }
  RSVD_NCCL(ncclAllReduce(p, p, size_t(count), ncclDouble, ncclMax, h.comm->c, h.stream));
}

void allgather(Handle& h, const double* send, double* recv, int64_t count) {
  if (!h.dist()) {
    if (send != recv)
      RSVD_CUDA(cudaMemcpyAsync(recv, send, size_t(count) * 8, cudaMemcpyDeviceToDevice, h.stream));
    return;
  }
  if (h.vcomm) {
    vcoll(h, send, recv, [&](const VPtrs& ptrs) {
      launch_k(h, vc_gather_kernel, vgrid(h, count * h.vcomm->n), 256, 0, ptrs, h.vcomm->n, count);
    });
    return;
  }
  RSVD_NCCL(ncclAllGather(send, recv, size_t(count), ncclDouble, h.comm->c, h.stream));
}

// Contiguous (sharded) matrix reductions: dense copy when ld != rows.
void allreduce_mat(Handle& h, DMat X) {
  if (!h.dist() || X.rows * X.cols == 0) return;
  if (X.ld == X.rows) {
    allreduce_sum(h, X.p, X.rows * X.cols);
    return;
  }
  double* tmp = h.ws.alloc(X.rows * X.cols);
  RSVD_CUDA(cudaMemcpy2DAsync(tmp, X.rows * 8, X.p, X.ld * 8, X.rows * 8, X.cols,
                              cudaMemcpyDeviceToDevice, h.stream));
  allreduce_sum(h, tmp, X.rows * X.cols);
  RSVD_CUDA(cudaMemcpy2DAsync(X.p, X.ld * 8, tmp, X.rows * 8, X.rows * 8, X.cols,
                              cudaMemcpyDeviceToDevice, h.stream));
}

// Global row count and this rank's row offset (host values; one tiny
// allgather, synchronizing).
void shard_rows(Handle& h, int64_t m_local, int64_t* m_global, int64_t* row_offset) {
  if (!h.dist()) {
    *m_global = m_local;
    *row_offset = 0;
    return;
  }
  if (h.shard_m_global > 0) {  // the caller's shard descriptor (rsvd_set_shard): no exchange
    if (h.shard_row_off < 0 || h.shard_row_off + m_local > h.shard_m_global)
      throw_dim("shard descriptor: rows exceed the global row count");
    *m_global = h.shard_m_global;
    *row_offset = h.shard_row_off;
    return;
  }
  if (h.vcomm) {  // host values: exchanged among the rank threads, no device work
    VComm& v = *h.vcomm;
    v.val[size_t(h.rank)] = m_local;
    if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
    int64_t tot = 0, off = 0;
    for (int r = 0; r < v.n; ++r) {
      if (r == h.rank) off = tot;
      tot += v.val[size_t(r)];
    }
    if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
    *m_global = tot;
    *row_offset = off;
    return;
  }
  double* d = h.ws.alloc(1 + h.nranks);
  const double v = double(m_local);
  RSVD_CUDA(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, h.stream));
  allgather(h, d, d + 1, 1);
  std::vector<double> all(size_t(h.nranks));
  RSVD_CUDA(cudaMemcpyAsync(all.data(), d + 1, 8 * size_t(h.nranks), cudaMemcpyDeviceToHost,
                            h.stream));
  stream_sync(h);
  int64_t tot = 0, off = 0;
  for (int r = 0; r < h.nranks; ++r) {
    if (r == h.rank) off = tot;
    tot += int64_t(all[size_t(r)]);
  }
  *m_global = tot;
  *row_offset = off;
}

}  // namespace rsvdb

namespace rsvdb {

void shard_layout(Handle& h, int64_t m_local, std::vector<int64_t>* rows, std::vector<int64_t>* offs) {
  const int R = h.nranks;
  rows->assign(size_t(R), 0);
  offs->assign(size_t(R), 0);
  if (!h.dist()) {
    (*rows)[0] = m_local;
    return;
  }
  std::vector<double> all(static_cast<size_t>(R));
  if (h.vcomm) {
    VComm& v = *h.vcomm;
    v.val[size_t(h.rank)] = m_local;
    if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
    for (int r = 0; r < R; ++r) all[size_t(r)] = double(v.val[size_t(r)]);
    if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
  } else {
    double* d = h.ws.alloc(1 + R);
    const double val = double(m_local);
    RSVD_CUDA(cudaMemcpyAsync(d, &val, 8, cudaMemcpyHostToDevice, h.stream));
    allgather(h, d, d + 1, 1);
    RSVD_CUDA(cudaMemcpyAsync(all.data(), d + 1, 8 * size_t(R), cudaMemcpyDeviceToHost, h.stream));
    stream_sync(h);
  }
  int64_t off = 0;
  for (int r = 0; r < R; ++r) {
    (*rows)[size_t(r)] = int64_t(all[size_t(r)]);
    (*offs)[size_t(r)] = off;
    off += (*rows)[size_t(r)];
  }
}

void peer_exchange(Handle& h, const double* send, int64_t sld, int64_t sr, int64_t sc, int to,
                   double* recv, int64_t rr, int64_t rc, int from) {
  if (h.vcomm) {
    // same device, same process: the receiver copies straight from the
    // sender's buffer (pointers exchanged among the rank threads)
    VComm& v = *h.vcomm;
    v.in[size_t(h.rank)] = send;
    v.val[size_t(h.rank)] = sld;
    if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
    const double* src = v.in[size_t(from)];
    const int64_t lds = v.val[size_t(from)];
    if (rr * rc > 0)
      RSVD_CUDA(cudaMemcpy2DAsync(recv, size_t(rr) * 8, src, size_t(lds) * 8, size_t(rr) * 8, size_t(rc),
                                  cudaMemcpyDeviceToDevice, h.stream));
    if (!v.barrier()) throw Error(RSVD_ERR_NCCL, "virtual communicator: a peer rank failed");
    return;
  }
  // NCCL: pack the strided block, then one send / recv pair
  double* pack = nullptr;
  if (sr * sc > 0) {
    pack = h.ws.alloc(sr * sc);
    RSVD_CUDA(cudaMemcpy2DAsync(pack, size_t(sr) * 8, send, size_t(sld) * 8, size_t(sr) * 8, size_t(sc),
                                cudaMemcpyDeviceToDevice, h.stream));
  }
  RSVD_NCCL(ncclGroupStart());
  if (sr * sc > 0) RSVD_NCCL(ncclSend(pack, size_t(sr * sc), ncclDouble, to, h.comm->c, h.stream));
  if (rr * rc > 0) RSVD_NCCL(ncclRecv(recv, size_t(rr * rc), ncclDouble, from, h.comm->c, h.stream));
  RSVD_NCCL(ncclGroupEnd());
}

}  // namespace rsvdb
