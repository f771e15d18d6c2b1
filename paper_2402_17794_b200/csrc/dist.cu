// Row-sharded multi-GPU plumbing: one process per GPU, NCCL over NVLink /
// NVSwitch.  The reference is single-threaded (README.md:152); the only data
// that crosses GPUs in this engine are the small partial products the
// north_star names: n x l / l x n (A^T Y, Q^T A, A^T Psi), l x l Gram / R /
// inner-product partials, and scalars.  A itself never moves.
//
// Determinism: NCCL_ALGO / NCCL_PROTO can be pinned by the caller (bench.py
// pins Ring/Simple) so reruns are bitwise identical.
#include <nccl.h>

#include <cstring>

#include "common.cuh"
#include "dist.cuh"

namespace rsvdb {

struct Comm {
  ncclComm_t c = nullptr;
};

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
  RSVD_NCCL(ncclAllReduce(p, p, size_t(count), ncclDouble, ncclSum, h.comm->c, h.stream));
}

void allreduce_max(Handle& h, double* p, int64_t count) {
  if (!h.dist() || count == 0) return;
  RSVD_NCCL(ncclAllReduce(p, p, size_t(count), ncclDouble, ncclMax, h.comm->c, h.stream));
}

void allgather(Handle& h, const double* send, double* recv, int64_t count) {
  if (!h.dist()) {
    if (send != recv)
      RSVD_CUDA(cudaMemcpyAsync(recv, send, size_t(count) * 8, cudaMemcpyDeviceToDevice, h.stream));
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
