// NCCL plumbing for row-sharded A (dist.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace rsvdb {
void nccl_unique_id(void* out128);
void comm_create(Handle& h, int rank, int nranks, const void* id128);
void comm_destroy(Handle& h);
void allreduce_sum(Handle& h, double* p, int64_t count);
void allreduce_max(Handle& h, double* p, int64_t count);
void allgather(Handle& h, const double* send, double* recv, int64_t count);
void allreduce_mat(Handle& h, DMat X);
void shard_rows(Handle& h, int64_t m_local, int64_t* m_global, int64_t* row_offset);
// Every rank's local row count and first row (collective).
void shard_layout(Handle& h, int64_t m_local, std::vector<int64_t>* rows, std::vector<int64_t>* offs);
// Point-to-point step of a ring: send the (sr x sc, ld sld) block at `send`
// to rank `to` and receive an (rr x rc, dense) block from rank `from` into
// `recv` (collective over all ranks, one partner each way).
void peer_exchange(Handle& h, const double* send, int64_t sld, int64_t sr, int64_t sc, int to,
                   double* recv, int64_t rr, int64_t rc, int from);
// Virtual (in-process, one device) communicator, see dist.cu.
VComm* vcomm_create(int nranks);
void vcomm_destroy(VComm* v);
void vcomm_attach(Handle& h, VComm* v, int rank);
void vcomm_fail(Handle& h);  // release the peers of a rank whose call failed
}  // namespace rsvdb
