// NCCL plumbing for row-sharded A (dist.cu).
#pragma once
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
}  // namespace rsvdb
