#pragma once
#include <vector>

#include "engine.hpp"

namespace stgp {
// sum-all-reduce of a device buffer over the context's communicator (no-op single rank)
void allreduce_sum(stgp_ctx* ctx, double* dev, size_t count);
void allreduce_host(stgp_ctx* ctx, std::vector<double>& v);
// neighbour rows [r0, r1) computed by this rank -> every rank holds all n rows
void gather_rows(stgp_ctx* ctx, int32_t* idx, double* dist, long long n, int m_v, int r0, int r1);
// Every rank filled slab `rank` (slab_doubles each, contiguous from buf; the rest of the first
// n_cols * ld doubles zero): afterwards all ranks hold all slabs.  NCCL: one in-place ncclAllGather;
// host hook: a sum all-reduce of the zero-filled buffer (x + 0 = x).
void allgather_cols(stgp_ctx* ctx, double* buf, size_t slab_doubles, long long n_cols, int ld);
// contiguous index shard [begin, end) of this context
void shard_rows(const stgp_ctx* ctx, int n, int& begin, int& end);
}  // namespace stgp
