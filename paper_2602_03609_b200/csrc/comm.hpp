#pragma once
#include <vector>

#include "engine.hpp"

namespace stgp {
// sum-all-reduce of a device buffer over the context's communicator (no-op single rank)
void allreduce_sum(stgp_ctx* ctx, double* dev, size_t count);
void allreduce_host(stgp_ctx* ctx, std::vector<double>& v);
// neighbour rows [r0, r1) computed by this rank -> every rank holds all n rows
void gather_rows(stgp_ctx* ctx, int32_t* idx, double* dist, long long n, int m_v, int r0, int r1);
// contiguous index shard [begin, end) of this context
void shard_rows(const stgp_ctx* ctx, int n, int& begin, int& end);
}  // namespace stgp
