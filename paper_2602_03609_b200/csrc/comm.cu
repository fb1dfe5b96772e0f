// Multi-GPU plumbing: one process per GPU, observations sharded by contiguous
// index ranges; partial sums are all-reduced with NCCL over
// NVLink/NVSwitch.  Without a communicator a context returns its shard's
// partials (used by the single-GPU shard emulation tests).
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "comm.hpp"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

void allreduce_sum(stgp_ctx* ctx, double* dev, size_t count) {
  if (ctx->world == 1 || count == 0) return;
  if (!ctx->comm && ctx->host_allreduce) {
    std::vector<double> h(count);
    STGP_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->host_allreduce(ctx->host_allreduce_user, h.data(), static_cast<int64_t>(count)) != 0)
      throw Error(kInternal, "host all-reduce callback failed");
    STGP_CUDA(cudaMemcpyAsync(dev, h.data(), sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  if (!ctx->comm) return;
  const ncclResult_t r = ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, reinterpret_cast<ncclComm_t>(ctx->comm),
                                       ctx->stream);
  if (r != ncclSuccess) throw Error(kInternal, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
}

void allreduce_host(stgp_ctx* ctx, std::vector<double>& v) {
  if (ctx->world == 1 || v.empty()) return;
  if (!ctx->comm && ctx->host_allreduce) {
    if (ctx->host_allreduce(ctx->host_allreduce_user, v.data(), static_cast<int64_t>(v.size())) != 0)
      throw Error(kInternal, "host all-reduce callback failed");
    return;
  }
  if (!ctx->comm) return;
  DevBuf<double> d;
  d.upload(v.data(), v.size(), ctx->stream);
  allreduce_sum(ctx, d.get(), v.size());
  d.download(v.data(), v.size(), ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
}

namespace {
__global__ void gather_pack_kernel(long long total, int m_v, int r0, int r1, const int32_t* idx, const double* dist,
                                   double* bi, double* bd) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = e / m_v;
    const bool own = row >= r0 && row < r1;
    bi[e] = own ? static_cast<double>(idx[e]) + 1.0 : 0.0;
    bd[e] = own && dist ? dist[e] : 0.0;
  }
}
__global__ void gather_unpack_kernel(long long total, const double* bi, const double* bd, int32_t* idx, double* dist) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    idx[e] = static_cast<int32_t>(bi[e]) - 1;
    if (dist) dist[e] = bd[e];
  }
}
}  // namespace

// Every rank computed neighbour rows [r0, r1) of its shard; afterwards all ranks hold all rows.
// NCCL: the ranks' row ranges are exchanged once (a 2 x world host all-reduce), then the int32 indices
// and f64 distances of the own rows go out in one ncclAllGather each, padded to the longest range, and
// land at their ranges with device copies: 12 bytes per neighbour slot, stream ordered, no host sync.
// Host hook (in-process test ranks): a sum all-reduce of zero-filled buffers, indices stored as idx + 1
// (exact in f64; distances are >= +0, so x + 0 = x bit for bit).
void gather_rows(stgp_ctx* ctx, int32_t* idx, double* dist, long long n, int m_v, int r0, int r1) {
  if (ctx->world == 1 || n == 0) return;
  if (ctx->comm) {
    std::vector<double> rng(static_cast<size_t>(2 * ctx->world), 0.0);
    rng[static_cast<size_t>(2 * ctx->rank)] = r0;
    rng[static_cast<size_t>(2 * ctx->rank + 1)] = r1;
    allreduce_host(ctx, rng);
    long long maxrows = 0;
    for (int k = 0; k < ctx->world; ++k)
      maxrows = std::max<long long>(maxrows, static_cast<long long>(rng[2 * k + 1] - rng[2 * k]));
    const size_t slot = static_cast<size_t>(std::max<long long>(maxrows, 1)) * m_v;
    DevBuf<int32_t> si(slot), ri(slot * ctx->world);
    DevBuf<double> sd(slot), rd(slot * ctx->world);
    const size_t own = static_cast<size_t>(r1 - r0) * m_v;
    if (own) {
      STGP_CUDA(cudaMemcpyAsync(si.get(), idx + static_cast<size_t>(r0) * m_v, own * 4, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      if (dist)
        STGP_CUDA(cudaMemcpyAsync(sd.get(), dist + static_cast<size_t>(r0) * m_v, own * 8, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
    }
    ncclComm_t c = reinterpret_cast<ncclComm_t>(ctx->comm);
    ncclResult_t r = ncclAllGather(si.get(), ri.get(), slot, ncclInt32, c, ctx->stream);
    if (r == ncclSuccess && dist) r = ncclAllGather(sd.get(), rd.get(), slot, ncclDouble, c, ctx->stream);
    if (r != ncclSuccess) throw Error(kInternal, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    for (int k = 0; k < ctx->world; ++k) {
      const long long k0 = static_cast<long long>(rng[2 * k]), k1 = static_cast<long long>(rng[2 * k + 1]);
      if (k == ctx->rank || k1 <= k0) continue;
      const size_t cnt = static_cast<size_t>(k1 - k0) * m_v;
      STGP_CUDA(cudaMemcpyAsync(idx + k0 * m_v, ri.get() + k * slot, cnt * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      if (dist)
        STGP_CUDA(cudaMemcpyAsync(dist + k0 * m_v, rd.get() + k * slot, cnt * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));  // the staging buffers are freed at scope exit
    return;
  }
  const long long total = n * m_v;
  DevBuf<double> bi(static_cast<size_t>(total)), bd(static_cast<size_t>(total));
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, ctx->num_sms * 32LL));
  gather_pack_kernel<<<grid, 256, 0, ctx->stream>>>(total, m_v, r0, r1, idx, dist, bi.get(), bd.get());
  ++ctx->launches;
  allreduce_sum(ctx, bi.get(), static_cast<size_t>(total));
  allreduce_sum(ctx, bd.get(), static_cast<size_t>(total));
  gather_unpack_kernel<<<grid, 256, 0, ctx->stream>>>(total, bi.get(), bd.get(), idx, dist);
  ++ctx->launches;
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
}

void allgather_cols(stgp_ctx* ctx, double* buf, size_t slab_doubles, long long n_cols, int ld) {
  if (ctx->world == 1) return;
  if (ctx->comm) {
    const ncclResult_t r = ncclAllGather(buf + static_cast<size_t>(ctx->rank) * slab_doubles, buf, slab_doubles,
                                         ncclDouble, reinterpret_cast<ncclComm_t>(ctx->comm), ctx->stream);
    if (r != ncclSuccess) throw Error(kInternal, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    return;
  }
  allreduce_sum(ctx, buf, static_cast<size_t>(n_cols) * ld);
}

void shard_rows(const stgp_ctx* ctx, int n, int& begin, int& end) {
  begin = static_cast<int>(static_cast<long long>(n) * ctx->rank / ctx->world);
  end = static_cast<int>(static_cast<long long>(n) * (ctx->rank + 1) / ctx->world);
}

}  // namespace stgp

extern "C" {

int stgp_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    stgp::g_last_error = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return STGP_ERR_INTERNAL;
  }
  std::memcpy(out128, &id, sizeof(id));
  return STGP_OK;
}

int stgp_ctx_init_nccl(stgp_ctx* ctx, const void* uid, int rank, int world) {
  if (!ctx || !uid || world < 1 || rank < 0 || rank >= world) {
    stgp::g_last_error = "stgp_ctx_init_nccl: bad argument";
    return STGP_ERR_CONFIG;
  }
  cudaSetDevice(ctx->device);
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm;
  const ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) {
    stgp::g_last_error = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
    return STGP_ERR_INTERNAL;
  }
  ctx->comm = reinterpret_cast<ncclComm*>(comm);
  ctx->rank = rank;
  ctx->world = world;
  return STGP_OK;
}

int stgp_ctx_set_host_allreduce(stgp_ctx* ctx, stgp_allreduce_fn fn, void* user) {
  if (!ctx) {
    stgp::g_last_error = "null context";
    return STGP_ERR_CONFIG;
  }
  ctx->host_allreduce = fn;
  ctx->host_allreduce_user = user;
  return STGP_OK;
}

void stgp_ctx_release_comm(stgp_ctx* ctx) {
  if (ctx && ctx->comm) {
    ncclCommDestroy(reinterpret_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
  }
}

}  // extern "C"
