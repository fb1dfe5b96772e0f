// Shared host/device utilities for the stgp B200 engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace stgp {

// Error classes of the reference (types.hpp:26-38) mapped to ABI return codes.
enum ErrCode : int { kOk = 0, kInternal = 1, kConfig = 2, kData = 3, kNumeric = 4 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(kConfig, m); }
[[noreturn]] inline void data_error(const std::string& m) { throw Error(kData, m); }
[[noreturn]] inline void numeric_error(const std::string& m) { throw Error(kNumeric, m); }

#define STGP_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::stgp::Error(::stgp::kInternal, std::string("CUDA error: ") +              \
                                                 cudaGetErrorString(e_) + " at " +       \
                                                 __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define STGP_LAUNCH_CHECK() STGP_CUDA(cudaGetLastError())

// Device-side bounds checks of the checked build (`make checks`: -DSTGP_DEVICE_CHECKS, library
// libstgp_b200_checks.so, selected with STGP_LIB): a violated index bound traps the kernel, which
// surfaces as a CUDA error on the next synchronisation.  compute-sanitizer is closed on the GPU pool;
// the test suite run against the checked build is its substitute (profiles/r02/device_checks.log).
#ifdef STGP_DEVICE_CHECKS
#define STGP_DCHECK(cond)    \
  do {                       \
    if (!(cond)) __trap();   \
  } while (0)
#else
#define STGP_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

// Device memory for DevBuf (engine.cu): the device's memory pool with an unbounded release
// threshold, so steady-state allocations and frees stay inside the process instead of going to
// the driver (cudaMalloc / cudaFree calls blocked the host for up to 1.7 s at random on the B200
// boxes).  dev_free keeps cudaFree's semantics: it waits for the device before the block can be
// reused.  STGP_POOL=0 restores cudaMalloc / cudaFree.
void* dev_alloc(size_t bytes);
void dev_free(void* p);

// Owning device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) dev_free(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    ensure(count);
    if (count) STGP_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(T* h, size_t count, cudaStream_t s) const {
    if (count) STGP_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void zero(cudaStream_t s) {
    if (n) STGP_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  T* get() const { return p; }
};

// Covariance hyperparameters (covariance.hpp:23-38), identical layout to the ABI struct.
struct Params {
  double sigma2, sigma1_2, a, c, alpha, nu, beta, delta;
};

// Temporal factors of one time lag (covariance.hpp:89-96), tabulated on the host.
struct TF {
  double pow_mE, pow_mbh, inv_T, log_T, u2a, u2a_logu;
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace stgp
