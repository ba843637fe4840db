// common.cuh — error plumbing, device buffers and warp/block primitives shared
// by every translation unit of libgg.so (sm_100a only).
#pragma once
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys/ncu timelines
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>
#include <stdexcept>
#include <vector>
#include <mutex>
#include <chrono>
#include "../../include/gg.h"

namespace gg {

// ---------------------------------------------------------------------------
// Errors: C++ exceptions inside the library, gg_status + thread-local message
// at the C boundary (see api.cu: GG_API_BEGIN / GG_API_END).
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline std::string strf(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return std::string(buf);
}

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define GG_CUDA(x)                                                                 \
  do {                                                                             \
    cudaError_t e__ = (x);                                                         \
    if (e__ != cudaSuccess) {                                                      \
      cudaGetLastError();                                                          \
      ::gg::fail(e__ == cudaErrorMemoryAllocation ? GG_ERR_OOM : GG_ERR_CUDA,       \
                 ::gg::strf("%s failed: %s (%s:%d)", #x, cudaGetErrorString(e__),   \
                            __FILE__, __LINE__));                                  \
    }                                                                              \
  } while (0)

#define GG_LAUNCH_CHECK() GG_CUDA(cudaGetLastError())

void set_last_error(const std::string& m);
void count_launch(int n = 1);     // per-thread launch counter (stats.gpu_launches)
int64_t launches_now();

// ---------------------------------------------------------------------------
// Device buffer (RAII, cudaMalloc on the current device)
// ---------------------------------------------------------------------------
// Device memory comes from a per-device caching pool (engine.cu): freed
// blocks are kept by size class and handed out again, so the per-call
// buffers of a query (parents, frontiers, marks, queues) cost no
// cudaMalloc/cudaFree -- which synchronise the device and take milliseconds
// for GB-sized blocks.  All library work is ordered on the legacy default
// stream, so a block freed after its last use can be reused by later work.
void* pool_alloc(size_t bytes, size_t* granted);
void pool_free(void* p, size_t granted);
void pool_trim();  // return every cached block to the driver
void pool_counters(int64_t* mallocs, int64_t* frees, int64_t* cached);

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t granted = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), granted(o.granted) { o.p = nullptr; o.n = 0; o.granted = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; granted = o.granted;
      o.p = nullptr; o.n = 0; o.granted = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count == 0) count = 1;  // keep a valid pointer for empty arrays
    p = static_cast<T*>(pool_alloc(count * sizeof(T), &granted));
    n = count;
  }
  void release() {
    if (p) pool_free(p, granted);
    p = nullptr;
    n = 0;
    granted = 0;
  }
  void zero(cudaStream_t s = 0) { if (p) GG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

// Scratch for CUB temp storage that only grows.
struct Scratch {
  DevBuf<uint8_t> buf;
  void* get(size_t bytes) {
    if (buf.n < bytes) buf.alloc(bytes + (bytes >> 3));
    return buf.p;
  }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) GG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// RAII NVTX range (SURVEY §5 tracing): the driver phases show up named in
// nsys / ncu --nvtx timelines; a no-op without a profiler attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

inline double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

int sm_count(int dev);
int64_t l2_bytes(int dev);

inline unsigned grid_for(int64_t work, int block, int dev, int per_sm = 8) {
  int64_t want = (work + block - 1) / block;
  int64_t cap = (int64_t)sm_count(dev) * per_sm;
  if (want < 1) want = 1;
  return (unsigned)(want < cap ? want : cap);
}

// ---------------------------------------------------------------------------
// Device primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

// Load of data written earlier in the same cooperative launch, separated by
// a grid barrier: cg::grid_group::sync fences (CCTL.IVALL: the SM's L1 is
// invalidated after its last block arrives), so a plain L1-cached load sees
// the pre-barrier writes -- unlike ld.global.nc, which may serve stale data
// for the launch's lifetime, and unlike ld.global.cg, which skips L1.
template <class T>
__device__ __forceinline__ T ld_fresh(const T* p) { return *p; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Counter-based RNG (splitmix64 finaliser) for the synthetic generators.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Streaming loads that should not displace L2-resident vertex data
// (ld.global.cs: evict-first in L1 and L2).
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ int4 ld_stream4(const int4* p) { return __ldcs(p); }
__device__ __forceinline__ int64_t ld_stream64(const int64_t* p) {
  return (int64_t)__ldcs(reinterpret_cast<const long long*>(p));
}

}  // namespace gg
