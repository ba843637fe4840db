// Random-gather microbenchmark: can bulk copies (cp.async.bulk, the TMA
// engine's 1-D form) fetch random 16-byte items from an L2-resident window
// faster than LDG gathers, whose L1->XBAR miss-request interface caps at ~1
// request per clock per SM (profiles/r02/microbench_l2_gathers_dsmem.txt)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mb_tma_gather tools/mb_tma_gather.cu
//
// Mode 0: each thread LDGs 8-byte items at random 16-byte-aligned offsets.
// Mode 1: each thread issues cp.async.bulk of 16 bytes per item into its
//         own shared-memory slots, one mbarrier per warp (expect_tx), wait,
//         then reads one 8-byte word of each slot (so the data is used).
// Reported: items per second and items per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int kItems>
__global__ void k_ldg(const double2* __restrict__ win, uint32_t nslots, int iters, double* sink) {
  double acc = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    double v[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      s = hash32(s + q + 1);
      v[q] = __ldg(reinterpret_cast<const double*>(win + (s % nslots)));
    }
#pragma unroll
    for (int q = 0; q < kItems; ++q) acc += v[q];
  }
  if (acc == 1234.5) *sink = acc;
}

template <int kItems>
__global__ void k_bulk(const double2* __restrict__ win, uint32_t nslots, int iters, double* sink) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* slots = reinterpret_cast<double2*>(smem);                          // blockDim * kItems
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + blockDim.x * kItems * 16);  // one per warp
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + wid);
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(32));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  double acc = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t phase = 0;
  for (int it = 0; it < iters; ++it) {
    // every lane arrives expecting its own bytes, then issues its copies
    uint64_t st;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
                 : "=l"(st) : "r"(bar), "r"(kItems * 16) : "memory");
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      s = hash32(s + q + 1);
      const double2* src = win + (s % nslots);
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(slots + threadIdx.x * kItems + q);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                   :: "r"(dst), "l"(src), "r"(bar) : "memory");
    }
    uint32_t done = 0;
    for (int spin = 0; !done; ++spin) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(bar), "r"(phase) : "memory");
      if (spin > (1 << 22)) {  // bounded: never hang the GPU on a wrong tx count
        *sink = -1.0;
        return;
      }
    }
    phase ^= 1;
#pragma unroll
    for (int q = 0; q < kItems; ++q) acc += slots[threadIdx.x * kItems + q].x;
    __syncwarp();
  }
  if (acc == 1234.5) *sink = acc;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));  // kHz
  const size_t win_bytes = 40u << 20;  // L2-resident window
  const uint32_t nslots = (uint32_t)(win_bytes / 16);
  double2* win;
  double* sink;
  CK(cudaMalloc(&win, win_bytes));
  CK(cudaMemset(win, 0, win_bytes));
  CK(cudaMalloc(&sink, 8));
  constexpr int kItems = 8;
  const int iters = 200;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int threads : {256, 512, 1024}) {
    for (int per_sm : {1, 2}) {
      if (threads * per_sm > 2048) continue;
      const int grid = sms * per_sm;
      const size_t smem = (size_t)threads * kItems * 16 + (threads / 32) * 8;
      CK(cudaFuncSetAttribute(k_bulk<kItems>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
          CK(cudaEventRecord(a));
          if (mode == 0) k_ldg<kItems><<<grid, threads>>>(win, nslots, iters, sink);
          else k_bulk<kItems><<<grid, threads, smem>>>(win, nslots, iters, sink);
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          CK(cudaGetLastError());
          double hs = 0;
          CK(cudaMemcpy(&hs, sink, 8, cudaMemcpyDeviceToHost));
          if (hs == -1.0) { printf("bulk wait timed out\n"); return 2; }
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (rep == 0) continue;  // warm-up
          const double items = (double)grid * threads * kItems * iters;
          const double per_s = items / (ms * 1e-3);
          printf("%s threads %4d x %d/SM smem %6zu B: %.3f ms, %.1f G items/s, %.3f items/clk/SM (at %d MHz)\n",
                 mode ? "bulk16" : "ldg8  ", threads, per_sm, mode ? smem : (size_t)0, ms, per_s / 1e9,
                 per_s / (sms * (clk * 1e3)), clk / 1000);
        }
      }
    }
  }
  return 0;
}
