// Microbenchmark: dependent-chain latency of the operations on the fused
// SSSP's critical path (one thread; L2-resident data): global load through
// L1/TEX (__ldg), volatile load, 64-bit atomicMin with and without a used
// result, 32-bit atomicAdd, shared-memory atomicAdd, __syncthreads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mb_latency tools/mb_latency.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

__global__ void k_lat(unsigned long long* a, const uint32_t* chain, int n, unsigned long long* out) {
  __shared__ unsigned s_ctr;
  s_ctr = 0;  // launched with one thread
  uint32_t j = 0;
  // warm
  for (int i = 0; i < n; ++i) j = __ldg(chain + j);
  unsigned long long t0 = clk();
  for (int i = 0; i < n; ++i) j = __ldg(chain + j);
  unsigned long long t1 = clk();
  out[0] = (t1 - t0) / n;
  for (int i = 0; i < n; ++i) j = *((volatile const uint32_t*)chain + j);
  unsigned long long t2 = clk();
  out[1] = (t2 - t1) / n;
  unsigned long long v = j;
  for (int i = 0; i < n; ++i) v = atomicMin(a + (v & 1023) * 16, v + 5) & 0xffff;
  unsigned long long t3 = clk();
  out[2] = (t3 - t2) / n;
  unsigned w = (unsigned)v;
  for (int i = 0; i < n; ++i) w = atomicAdd((unsigned*)a + 64 * 1024 + (w & 1023) * 32, 1u) & 0xffff;
  unsigned long long t4 = clk();
  out[3] = (t4 - t3) / n;
  for (int i = 0; i < n; ++i) w = atomicAdd(&s_ctr, w & 1) & 0xff;
  unsigned long long t5 = clk();
  out[4] = (t5 - t4) / n;
  out[5] = w;
}

// relax-like chain: load from a random slot of arr (ids), then atomicMin on a
// random slot of dist; `span` sets the footprint (L2-resident vs DRAM)
__global__ void k_relax(const uint32_t* arr, unsigned long long* dist, uint64_t span, int n,
                        unsigned long long* out, int slot) {
  uint64_t x = 12345 + slot;
  uint32_t j = 0;
  unsigned long long t0 = clk();
  for (int i = 0; i < n; ++i) {
    x = x * 6364136223846793005ULL + 1442695040888963407ULL + j;
    j = __ldg(arr + ((x >> 20) % span));
    x = x * 6364136223846793005ULL + 1442695040888963407ULL;
    j += (uint32_t)atomicMin(dist + ((x >> 20) + j) % span, 5ULL + i) & 1;
  }
  unsigned long long t1 = clk();
  out[slot] = (t1 - t0) / n;
}

__global__ void k_sync(int n, unsigned long long* out) {
  unsigned long long t0 = clk();
  for (int i = 0; i < n; ++i) __syncthreads();
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) out[6] = (t1 - t0) / n;
}

int main() {
  const int n = 4096, len = 1 << 20;
  uint32_t* h = new uint32_t[len];
  // random cyclic permutation over 1M entries (4 MB: L2-resident)
  for (int i = 0; i < len; ++i) h[i] = i;
  unsigned long long s = 88172645463325252ULL;
  for (int i = len - 1; i > 0; --i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    int k = s % i;
    uint32_t t = h[i]; h[i] = h[k]; h[k] = t;
  }
  uint32_t* nx = new uint32_t[len];
  for (int i = 0; i < len; ++i) nx[h[i]] = h[(i + 1) % len];
  uint32_t* chain;
  unsigned long long *a, *out;
  cudaMalloc(&chain, len * 4);
  cudaMalloc(&a, 1 << 24);
  cudaMalloc(&out, 64);
  cudaMemcpy(chain, nx, len * 4, cudaMemcpyHostToDevice);
  cudaMemset(a, 0xff, 1 << 24);
  k_lat<<<1, 1>>>(a, chain, n, out);
  k_sync<<<1, 256>>>(n, out);
  unsigned long long o[8];
  cudaMemcpy(o, out, 64, cudaMemcpyDeviceToHost);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const char* names[] = {"__ldg L2 hit (chase)", "volatile ld L2 hit (chase)", "atomicMin u64 (used result)",
                         "atomicAdd u32 global (used)", "atomicAdd smem (used)", "", "__syncthreads 256 thr"};
  for (int i : {0, 1, 2, 3, 4, 6})
    printf("%-32s %6llu cycles  %.0f ns\n", names[i], o[i], o[i] / (clk_khz * 1e-6));
  {
    uint32_t* arr;
    unsigned long long* dist;
    const uint64_t big = 1ull << 27;  // 512 MB ids / 1 GB dist
    cudaMalloc(&arr, big * 4);
    cudaMalloc(&dist, big * 8);
    cudaMemset(arr, 0, big * 4);
    cudaMemset(dist, 0xff, big * 8);
    const uint64_t spans[] = {1ull << 16, 1ull << 20, 1ull << 22, big};
    for (int k = 0; k < 4; ++k) {
      k_relax<<<1, 1>>>(arr, dist, spans[k], 256, out, 0);  // warm-up
      k_relax<<<1, 1>>>(arr, dist, spans[k], 2048, out, 0);
      cudaMemcpy(o, out, 8, cudaMemcpyDeviceToHost);
      printf("relax chain (ld + atomicMin), span %10llu entries: %6llu cycles  %.0f ns\n",
             (unsigned long long)spans[k], o[0], o[0] / (clk_khz * 1e-6));
    }
  }
  printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
