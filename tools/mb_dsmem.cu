// Microbenchmark: random f64 gathers from an L2-resident window vs from a
// cluster's distributed shared memory (the PageRank hot-kernel question:
// does a cluster-wide hot-contribution cache beat L2 gathers?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_dsmem tools/mb_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// mode 0: global gathers over [0, n); mode 1: smem-local gathers (per CTA cache of ncache);
// mode 2: DSMEM gathers over the cluster (ncache per CTA, csize CTAs);
// mode 3: mixed: fraction pct% to DSMEM, rest global.
template <int kU>
__global__ void k_gather(const double* __restrict__ a, uint32_t n, int iters, int mode, int ncache, int pct,
                         double* out) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < ncache; i += blockDim.x) s[i] = a[i + blockIdx.x % 7];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned csize = cl.num_blocks();
  cl.sync();
  uint32_t st = hash32(blockIdx.x * blockDim.x + threadIdx.x + 12345);
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double v[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      st = hash32(st + q);
      if (mode == 0) {
        v[q] = __ldg(a + (st % n));
      } else if (mode == 1) {
        v[q] = s[st % ncache];
      } else {
        const bool ds = mode == 2 || (int)(st % 100) < pct;
        if (ds) {
          const uint32_t k = (st >> 7) % (ncache * csize);
          const double* p = cl.map_shared_rank(s, k / ncache);
          v[q] = p[k % ncache];
        } else {
          v[q] = __ldg(a + (st % n));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) acc += v[q];
  }
  cl.sync();
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const uint32_t n = 47u * 1024 * 1024 / 8, nmax = 94u * 1024 * 1024 / 8;
  double *a, *out;
  cudaMalloc(&a, (size_t)nmax * 8);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, (size_t)nmax * 8);
  const int threads = 1024, iters = 512;
  const int ncache = 16384;  // 128 KB per CTA
  auto fn = k_gather<8>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ncache * 8);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  // L1 capacity probe: global gathers with 0 / 64 / 128 / 192 KB of shared memory and 256..1024 threads
  for (int smem_kb : {0, 64, 128, 192}) {
    for (int thr : {256, 512, 1024}) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
      cudaEvent_t t0, t1;
      cudaEventCreate(&t0);
      cudaEventCreate(&t1);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, thr, smem_kb * 1024);
      const int grid = sms * per_sm;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(t0);
        k_gather<8><<<grid, thr, smem_kb * 1024>>>(a, n, iters, 0, 0, 0, out);
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
      }
      float ms_ = 0;
      cudaEventElapsedTime(&ms_, t0, t1);
      const double loads = (double)grid * thr * iters * 8;
      printf("global gathers smem %3d KB, %4d thr x %d CTA/SM: %7.1f G loads/s  %.3f /clk/SM\n", smem_kb, thr,
             per_sm, loads / ms_ / 1e6, loads / (ms_ * 1e-3) / (clk * 1e3) / sms);
    }
  }
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ncache * 8);
  for (uint32_t wmb : {1u, 8u, 24u, 47u, 70u, 94u}) {  // window size probe (1024 thr, 128 KB smem)
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const uint32_t nw = wmb * 1024 * 1024 / 8;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(t0);
      k_gather<8><<<sms, 1024, ncache * 8>>>(a, nw, iters, 0, 0, 0, out);
      cudaEventRecord(t1);
      cudaEventSynchronize(t1);
    }
    float ms_ = 0;
    cudaEventElapsedTime(&ms_, t0, t1);
    const double loads = (double)sms * 1024 * iters * 8;
    printf("window %3u MB: %7.1f G loads/s  %.3f /clk/SM\n", wmb, loads / ms_ / 1e6,
           loads / (ms_ * 1e-3) / (clk * 1e3) / sms);
  }
  for (int cs : {1, 2}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = ncache * 8;
    cfg.gridDim = dim3((sms / cs) * cs);
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)fn, &cfg);
    printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, ncl, ncl * cs, cudaGetErrorString(e));
    if (ncl <= 0) continue;
    cfg.gridDim = dim3(ncl * cs);
    struct M { int mode, pct; const char* name; } ms[] = {
        {0, 0, "global L2 window 47MB"}, {1, 0, "smem local"}, {2, 0, "dsmem cluster"},
        {3, 25, "mixed 25% dsmem"}, {3, 50, "mixed 50% dsmem"}};
    for (auto m : ms) {
      if (cs == 1 && m.mode >= 2) continue;
      cudaEvent_t t0, t1;
      cudaEventCreate(&t0);
      cudaEventCreate(&t1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(t0);
        cudaLaunchKernelEx(&cfg, fn, (const double*)a, n, iters, m.mode, ncache, m.pct, out);
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
      }
      float ms_ = 0;
      cudaEventElapsedTime(&ms_, t0, t1);
      const double loads = (double)cfg.gridDim.x * threads * iters * 8;
      const double per_clk_sm = loads / (ms_ * 1e-3) / (clk * 1e3) / cfg.gridDim.x;
      printf("  %-24s %8.3f ms  %7.1f G loads/s  %.3f loads/clk/SM  (%s)\n", m.name, ms_, loads / ms_ / 1e6,
             per_clk_sm, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
