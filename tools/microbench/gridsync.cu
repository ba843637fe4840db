// Cost of one cooperative-groups grid barrier on this GPU, for 1..8 CTAs/SM
// of 256 threads (bounds the fused delta-stepping round, sssp.cu).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, unsigned long long* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned long long x = 0;
  for (int i = 0; i < iters; ++i) {
    x += i;
    g.sync();
  }
  if (x == 42) *sink = x;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  for (int per = 1; per <= 8; per *= 2) {
    int blocks = sms * per, iters = 20000;
    void* args[] = {&iters, &sink};
    cudaLaunchCooperativeKernel((void*)k_sync, blocks, 256, args, 0, 0);  // warm
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_sync, blocks, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync: %4d CTAs x 256 threads: %.3f us per barrier (%s)\n", blocks, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
