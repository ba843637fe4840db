// Microbenchmark: L2/HBM atomic + gather throughput on B200 (design input for PR kernels).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}

__global__ void gen_idx(uint32_t* idx, size_t n, uint32_t window, int sorted_chunks){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ idx[i] = hash32((uint32_t)i*2654435761u + 12345u) % window; }
}
__global__ void red_f64(const uint32_t* __restrict__ idx, double* acc, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ atomicAdd(acc+__ldcs(idx+i), 1.0); }
}
__global__ void red_f32(const uint32_t* __restrict__ idx, float* acc, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ atomicAdd(acc+__ldcs(idx+i), 1.0f); }
}
__global__ void red_u32(const uint32_t* __restrict__ idx, unsigned* acc, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ atomicAdd(acc+__ldcs(idx+i), 1u); }
}
__global__ void gather_f32(const uint32_t* __restrict__ idx, const float* __restrict__ x, float* out, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; float s=0;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ s += __ldg(x+__ldcs(idx+i)); }
  if(s==-1.f) out[0]=s;
}
__global__ void smem_f64(const uint32_t* __restrict__ idx, double* out, size_t n, int win){
  extern __shared__ double sm[];
  for(int j=threadIdx.x;j<win;j+=blockDim.x) sm[j]=0; __syncthreads();
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ atomicAdd(sm + (__ldcs(idx+i) % win), 1.0); }
  __syncthreads(); if(threadIdx.x==0 && sm[0]==-1) out[0]=sm[0];
}
__global__ void smem_f32(const uint32_t* __restrict__ idx, float* out, size_t n, int win){
  extern __shared__ float smf[];
  for(int j=threadIdx.x;j<win;j+=blockDim.x) smf[j]=0; __syncthreads();
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ atomicAdd(smf + (__ldcs(idx+i) % win), 1.0f); }
  __syncthreads(); if(threadIdx.x==0 && smf[0]==-1) out[0]=smf[0];
}
__global__ void stream_read(const int4* __restrict__ p, size_t n, int* out){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; int s=0;
  for(; i<n; i+= (size_t)gridDim.x*blockDim.x){ int4 v=__ldcs(p+i); s^=v.x^v.y^v.z^v.w; }
  if(s==0x12345) out[0]=s;
}
int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  printf("%s SMs=%d L2=%d MB\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize>>20);
  const size_t n = 1ull<<28;
  uint32_t* idx; CK(cudaMalloc(&idx, n*4));
  void* big; CK(cudaMalloc(&big, 2ull<<30));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grid = pr.multiProcessorCount*8, blk=256; float ms;
  // stream read 2GB
  stream_read<<<grid,blk>>>((int4*)big,(2ull<<30)/16,(int*)idx); cudaEventRecord(a);
  for(int r=0;r<3;r++) stream_read<<<grid,blk>>>((int4*)big,(2ull<<30)/16,(int*)idx);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("stream read: %.1f GB/s\n", 3*2.0*(1<<30)/ms/1e6);
  size_t wins_b[] = {4ull<<20, 16ull<<20, 48ull<<20, 96ull<<20, 256ull<<20, 1ull<<30};
  for(size_t wb: wins_b){
    uint32_t w64 = wb/8, w32 = wb/4;
    gen_idx<<<grid,blk>>>(idx,n,w64,0); CK(cudaDeviceSynchronize());
    cudaMemset(big,0,wb);
    red_f64<<<grid,blk>>>(idx,(double*)big,n); cudaEventRecord(a);
    red_f64<<<grid,blk>>>(idx,(double*)big,n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("win %5zu MB red.f64 random: %.1f Gop/s\n", wb>>20, n/ms/1e6);
    gen_idx<<<grid,blk>>>(idx,n,w32,0); CK(cudaDeviceSynchronize());
    red_f32<<<grid,blk>>>(idx,(float*)big,n); cudaEventRecord(a);
    red_f32<<<grid,blk>>>(idx,(float*)big,n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("win %5zu MB red.f32 random: %.1f Gop/s\n", wb>>20, n/ms/1e6);
    red_u32<<<grid,blk>>>(idx,(unsigned*)big,n); cudaEventRecord(a);
    red_u32<<<grid,blk>>>(idx,(unsigned*)big,n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("win %5zu MB red.u32 random: %.1f Gop/s\n", wb>>20, n/ms/1e6);
    gather_f32<<<grid,blk>>>(idx,(float*)big,(float*)idx,n); cudaEventRecord(a);
    gather_f32<<<grid,blk>>>(idx,(float*)big,(float*)idx,n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("win %5zu MB gather.f32 random: %.1f Gop/s\n", wb>>20, n/ms/1e6);
  }
  for(int win: {4096, 12288, 24576}){
    gen_idx<<<grid,blk>>>(idx,n,1u<<30,0);
    CK(cudaFuncSetAttribute(smem_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
    CK(cudaFuncSetAttribute(smem_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
    int g2 = pr.multiProcessorCount * (win<=4096?6:(win<=12288?2:1));
    smem_f64<<<g2,512,win*8>>>(idx,(double*)big,n,win); cudaEventRecord(a);
    smem_f64<<<g2,512,win*8>>>(idx,(double*)big,n,win); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);
    printf("smem win %d f64 atomicAdd: %.1f Gop/s\n", win, n/ms/1e6);
    smem_f32<<<g2,512,win*4>>>(idx,(float*)big,n,win); cudaEventRecord(a);
    smem_f32<<<g2,512,win*4>>>(idx,(float*)big,n,win); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);
    printf("smem win %d f32 atomicAdd: %.1f Gop/s\n", win, n/ms/1e6);
  }
  return 0;
}
