// Probe: host->HBM bandwidth via copy engine vs SM zero-copy 16B loads from mapped pinned memory.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)

template<int U>
__global__ void zc_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = tid; base < n16; base += stride * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + u * stride; if (i < n16) v[u] = __ldcs(src + i); }
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + u * stride; if (i < n16) dst[i] = v[u]; }
  }
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("dev %s SMs %d pciBus %d\n", p.name, p.multiProcessorCount, p.pciBusID);
  size_t bytes = 512ull << 20;
  void* h; CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  memset(h, 1, bytes);
  void* d; CK(cudaMalloc(&d, bytes));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float best = 1e9, ms;
  for (int i = 0; i < 10; ++i) {
    CK(cudaEventRecord(a, s)); CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  printf("CE H2D memcpy 512MiB: %.2f GB/s\n", bytes / best / 1e6);
  best = 1e9;
  for (int i = 0; i < 10; ++i) {
    CK(cudaEventRecord(a, s)); CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  printf("CE D2H memcpy 512MiB: %.2f GB/s\n", bytes / best / 1e6);
  // SM zero-copy
  size_t zbytes = 64ull << 20; size_t n16 = zbytes / 16;
  int grids[] = {8, 16, 32, 64, 148, 296};
  int blocks[] = {256, 512, 1024};
  for (int gi = 0; gi < 6; ++gi) for (int bi = 0; bi < 3; ++bi) {
    int g = grids[gi], bl = blocks[bi];
    for (int u : {1, 4, 8}) {
      best = 1e9;
      for (int i = 0; i < 5; ++i) {
        CK(cudaEventRecord(a, s));
        if (u == 1) zc_copy<1><<<g, bl, 0, s>>>((const int4*)h, (int4*)d, n16);
        else if (u == 4) zc_copy<4><<<g, bl, 0, s>>>((const int4*)h, (int4*)d, n16);
        else zc_copy<8><<<g, bl, 0, s>>>((const int4*)h, (int4*)d, n16);
        CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
      }
      printf("SM zero-copy grid %d block %d unroll %d: %.2f GB/s (%.3f ms for 64MiB)\n", g, bl, u, zbytes / best / 1e6, best);
    }
  }
  // chunk-sized copies: 5 MiB batches
  return 0;
}
