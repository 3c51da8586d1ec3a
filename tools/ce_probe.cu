// Probe: how the copy engines' H2D rate depends on the segment size of a gathered 16 MiB layer
// load (L8: 16 chunks x 1 MiB per layer), and whether an SM gather running beside a copy-engine
// batch adds anything once the link is busy.  Scattered segments: sources at random segment-
// aligned offsets of a 512 MiB pinned (hugepage-advised) buffer, destinations shuffled in HBM.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <random>
#include <sys/mman.h>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)

struct Seg { const int4* src; int4* dst; };

// one warp per segment, 4 x 16 B in flight per lane (the product gather's inner loop)
__global__ void seg_gather(const Seg* segs, int n, int seg16) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < n; s += nw) {
    const int4* src = segs[s].src; int4* dst = segs[s].dst;
    for (int i = lane; i < seg16; i += 128) {
      int4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) if (i + 32 * u < seg16) v[u] = __ldcs(src + i + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) if (i + 32 * u < seg16) dst[i + 32 * u] = v[u];
    }
  }
}

int main() {
  CK(cudaSetDevice(0));
  const size_t host_bytes = 512ull << 20, layer = 16ull << 20, dev_bytes = 64ull << 20;
  void* h = mmap(nullptr, host_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(h, host_bytes, MADV_HUGEPAGE);
  memset(h, 1, host_bytes);
  CK(cudaHostRegister(h, host_bytes, cudaHostRegisterMapped));
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  void* d; CK(cudaMalloc(&d, dev_bytes));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, j; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&j));
  std::mt19937 rng(1);
  float ms;
  Seg* dsegs; CK(cudaMalloc(&dsegs, sizeof(Seg) * 8192));
  for (size_t seg : {16ull << 10, 64ull << 10, 256ull << 10, 1ull << 20, 16ull << 20}) {
    size_t n = layer / seg;
    std::vector<size_t> so(host_bytes / seg), dofs(dev_bytes / seg);
    for (size_t i = 0; i < so.size(); ++i) so[i] = i;
    for (size_t i = 0; i < dofs.size(); ++i) dofs[i] = i;
    std::shuffle(so.begin(), so.end(), rng); std::shuffle(dofs.begin(), dofs.end(), rng);
    std::vector<void*> src(n), srcd(n), dst(n); std::vector<size_t> sz(n, seg);
    std::vector<Seg> hs(n);
    for (size_t i = 0; i < n; ++i) {
      src[i] = (char*)h + so[i] * seg; srcd[i] = (char*)hd + so[i] * seg; dst[i] = (char*)d + dofs[i] * seg;
      hs[i] = {(const int4*)srcd[i], (int4*)dst[i]};
    }
    CK(cudaMemcpy(dsegs, hs.data(), sizeof(Seg) * n, cudaMemcpyHostToDevice));
    cudaMemcpyAttributes attr{}; attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
    size_t idx = 0, fail = 0;
    // (1) one cudaMemcpyBatchAsync
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
      CK(cudaEventRecord(a, s));
      CK(cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), n, &attr, &idx, 1, &fail, s));
      CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
    }
    printf("seg %7zu KiB x %5zu: CE batch %.1f us = %.2f GB/s\n", seg >> 10, n, best * 1e3, layer / best / 1e6);
    // (2) per-segment cudaMemcpyAsync
    best = 1e9;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(a, s));
      for (size_t i = 0; i < n; ++i) CK(cudaMemcpyAsync(dst[i], src[i], seg, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
    }
    printf("seg %7zu KiB x %5zu: CE per-seg memcpy %.1f us = %.2f GB/s\n", seg >> 10, n, best * 1e3, layer / best / 1e6);
    // (3) SM gather alone, 16 and 32 CTAs
    for (int g : {16, 32}) {
      best = 1e9;
      for (int r = 0; r < 20; ++r) {
        CK(cudaEventRecord(a, s));
        seg_gather<<<g, 256, 0, s>>>(dsegs, (int)n, (int)(seg / 16));
        CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
      }
      printf("seg %7zu KiB x %5zu: SM gather %d CTAs %.1f us = %.2f GB/s\n", seg >> 10, n, g, best * 1e3, layer / best / 1e6);
    }
    // (4) hybrid: CE batch for the first f of the segments on s2, SM gather for the rest on s
    for (int pct : {25, 50, 75, 90}) {
      size_t nc = n * pct / 100; if (nc == 0 || nc == n) continue;
      best = 1e9;
      for (int r = 0; r < 20; ++r) {
        CK(cudaEventRecord(a, s)); CK(cudaStreamWaitEvent(s2, a));
        CK(cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), nc, &attr, &idx, 1, &fail, s2));
        seg_gather<<<16, 256, 0, s>>>(dsegs + nc, (int)(n - nc), (int)(seg / 16));
        CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(s, j));
        CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
      }
      printf("seg %7zu KiB x %5zu: hybrid CE %d%% + SM %.1f us = %.2f GB/s\n", seg >> 10, n, pct, best * 1e3, layer / best / 1e6);
    }
  }
  // (5) back-to-back layers: 32 CE batches of 64 x 256 KiB on one stream (pipeline shape)
  {
    size_t seg = 256ull << 10, n = layer / seg;
    std::vector<void*> src(n), dst(n); std::vector<size_t> sz(n, seg);
    for (size_t i = 0; i < n; ++i) { src[i] = (char*)h + ((i * 37) % (host_bytes / seg)) * seg; dst[i] = (char*)d + i * seg; }
    cudaMemcpyAttributes attr{}; attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    size_t idx = 0, fail = 0;
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(a, s));
      for (int l = 0; l < 32; ++l) CK(cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), n, &attr, &idx, 1, &fail, s));
      CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
    }
    printf("32 layers x 64 x 256 KiB CE batches back to back: %.3f ms = %.2f GB/s\n", best, 32 * layer / best / 1e6);
  }
  return 0;
}
