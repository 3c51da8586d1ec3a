// Probe: host link with traffic in both directions at once (H2D + D2H copy-engine copies on two
// streams), against each direction alone.  Pinned (cudaHostAlloc) buffers, 256 MiB each way.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)
int main() {
  CK(cudaSetDevice(0));
  const size_t n = 256ull << 20;
  void *hi, *ho, *di, *dout;
  CK(cudaHostAlloc(&hi, n, 0)); CK(cudaHostAlloc(&ho, n, 0));
  CK(cudaMalloc(&di, n)); CK(cudaMalloc(&dout, n));
  cudaStream_t s1, s2; CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c, d; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&c)); CK(cudaEventCreate(&d));
  float ms, ms2;
  for (size_t chunk : {size_t(n), size_t(1) << 20}) {
    float h2d = 1e9, d2h = 1e9, both = 1e9, bh = 0, bd = 0;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(a, s1));
      for (size_t o = 0; o < n; o += chunk) CK(cudaMemcpyAsync((char*)di + o, (char*)hi + o, chunk, cudaMemcpyHostToDevice, s1));
      CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); if (ms < h2d) h2d = ms;
      CK(cudaEventRecord(a, s2));
      for (size_t o = 0; o < n; o += chunk) CK(cudaMemcpyAsync((char*)ho + o, (char*)dout + o, chunk, cudaMemcpyDeviceToHost, s2));
      CK(cudaEventRecord(b, s2)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b)); if (ms < d2h) d2h = ms;
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1)); CK(cudaStreamWaitEvent(s2, a));
      for (size_t o = 0; o < n; o += chunk) {
        CK(cudaMemcpyAsync((char*)di + o, (char*)hi + o, chunk, cudaMemcpyHostToDevice, s1));
        CK(cudaMemcpyAsync((char*)ho + o, (char*)dout + o, chunk, cudaMemcpyDeviceToHost, s2));
      }
      CK(cudaEventRecord(b, s1)); CK(cudaEventRecord(c, s2));
      CK(cudaEventSynchronize(b)); CK(cudaEventSynchronize(c));
      CK(cudaEventElapsedTime(&ms, a, b)); CK(cudaEventElapsedTime(&ms2, a, c));
      float m = ms > ms2 ? ms : ms2;
      if (m < both) { both = m; bh = ms; bd = ms2; }
    }
    printf("chunk %zu KiB: H2D alone %.2f GB/s, D2H alone %.2f GB/s; both at once: H2D %.2f GB/s, D2H %.2f GB/s (%.3f ms vs %.3f + %.3f)\n",
           chunk >> 10, n / h2d / 1e6, n / d2h / 1e6, n / bh / 1e6, n / bd / 1e6, both, h2d, d2h);
  }
  return 0;
}
