// Probe: does a CTA pair (tcgen05 cta_group::2, M = 256 across two SMs) lift the attention's MMA
// mix above the single-CTA 64-key ceiling (QK^T SS at M128 N64 is shared-memory-operand bound)?
// Each SM still computes 128 rows; B (K or V) is split across the pair, halving its smem reads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_23049_b200/csrc/kernels tools/umma2_probe.cu -o tools/umma2_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

using namespace pcr::ptx;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kQ = 0, kK = 65536, kV = 98304, kBar = 131072, kSmem = kBar + 128 + 1024;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"(uint16_t(3)) : "memory");
}

// MODE 0: QK^T only, 64 keys (N = 64 across the pair: 32 key rows per CTA)
// MODE 1: the attention's 64-key mix per Q-tile pair: 2 x QK^T (N 64) + 2 x PV (N = d 128, 64 per CTA)
// MODE 2: QK^T only, 128 keys
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe2(int iters, float* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + kBar + 64);
  for (int i = threadIdx.x; i < kBar / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tbase)), "r"(512));
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = *tbase;
  const uint32_t rank = cta_rank();
  if (rank == 0 && threadIdx.x < 32) {
    const uint64_t qd = smem_desc_sw128(smem_u32(smem + kQ), 16, 1024);
    const uint64_t kd = smem_desc_sw128(smem_u32(smem + kK), 16, 1024);
    const uint64_t vd = smem_desc_sw128(smem_u32(smem + kV), 8192, 1024);
    const uint32_t id_qk64 = idesc_bf16_f32(256, 64, 0, 0), id_qk128 = idesc_bf16_f32(256, 128, 0, 0);
    const uint32_t id_pv = idesc_bf16_f32(256, 128, 0, 1);
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
        const int half_k = (MODE == 2 ? 64 : 32) * 128;  // bytes of one 64-column half of this CTA's K rows
        for (int t = 0; t < 2; ++t) {
          if (MODE != 2) {
            if (MODE == 1)
              for (int kk = 0; kk < 4; ++kk)  // PV_t: A = P_t in TMEM, K = 64 keys
                mma2_ts(tm + 256 + t * 128, tm + t * 64 + kk * 8, vd + (kk * 2048 >> 4), id_pv, 1);
            for (int kk = 0; kk < 8; ++kk)
              mma2_ss(tm + t * 64, qd + ((t * 32768 + (kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                      kd + (((kk >> 2) * half_k + (kk & 3) * 32) >> 4), id_qk64, kk > 0);
          } else {
            for (int kk = 0; kk < 8; ++kk)
              mma2_ss(tm + t * 128, qd + ((t * 32768 + (kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                      kd + (((kk >> 2) * half_k + (kk & 3) * 32) >> 4), id_qk128, kk > 0);
          }
        }
      }
      __syncwarp();
    }
    if (elect_one()) commit2_mc(bar);
    __syncwarp();
  }
  if (threadIdx.x < 32) {
    mbar_wait(bar, 0);
    tc_fence_after();
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float v[32];
    tmem_ld32(tm, v);
    tmem_ld_wait();
    if (v[0] == 12345.f) sink[0] = v[1];
  }
  tc_fence_before();
  cluster_sync();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
}

template <int MODE>
void run(const char* name, double flop_per_iter_per_pair) {
  auto k = probe2<MODE>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  float* sink; CK(cudaMalloc(&sink, 4));
  const int iters = 4000, ctas = 148;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  k<<<ctas, 128, kSmem>>>(50, sink);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a));
    k<<<ctas, 128, kSmem>>>(iters, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  CK(cudaGetLastError());
  const double tf = flop_per_iter_per_pair * iters * (ctas / 2) / (best * 1e-3) / 1e12;
  printf("{\"mode\": %d, \"name\": \"%s\", \"ms\": %.3f, \"tflops\": %.1f}\n", MODE, name, best, tf);
  fflush(stdout);
  cudaFree(sink);
}

int main() {
  const double qk = 2.0 * 256 * 64 * 128, pv = 2.0 * 256 * 128 * 64;
  run<0>("cta_group::2 QK^T SS M256 N64 K128 x2 tiles", 2 * qk);
  run<1>("cta_group::2 64-key mix: 2x QK SS + 2x PV TS", 2 * (qk + pv));
  run<2>("cta_group::2 QK^T SS M256 N128 K128 x2 tiles", 2 * 2 * qk);
  return 0;
}
