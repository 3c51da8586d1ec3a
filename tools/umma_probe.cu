// Probe: tcgen05.mma throughput on this B200 for the MMA shapes the suffix attention issues,
// one CTA per SM, no softmax, no TMA (operands resident in smem / TMEM):
//   SS N=64/128/256 (QK^T with Q and K in smem), TS (A from TMEM) N=64 K-major and N=128 MN-major
//   (PV with P in TMEM), and the attention's per-key-tile MMA mixes.  The answer decides whether a
//   64-key QK^T with Q re-read from smem every tile is shared-memory-operand bound.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_23049_b200/csrc/kernels tools/umma_probe.cu -o tools/umma_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

using namespace pcr::ptx;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}

constexpr int kQ = 0, kK = 65536, kV = 131072, kBar = 196608, kSmem = kBar + 128 + 1024;

// One Q tile (128 x 128 bf16, two 64-column SW128 halves of 16 KB) at q; keys x 128 K tile at k.
__device__ __forceinline__ void qk_ss(uint32_t d, uint64_t qd, uint64_t kd, int n, int halfk, uint32_t idesc) {
  for (int kk = 0; kk < 8; ++kk)
    mma_bf16_ss(d, qd + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), kd + (((kk >> 2) * halfk + (kk & 3) * 32) >> 4),
                idesc, kk > 0);
}
__device__ __forceinline__ void qk_ts(uint32_t d, uint32_t qt, uint64_t kd, int halfk, uint32_t idesc) {
  for (int kk = 0; kk < 8; ++kk)
    mma_ts(d, qt + kk * 8, kd + (((kk >> 2) * halfk + (kk & 3) * 32) >> 4), idesc, kk > 0);
}
__device__ __forceinline__ void pv_ts(uint32_t d, uint32_t pt, uint64_t vd, int keys, uint32_t idesc) {
  for (int kk = 0; kk < keys / 16; ++kk) mma_ts(d, pt + kk * 8, vd + (kk * 2048 >> 4), idesc, 1);
}

__device__ __forceinline__ void spin(int units) {
  if (units == 0) return;
  const long long t0 = clock64();
  while (clock64() - t0 < 150LL * units) {
  }
}

template <int MODE>
__global__ void __launch_bounds__(384, 1) probe(int iters, float* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(smem + kBar + 64);
  for (int i = threadIdx.x; i < kBar / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;  // bf16 2^-7 pairs
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { for (int b = 0; b < 6; ++b) mbar_init(bar + b, 1 + (b == 4 ? 0 : 0)); fence_mbar_init(); mbar_arrive(bar + 5); }
  if (threadIdx.x < 32) tmem_alloc<512>(tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tbase;
  if (MODE >= 30 && threadIdx.x >= 128) {  // 8 extra warps polling an mbarrier until the issuer is done
    if (MODE == 30) mbar_wait(bar + 4, 0);
    if (MODE == 31) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar + 4)), "r"(0), "r"(1000000) : "memory");
    }
  }
  if (threadIdx.x < 32) {
    const uint64_t qd = smem_desc_sw128(smem_u32(smem + kQ), 16, 1024);
    const uint64_t kd = smem_desc_sw128(smem_u32(smem + kK), 16, 1024);
    const uint64_t vd64 = smem_desc_sw128(smem_u32(smem + kV), 64 * 128, 1024);
    const uint64_t vd128 = smem_desc_sw128(smem_u32(smem + kV), 128 * 128, 1024);
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
        if (MODE == 0) qk_ss(tm, qd, kd, 64, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
        if (MODE == 1) qk_ss(tm, qd, kd, 128, 128 * 128, idesc_bf16_f32(128, 128, 0, 0));
        if (MODE == 2) qk_ss(tm, qd, kd, 256, 256 * 128, idesc_bf16_f32(128, 256, 0, 0));
        if (MODE == 3) qk_ts(tm, tm + 128, kd, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
        if (MODE == 4) pv_ts(tm + 256, tm, vd64, 64, idesc_bf16_f32(128, 128, 0, 1));
        if (MODE == 5) {  // current kernel: per 64-key tile, 2 Q tiles: QK^T SS N=64, PV TS N=128 K=64
          for (int t = 0; t < 2; ++t) qk_ss(tm + t * 64, qd + (t * 32768 >> 4), kd, 64, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
          for (int t = 0; t < 2; ++t) pv_ts(tm + 256 + t * 128, tm + t * 64, vd64, 64, idesc_bf16_f32(128, 128, 0, 1));
        }
        if (MODE == 6) {  // Q in TMEM: QK^T TS N=64
          for (int t = 0; t < 2; ++t) qk_ts(tm + t * 64, tm + 128 + t * 64, kd, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
          for (int t = 0; t < 2; ++t) pv_ts(tm + 256 + t * 128, tm + t * 64, vd64, 64, idesc_bf16_f32(128, 128, 0, 1));
        }
        if (MODE == 7) {  // 128-key tiles, QK^T SS N=128, PV TS K=128
          for (int t = 0; t < 2; ++t) qk_ss(tm + t * 128, qd + (t * 32768 >> 4), kd, 128, 128 * 128, idesc_bf16_f32(128, 128, 0, 0));
          for (int t = 0; t < 2; ++t) pv_ts(tm + 256 + t * 128, tm + t * 128, vd128, 128, idesc_bf16_f32(128, 128, 0, 1));
        }
        if (MODE >= 10 && MODE <= 15) {  // mix 64-key SS with (MODE-10) tcgen05.commit per iteration
          for (int t = 0; t < 2; ++t) {
            pv_ts(tm + 256 + t * 128, tm + t * 64, vd64, 64, idesc_bf16_f32(128, 128, 0, 1));
            if (MODE - 10 >= 2 + t) mma_commit(bar + 1 + t);
          }
          if (MODE - 10 >= 5) mma_commit(bar + 3);
          for (int t = 0; t < 2; ++t) {
            qk_ss(tm + t * 64, qd + (t * 32768 >> 4), kd, 64, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
            if (MODE - 10 >= 1 + 3 * t) mma_commit(bar + 4 + t);
          }
        }
        if (MODE >= 20 && MODE <= 24) {  // mix 64-key SS with a busy gap of (MODE-20)*150 clk between groups
          for (int t = 0; t < 2; ++t) {
            pv_ts(tm + 256 + t * 128, tm + t * 64, vd64, 64, idesc_bf16_f32(128, 128, 0, 1));
            spin(MODE - 20);
          }
          for (int t = 0; t < 2; ++t) {
            qk_ss(tm + t * 64, qd + (t * 32768 >> 4), kd, 64, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
            spin(MODE - 20);
          }
        }
        if (MODE == 25 || MODE == 26) {  // the kernel's pattern: 4 K/V stages, S buffers (2t + it&1), order PV_t, S_t(it+2)
          const int st = it & 3, b = it & 1;
          const uint64_t kds = smem_desc_sw128(smem_u32(smem + kK + st * 16384), 16, 1024);
          const uint64_t vds = smem_desc_sw128(smem_u32(smem + kK + 65536 + st * 16384), 64 * 128, 1024);
          for (int t = 0; t < 2; ++t) {
            pv_ts(tm + 256 + t * 128, tm + (2 * t + b) * 64, vds, 64, idesc_bf16_f32(128, 128, 0, 1));
            if (MODE == 26) mma_commit(bar + 1 + t);
            qk_ss(tm + (2 * t + b) * 64, qd + (t * 32768 >> 4), kds, 64, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
            if (MODE == 26) mma_commit(bar + 3 + t);
          }
        }
        if ((MODE >= 27 && MODE <= 29) || MODE >= 30) {  // kernel pattern with, between groups: 27 fence::after_thread_sync,
                                          // 28 wait on a completed mbarrier + fence, 29 wait only
          const int st = it & 3, b = it & 1;
          const uint64_t kds = smem_desc_sw128(smem_u32(smem + kK + st * 16384), 16, 1024);
          const uint64_t vds = smem_desc_sw128(smem_u32(smem + kK + 65536 + st * 16384), 64 * 128, 1024);
          for (int t = 0; t < 2; ++t) {
            if (MODE >= 28) mbar_wait(bar + 5, 0);
            if (MODE <= 28 || MODE >= 30) tc_fence_after();
            pv_ts(tm + 256 + t * 128, tm + (2 * t + b) * 64, vds, 64, idesc_bf16_f32(128, 128, 0, 1));
            if (MODE >= 28) mbar_wait(bar + 5, 0);
            if (MODE <= 28 || MODE >= 30) tc_fence_after();
            qk_ss(tm + (2 * t + b) * 64, qd + (t * 32768 >> 4), kds, 64, 64 * 128, idesc_bf16_f32(128, 64, 0, 0));
          }
        }
        if (MODE == 8) {  // 128-key tiles with Q in TMEM would need 768 columns: N=128 QK^T TS only
          for (int t = 0; t < 2; ++t) qk_ts(tm + t * 128, tm + 256 + t * 64, kd, 128 * 128, idesc_bf16_f32(128, 128, 0, 0));
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(bar);
    __syncwarp();
    if (MODE >= 30 && elect_one()) mbar_arrive(bar + 4);
    mbar_wait(bar, 0);
    tc_fence_after();
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float v[32];
    tmem_ld32(tm + (uint32_t((threadIdx.x & 31) * 0) << 16), v);
    tmem_ld_wait();
    if (v[0] == 12345.f) sink[0] = v[1];
    tmem_dealloc<512>(tm);
  }
}

template <int MODE>
void run(const char* name, double flop_per_iter) {
  auto k = probe<MODE>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  float* sink; CK(cudaMalloc(&sink, 4));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int iters = 4000;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  const int thr = MODE >= 30 ? 384 : 128;
  k<<<sms, thr, kSmem>>>(100, sink);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a));
    k<<<sms, thr, kSmem>>>(iters, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  CK(cudaGetLastError());
  const double tf = flop_per_iter * iters * sms / (best * 1e-3) / 1e12;
  printf("{\"mode\": %d, \"name\": \"%s\", \"ms\": %.3f, \"tflops\": %.1f}\n", MODE, name, best, tf);
  fflush(stdout);
  cudaFree(sink);
}

int main() {
  const double qk64 = 2.0 * 128 * 64 * 128, qk128 = 2 * qk64, qk256 = 4 * qk64, pv64 = 2.0 * 128 * 128 * 64;
  run<0>("SS M128 N64 K128 (QK^T, 64 keys)", qk64);
  run<1>("SS M128 N128 K128 (QK^T, 128 keys)", qk128);
  run<2>("SS M128 N256 K128", qk256);
  run<3>("TS M128 N64 K128 (QK^T, Q in TMEM)", qk64);
  run<4>("TS M128 N128 K64 MN-major B (PV, 64 keys)", pv64);
  run<5>("mix 64-key: 2x QK SS + 2x PV TS", 2 * (qk64 + pv64));
  run<6>("mix 64-key, Q in TMEM: 2x QK TS + 2x PV TS", 2 * (qk64 + pv64));
  run<7>("mix 128-key: 2x QK SS N128 + 2x PV TS K128", 2 * (qk128 + 2 * pv64));
  run<8>("TS M128 N128 K128 (QK^T, Q in TMEM, 128 keys)", 2 * qk128);
  run<10>("mix 64-key SS, 0 commits / iteration", 2 * (qk64 + pv64));
  run<11>("mix 64-key SS, 1 commit / iteration", 2 * (qk64 + pv64));
  run<12>("mix 64-key SS, 2 commits / iteration", 2 * (qk64 + pv64));
  run<20>("mix 64-key SS, no gap", 2 * (qk64 + pv64));
  run<21>("mix 64-key SS, 150 clk gap after each group", 2 * (qk64 + pv64));
  run<22>("mix 64-key SS, 300 clk gap after each group", 2 * (qk64 + pv64));
  run<23>("mix 64-key SS, 450 clk gap after each group", 2 * (qk64 + pv64));
  run<24>("mix 64-key SS, 600 clk gap after each group", 2 * (qk64 + pv64));
  run<25>("kernel pattern: 4 stages, S double buffer, PV_t then S_t", 2 * (qk64 + pv64));
  run<26>("kernel pattern + 4 commits / iteration", 2 * (qk64 + pv64));
  run<27>("kernel pattern + tcgen05.fence::after_thread_sync between groups", 2 * (qk64 + pv64));
  run<28>("kernel pattern + completed-mbarrier wait + fence between groups", 2 * (qk64 + pv64));
  run<29>("kernel pattern + completed-mbarrier wait between groups", 2 * (qk64 + pv64));
  run<30>("kernel pattern + waits, 8 warps spinning on an mbarrier (try_wait)", 2 * (qk64 + pv64));
  run<31>("kernel pattern + waits, 8 warps polling with a suspend-time hint", 2 * (qk64 + pv64));
  run<15>("mix 64-key SS, 5 commits / iteration", 2 * (qk64 + pv64));
  return 0;
}
