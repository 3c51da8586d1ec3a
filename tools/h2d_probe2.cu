// Probe: SM zero-copy host->HBM variants (does the request shape change the host-link efficiency?).
// r01 measured a flat 51.2 GB/s for 16-byte ld.global.cs at any grid/unroll against 55.6 GB/s for
// the copy engine (profiles/r01_box_probe.txt).  Variants here: L2 prefetch-size qualifiers on the
// load (.L2::128B / .L2::256B), 32-byte vector loads (ld.global.v8.b32, sm_100), TMA bulk copies
// host -> smem in 4/16 KiB pieces, and an L2 bulk prefetch of the source ahead of the loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/h2d_probe2 tools/h2d_probe2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e = (x);                                                                \
    if (e != cudaSuccess) {                                                             \
      printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e));              \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

template <int V>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 v;
  if (V == 0)
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (V == 1)
    asm volatile("ld.global.cs.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (V == 2)
    asm volatile("ld.global.cs.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// warp-contiguous: warp w copies a contiguous 16 KiB segment (like kv_gather's page segments)
template <int V, int U>
__global__ void __launch_bounds__(256) seg_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16,
                                                int seg16) {
  const int lane = threadIdx.x & 31;
  const int64_t n_seg = n16 / seg16;
  const int64_t warps = int64_t(gridDim.x) * 8;
  for (int64_t s = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); s < n_seg; s += warps) {
    const uint4* a = src + s * seg16;
    uint4* b = dst + s * seg16;
    for (int base = lane; base < seg16; base += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld16<V>(a + base + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) b[base + 32 * u] = v[u];
    }
  }
}

// 32-byte vectors per lane
template <int U>
__global__ void __launch_bounds__(256) seg_copy32(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16,
                                                  int seg16) {
  const int lane = threadIdx.x & 31;
  const int64_t n_seg = n16 / seg16;
  const int64_t warps = int64_t(gridDim.x) * 8;
  for (int64_t s = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); s < n_seg; s += warps) {
    const uint4* a = src + s * seg16;
    uint4* b = dst + s * seg16;
    for (int base = 2 * lane; base < seg16; base += 64 * U) {
      uint32_t r[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]),
                       "=r"(r[u][6]), "=r"(r[u][7])
                     : "l"(a + base + 64 * u));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        b[base + 64 * u] = make_uint4(r[u][0], r[u][1], r[u][2], r[u][3]);
        b[base + 64 * u + 1] = make_uint4(r[u][4], r[u][5], r[u][6], r[u][7]);
      }
    }
  }
}

// L2 bulk prefetch of the next segments (cp.async.bulk.prefetch.L2) ahead of plain 16-byte loads
template <int U>
__global__ void __launch_bounds__(256) seg_copy_pf(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16,
                                                   int seg16) {
  const int lane = threadIdx.x & 31;
  const int64_t n_seg = n16 / seg16;
  const int64_t warps = int64_t(gridDim.x) * 8;
  for (int64_t s = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); s < n_seg; s += warps) {
    const uint4* a = src + s * seg16;
    uint4* b = dst + s * seg16;
    if (lane == 0 && s + warps < n_seg)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (s + warps) * seg16), "r"(seg16 * 16)
                   : "memory");
    for (int base = lane; base < seg16; base += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld16<0>(a + base + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) b[base + 32 * u] = v[u];
    }
  }
}

// TMA bulk: one elected thread per CTA streams pieces host -> smem -> HBM (2 stages)
template <int PIECE>
__global__ void __launch_bounds__(32) tma_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                               int64_t bytes) {
  __shared__ __align__(128) uint8_t buf[2][PIECE];
  __shared__ __align__(8) uint64_t full[2];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 2; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&full[s]))));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[2] = {0, 0};
  const int64_t n = bytes / PIECE;
  int it = 0;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x, ++it) {
    const int st = it & 1;
    const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(buf[st]));
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&full[st]));
    if (it >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(PIECE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb),
                 "l"(src + i * PIECE), "r"(PIECE), "r"(bar)
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar),
        "r"(phase[st])
        : "memory");
    phase[st] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + i * PIECE), "r"(sb), "r"(PIECE)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  CK(cudaSetDevice(0));
  const size_t bytes = 256ull << 20;
  void* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  memset(h, 1, bytes);
  void* d;
  CK(cudaMalloc(&d, bytes));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time = [&](const char* name, auto&& launch) {
    float best = 1e9, ms;
    for (int i = 0; i < 6; ++i) {
      CK(cudaEventRecord(a, s));
      launch();
      CK(cudaGetLastError());
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    printf("%-48s %7.2f GB/s\n", name, bytes / best / 1e6);
  };
  time("CE cudaMemcpyAsync 256 MiB", [&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s)); });
  const int64_t n16 = bytes / 16;
  const int seg16 = 1024;  // 16 KiB segments
  for (int g : {16, 32}) {
    char nm[96];
    snprintf(nm, sizeof nm, "16B .cs            grid %d u4", g);
    time(nm, [&] { seg_copy<0, 4><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
    snprintf(nm, sizeof nm, "16B .cs.L2::128B   grid %d u4", g);
    time(nm, [&] { seg_copy<1, 4><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
    snprintf(nm, sizeof nm, "16B .cs.L2::256B   grid %d u4", g);
    time(nm, [&] { seg_copy<2, 4><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
    snprintf(nm, sizeof nm, "16B .nc.L2::256B   grid %d u4", g);
    time(nm, [&] { seg_copy<3, 4><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
    snprintf(nm, sizeof nm, "16B .cs.L2::256B   grid %d u8", g);
    time(nm, [&] { seg_copy<2, 8><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
    snprintf(nm, sizeof nm, "32B v8.b32         grid %d u2", g);
    time(nm, [&] { seg_copy32<2><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
    snprintf(nm, sizeof nm, "32B v8.b32         grid %d u4", g);
    time(nm, [&] { seg_copy32<4><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
    snprintf(nm, sizeof nm, "16B + bulk L2 prefetch grid %d u4", g);
    time(nm, [&] { seg_copy_pf<4><<<g, 256, 0, s>>>((const uint4*)h, (uint4*)d, n16, seg16); });
  }
  for (int g : {16, 64, 148}) {
    char nm[96];
    snprintf(nm, sizeof nm, "TMA bulk 4 KiB pieces  grid %d", g);
    time(nm, [&] { tma_copy<4096><<<g, 32, 0, s>>>((const uint8_t*)h, (uint8_t*)d, bytes); });
    snprintf(nm, sizeof nm, "TMA bulk 16 KiB pieces grid %d", g);
    time(nm, [&] { tma_copy<16384><<<g, 32, 0, s>>>((const uint8_t*)h, (uint8_t*)d, bytes); });
  }
  return 0;
}
