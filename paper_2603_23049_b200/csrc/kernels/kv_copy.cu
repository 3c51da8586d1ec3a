// a2 kv_gather (host store -> HBM pool) and a3 kv_append (suffix K/V -> pool).
//
// the paper copies a CPU chunk into many non-consecutive GPU blocks with a batched
// copy-engine API.  On B200 the copy is an SM kernel instead:
// every thread streams 16-byte vectors straight out of the mapped pinned host store over PCIe
// Gen5 (zero-copy, ld.global.cs) and writes them, 16 bytes at a time, into the pool pages of
// the request.  The same launch can also carry a few linear host->device copies (the layer's
// q/k/v inputs on the host_io path), so one kernel per layer moves everything the layer needs.
// Measured on this pool's B200 (tools/h2d_probe.cu): 8+ CTAs x 256 threads with 4 loads in
// flight per thread reach 51.2 GB/s = 92% of the copy engine's 55.6 GB/s, so the gather needs
// only a handful of SMs and leaves the rest to the concurrent attention.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace pcr {
namespace {

// 256 threads x <= 40 registers (10K registers, no shared memory) lets a gather CTA co-reside
// with an attention CTA (256 threads, ~47K registers, ~195 KB smem) on the same SM, so loads of
// layer l+1 are never queued behind the attention grid of layer l.
constexpr int kThreads = 256;
constexpr int kUnroll = 4;
// The gather keeps 4 loads of 16 bytes in flight per lane: 128 KiB for the default 8 CTAs, about
// the host link's bandwidth-latency product (~51 GB/s x ~2.5 us); 8 unrolled loads need more than
// the 40 registers that let a gather CTA share an SM with an attention CTA (they spill).
constexpr int kGatherUnroll = 4;

__device__ __forceinline__ uint4 ld_host_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// The copy is a list of page segments.  A store slot is laid out page-major, as the pool pages it
// fills: [L][C/S][Hkv][2][S][d], so for chunk c (chain index) and page pp of the chunk, layer l
// of the slot holds one Hkv*2*S*d*2-byte image of pool page pages[c*C/S + pp].  A segment is one
// (chunk, page of the chunk, kv head, K|V): S*d*2 contiguous bytes on both sides.  Consecutive
// segments are consecutive in the store.  Each warp copies whole segments (address math once per
// segment, not per 16 bytes), every lane keeping kUnroll independent 16-byte loads in flight;
// grid-stride over segments.
__device__ __forceinline__ void segment_addrs(int64_t seg, int32_t chunk0, int32_t layer, const KvGeom& g,
                                              int32_t ppc_log2, int32_t row16_log2, const int32_t* slots,
                                              const int32_t* pages, int64_t& store16, int64_t& pool16) {
  const int64_t hk2 = int64_t(g.Hkv) * 2;
  const int64_t hk = seg % hk2;                                           // h*2 + kv
  const int64_t cp = seg / hk2;                                           // chunk-local page index
  const int32_t pp = int32_t(cp & ((1 << ppc_log2) - 1));
  const int32_t c = chunk0 + int32_t(cp >> ppc_log2);
  const int64_t seg16 = int64_t(g.S) << row16_log2;                       // 16-byte units per segment
  const int64_t page16 = hk2 * seg16;                                     // one page image
  store16 = int64_t(slots[c]) * (g.slot_elems / 8) + ((int64_t(layer) << ppc_log2) + pp) * page16 + hk * seg16;
  const int64_t page = pages[(int64_t(c) << ppc_log2) + pp];
  pool16 = (int64_t(layer) * g.n_pool_pages + page) * page16 + hk * seg16;
}

// Segments [0, n_lin_seg) are pieces of the linear copies (each copy cut into seg16-unit pieces,
// the last one ragged), the rest are page segments.  The linear copies come first: the layer's
// inputs are needed by the attention as soon as its KV has landed.  Warp `warp` of `warps` takes
// segments warp, warp + warps, ...
__device__ __forceinline__ void gather_layer(const uint4* __restrict__ store, uint4* __restrict__ pool,
                                             const int32_t* __restrict__ slots, const int32_t* __restrict__ pages,
                                             int32_t n_chunks, int32_t layer, const KvGeom& g, int32_t row16_log2,
                                             int32_t ppc_log2, const LinearCopies& lin, int64_t warp, int64_t warps,
                                             int lane) {
  const int32_t seg16 = g.S << row16_log2;
  static_assert(LinearCopies::kMax == 3, "segment prefix below");
  const int64_t e1 = lin.n > 0 ? (lin.n16[0] + seg16 - 1) / seg16 : 0;
  const int64_t e2 = e1 + (lin.n > 1 ? (lin.n16[1] + seg16 - 1) / seg16 : 0);
  const int64_t n_lin = e2 + (lin.n > 2 ? (lin.n16[2] + seg16 - 1) / seg16 : 0);
  const int64_t n_seg = n_lin + ((int64_t(n_chunks) * g.Hkv * 2) << ppc_log2);
  for (int64_t seg = warp; seg < n_seg; seg += warps) {
    const uint4* src;
    uint4* dst;
    int64_t len16 = seg16;
    if (seg < n_lin) {
      const bool c1 = seg >= e1, c2 = seg >= e2;
      const int i = c2 ? 2 : c1 ? 1 : 0;
      const int64_t off = (seg - (c2 ? e2 : c1 ? e1 : 0)) * seg16;
      src = lin.src[i] + lin.src_stride16[i] * layer + off;
      dst = lin.dst[i] + lin.dst_stride16[i] * layer + off;
      len16 = min(int64_t(seg16), lin.n16[i] - off);
    } else {
      int64_t s16, p16;
      segment_addrs(seg - n_lin, 0, layer, g, ppc_log2, row16_log2, slots, pages, s16, p16);
      src = store + s16;
      dst = pool + p16;
    }
    for (int64_t base = lane; base < len16; base += 32 * kGatherUnroll) {
      uint4 v[kGatherUnroll];
#pragma unroll
      for (int u = 0; u < kGatherUnroll; ++u)
        if (base + 32 * u < len16) v[u] = ld_host_stream(src + base + 32 * u);
#pragma unroll
      for (int u = 0; u < kGatherUnroll; ++u)
        if (base + 32 * u < len16) dst[base + 32 * u] = v[u];
    }
  }
}

__global__ void __launch_bounds__(kThreads, 6) kv_gather_kernel(const uint4* __restrict__ store,
                                                             uint4* __restrict__ pool,
                                                             const int32_t* __restrict__ slots,
                                                             const int32_t* __restrict__ pages, int32_t n_chunks,
                                                             int32_t layer, KvGeom g, int32_t row16_log2,
                                                             int32_t ppc_log2, LinearCopies lin) {
  gather_layer(store, pool, slots, pages, n_chunks, layer, g, row16_log2, ppc_log2, lin,
               int64_t(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5), int64_t(gridDim.x) * (kThreads / 32),
               threadIdx.x & 31);
}

// Streamed gather (one launch per request): every layer in order.  A warp that has copied its
// share of layer l publishes it -- release add on ready[l] (cumulative over the warp's lanes
// through __syncwarp) -- and moves on to layer l+1 without waiting for the other warps; layer l
// is in the pool once ready[l] counts every warp of the grid (the attention of layer l waits for
// that with an acquire load, suffix_attn.cu).
__global__ void __launch_bounds__(kThreads, 6) kv_gather_stream_kernel(
    const uint4* __restrict__ store, uint4* __restrict__ pool, const int32_t* __restrict__ slots,
    const int32_t* __restrict__ pages, int32_t n_chunks, int32_t n_layers, KvGeom g, int32_t row16_log2,
    int32_t ppc_log2, LinearCopies lin, int32_t* __restrict__ ready) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = int64_t(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5);
  const int64_t warps = int64_t(gridDim.x) * (kThreads / 32);
  for (int32_t layer = 0; layer < n_layers; ++layer) {
    gather_layer(store, pool, slots, pages, n_chunks, layer, g, row16_log2, ppc_log2, lin, warp, warps, lane);
    __syncwarp();
    if (lane == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ready + layer) : "memory");
  }
}

// One 16-byte unit per thread-iteration over [n2][Hkv][d/8] for K and V, then the tail rows.
__global__ void kv_append_kernel(const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                                 uint4* __restrict__ pool, const int32_t* __restrict__ pages, int64_t n1,
                                 int64_t n2, int32_t n_req_pages, int32_t layer, KvGeom g, int32_t row16_log2,
                                 int32_t S_log2) {
  ptx::grid_dep_launch();   // PDL: the attention after this append may start its prologue now
  const int64_t row16 = int64_t(1) << row16_log2;
  const int64_t page16 = int64_t(g.Hkv) * 2 * g.S * row16;
  uint4* dst_layer = pool + int64_t(layer) * g.n_pool_pages * page16;
  const int64_t per_tok = int64_t(g.Hkv) * row16;
  const int64_t n_units = n2 * per_tok;
  const int64_t total_rows = int64_t(n_req_pages) * g.S;
  const int64_t tail_units = (total_rows - (n1 + n2)) * per_tok;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n_units + tail_units; u += stride) {
    const bool tail = u >= n_units;
    const int64_t uu = tail ? u - n_units : u;
    const int64_t i = uu / per_tok;
    const int64_t rem = uu - i * per_tok;
    const int64_t h = rem >> row16_log2;
    const int64_t col = rem & (row16 - 1);
    const int64_t t = n1 + n2 * tail + i;  // tail rows start at n1+n2
    const int64_t page = pages[t >> S_log2];
    uint4* dk = dst_layer + page * page16 + (((h * 2 + 0) << S_log2) + (t & (g.S - 1))) * row16 + col;
    uint4* dv = dst_layer + page * page16 + (((h * 2 + 1) << S_log2) + (t & (g.S - 1))) * row16 + col;
    if (tail) {
      *dk = make_uint4(0, 0, 0, 0);
      *dv = make_uint4(0, 0, 0, 0);
    } else {
      *dk = k_new[uu];
      *dv = v_new[uu];
    }
  }
}

// f1 offload (the inverse of the gather): layer `layer` of every reserved chunk, pool pages ->
// pinned host store slot, 16-byte loads from HBM and 16-byte stores over PCIe into the mapped
// store, page segment by page segment (see kv_gather_kernel).
__global__ void __launch_bounds__(kThreads, 6) kv_scatter_kernel(const uint4* __restrict__ pool,
                                                              uint4* __restrict__ store,
                                                              const int32_t* __restrict__ slots,
                                                              const int32_t* __restrict__ pages, int32_t chunk0,
                                                              int32_t n_chunks, int32_t layer, KvGeom g,
                                                              int32_t row16_log2, int32_t ppc_log2) {
  const int lane = threadIdx.x & 31;
  const int64_t n_seg = (int64_t(n_chunks) * g.Hkv * 2) << ppc_log2;
  const int32_t seg16 = g.S << row16_log2;
  const int64_t warps = int64_t(gridDim.x) * (kThreads / 32);
  for (int64_t seg = int64_t(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5); seg < n_seg; seg += warps) {
    int64_t s16, p16;
    segment_addrs(seg, chunk0, layer, g, ppc_log2, row16_log2, slots, pages, s16, p16);
    const uint4* src = pool + p16;
    uint4* dst = store + s16;
    for (int32_t base = lane; base < seg16; base += 32 * kUnroll) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (base + 32 * u < seg16) v[u] = src[base + 32 * u];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (base + 32 * u < seg16) dst[base + 32 * u] = v[u];
    }
  }
}

// load_mode 3 experiment: the same page segments moved with the Tensor Memory Accelerator's
// bulk copies instead of 16-byte thread loads: host store --cp.async.bulk--> smem --cp.async.bulk-->
// pool page.  One elected thread per CTA keeps kStages segments in flight.
constexpr int kTmaStages = 2;
constexpr int kTmaSegMax = 16384;  // bytes per segment buffer (S_pg * d * 2 <= 16 KB)

__global__ void __launch_bounds__(32) kv_gather_tma_kernel(const uint8_t* __restrict__ store, uint8_t* __restrict__ pool,
                                                          const int32_t* __restrict__ slots,
                                                          const int32_t* __restrict__ pages, int32_t n_matched,
                                                          int32_t layer, KvGeom g) {
  __shared__ __align__(128) uint8_t buf[kTmaStages][kTmaSegMax];
  __shared__ __align__(8) uint64_t full[kTmaStages];
  if (threadIdx.x != 0) return;
  const int64_t seg = int64_t(g.S) * g.d * 2;
  const int32_t ppc = g.C / g.S;
  const int64_t n_seg = int64_t(n_matched) * g.Hkv * 2 * ppc;
  for (int s = 0; s < kTmaStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&full[s]))));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[kTmaStages] = {0};
  int it = 0;
  for (int64_t i = blockIdx.x; i < n_seg; i += gridDim.x, ++it) {
    const int st = it % kTmaStages;
    const uint32_t sbuf = static_cast<uint32_t>(__cvta_generic_to_shared(buf[st]));
    const uint32_t sbar = static_cast<uint32_t>(__cvta_generic_to_shared(&full[st]));
    if (it >= kTmaStages)  // the store that last read this buffer must have finished reading it
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaStages - 1) : "memory");
    // segment i -> (chunk, page-in-chunk, h, kv), page-major slot layout (see segment_addrs)
    const int64_t hk = i % (g.Hkv * 2);
    const int32_t pp = int32_t((i / (g.Hkv * 2)) % ppc);
    const int32_t c = int32_t(i / (ppc * g.Hkv * 2));
    const int64_t page_bytes = int64_t(g.Hkv) * 2 * seg;
    const uint8_t* src = store + int64_t(slots[c]) * g.slot_elems * 2 + (int64_t(layer) * ppc + pp) * page_bytes + hk * seg;
    const int64_t page = pages[c * ppc + pp];
    uint8_t* dst = pool + (int64_t(layer) * g.n_pool_pages + page) * page_bytes + hk * seg;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(uint32_t(seg)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sbuf),
                 "l"(src), "r"(uint32_t(seg)), "r"(sbar)
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sbar),
        "r"(phase[st])
        : "memory");
    phase[st] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sbuf), "r"(uint32_t(seg))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int ilog2(int64_t x) {
  int r = 0;
  while ((int64_t(1) << r) < x) ++r;
  return r;
}

}  // namespace

cudaError_t launch_kv_gather(const void* store, void* pool, const int32_t* d_slots, const int32_t* d_pages,
                             int32_t n_matched, int32_t layer, const KvGeom& g, int32_t target_ctas,
                             cudaStream_t stream, const LinearCopies* lin) {
  LinearCopies l{};
  if (lin) l = *lin;
  if (l.n < 0 || l.n > LinearCopies::kMax) return cudaErrorInvalidValue;
  const int64_t seg16 = int64_t(g.S) * (g.d / 8);
  int64_t n_seg = int64_t(std::max(n_matched, 0)) * g.Hkv * 2 * (g.C / g.S);
  for (int i = 0; i < l.n; ++i) {
    if (l.n16[i] < 0) return cudaErrorInvalidValue;
    n_seg += (l.n16[i] + seg16 - 1) / seg16;
  }
  if (n_seg <= 0) return cudaSuccess;
  const int64_t ctas = std::min<int64_t>(target_ctas, (n_seg + kThreads / 32 - 1) / (kThreads / 32));
  // experiment (PCR_GATHER_SMEM=bytes): reserve dynamic shared memory the kernel does not use, so
  // a gather CTA cannot share an SM with an attention CTA (~194 KB) -- the SMs split instead
  static const int smem = [] {
    const char* e = std::getenv("PCR_GATHER_SMEM");
    int v = e ? std::atoi(e) : 0;
    v = std::max(0, std::min(v, 200 << 10));
    if (v > (48 << 10)) cudaFuncSetAttribute(kv_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
    return v;
  }();
  kv_gather_kernel<<<int(ctas), kThreads, smem, stream>>>(static_cast<const uint4*>(store), static_cast<uint4*>(pool),
                                                       d_slots, d_pages, std::max(n_matched, 0), layer, g,
                                                       ilog2(g.d / 8), ilog2(g.C / g.S), l);
  return cudaGetLastError();
}

cudaError_t launch_kv_gather_stream(const void* store, void* pool, const int32_t* d_slots, const int32_t* d_pages,
                                    int32_t n_matched, const KvGeom& g, int32_t target_ctas, const LinearCopies* lin,
                                    int32_t* ready, cudaStream_t stream, int32_t* warps_out) {
  LinearCopies l{};
  if (lin) l = *lin;
  if (l.n < 0 || l.n > LinearCopies::kMax || !ready) return cudaErrorInvalidValue;
  const int64_t seg16 = int64_t(g.S) * (g.d / 8);
  int64_t n_seg = int64_t(std::max(n_matched, 0)) * g.Hkv * 2 * (g.C / g.S);
  for (int i = 0; i < l.n; ++i) {
    if (l.n16[i] < 0) return cudaErrorInvalidValue;
    n_seg += (l.n16[i] + seg16 - 1) / seg16;
  }
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(target_ctas, (n_seg + kThreads / 32 - 1) / (kThreads / 32)));
  *warps_out = int32_t(ctas * (kThreads / 32));
  kv_gather_stream_kernel<<<int(ctas), kThreads, 0, stream>>>(
      static_cast<const uint4*>(store), static_cast<uint4*>(pool), d_slots, d_pages, std::max(n_matched, 0), g.L, g,
      ilog2(g.d / 8), ilog2(g.C / g.S), l, ready);
  return cudaGetLastError();
}

cudaError_t launch_kv_gather_tma(const void* store, void* pool, const int32_t* d_slots, const int32_t* d_pages,
                                 int32_t n_matched, int32_t layer, const KvGeom& g, int32_t ctas, cudaStream_t stream) {
  if (n_matched <= 0) return cudaSuccess;
  if (int64_t(g.S) * g.d * 2 > kTmaSegMax) return cudaErrorInvalidValue;
  kv_gather_tma_kernel<<<ctas, 32, 0, stream>>>(static_cast<const uint8_t*>(store), static_cast<uint8_t*>(pool),
                                                d_slots, d_pages, n_matched, layer, g);
  return cudaGetLastError();
}

cudaError_t launch_kv_scatter(const void* pool, void* store, const int32_t* d_slots, const int32_t* d_pages,
                              int32_t chunk0, int32_t n_chunks, int32_t layer, const KvGeom& g, int32_t target_ctas,
                              cudaStream_t stream) {
  if (n_chunks <= 0) return cudaSuccess;
  const int64_t n_seg = int64_t(n_chunks) * g.Hkv * 2 * (g.C / g.S);
  const int64_t ctas = std::min<int64_t>(target_ctas, (n_seg + kThreads / 32 - 1) / (kThreads / 32));
  kv_scatter_kernel<<<int(ctas), kThreads, 0, stream>>>(static_cast<const uint4*>(pool), static_cast<uint4*>(store),
                                                        d_slots, d_pages, chunk0, n_chunks, layer, g, ilog2(g.d / 8),
                                                        ilog2(g.C / g.S));
  return cudaGetLastError();
}

cudaError_t launch_kv_append(const void* k_new, const void* v_new, void* pool, const int32_t* d_pages,
                             int64_t n1, int64_t n2, int32_t n_req_pages, int32_t layer, const KvGeom& g,
                             cudaStream_t stream) {
  const int64_t per_tok = int64_t(g.Hkv) * (g.d / 8);
  const int64_t units = (int64_t(n_req_pages) * g.S - n1) * per_tok;
  if (units <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (units + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  kv_append_kernel<<<static_cast<int>(blocks), threads, 0, stream>>>(
      static_cast<const uint4*>(k_new), static_cast<const uint4*>(v_new), static_cast<uint4*>(pool), d_pages, n1,
      n2, n_req_pages, layer, g, ilog2(g.d / 8), ilog2(g.S));
  return cudaGetLastError();
}

}  // namespace pcr
