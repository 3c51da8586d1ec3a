// a2 kv_gather (host store -> HBM pool) and a3 kv_append (suffix K/V -> pool).
//
// "To efficiently copy KV cache from a CPU chunk to multiple non-consecutive GPU memory
// blocks, we leverage ... cudaMemcpyBatchAsync()".  On B200 the copy is an SM kernel instead:
// every thread streams 16-byte vectors straight out of the mapped pinned host store over PCIe
// Gen5 (zero-copy, ld.global.cs) and writes them, 16 bytes at a time, into the pool pages of
// the request.  Measured on this pool's B200 (tools/h2d_probe.cu): 8+ CTAs x 256 threads with
// 4 loads in flight per thread reach 51.2 GB/s = 92% of the copy engine's 55.6 GB/s, so the
// gather needs only a handful of SMs and leaves the rest to the concurrent attention.
#include "kernels.h"

namespace pcr {
namespace {

// 256 threads x <= 40 registers (10K registers, no shared memory) lets a gather CTA co-reside
// with an attention CTA (256 threads, ~47K registers, ~195 KB smem) on the same SM, so loads of
// layer l+1 are never queued behind the attention grid of layer l.
constexpr int kThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ld_host_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// grid = (ctas_per_chunk, n_matched).  Chunk c's layer block in the store is contiguous:
// [Hkv][2][C][d] starting at store + slot*slot_elems + layer*Hkv*2*C*d.
__global__ void __launch_bounds__(kThreads, 6) kv_gather_kernel(const uint4* __restrict__ store,
                                                             uint4* __restrict__ pool,
                                                             const int32_t* __restrict__ slots,
                                                             const int32_t* __restrict__ pages, int32_t layer,
                                                             KvGeom g, int32_t row16_log2, int32_t C_log2,
                                                             int32_t S_log2) {
  const int32_t c = blockIdx.y;
  const int64_t row16 = int64_t(1) << row16_log2;            // 16-byte units per d-row
  const int64_t block16 = int64_t(g.Hkv) * 2 * g.C * row16;   // units of one chunk-layer
  const uint4* src = store + (int64_t(slots[c]) * g.slot_elems + int64_t(layer) * g.Hkv * 2 * g.C * g.d) / 8;
  const int64_t page16 = int64_t(g.Hkv) * 2 * g.S * row16;
  uint4* dst_layer = pool + int64_t(layer) * g.n_pool_pages * page16;
  const int64_t stride = int64_t(gridDim.x) * kThreads;
  for (int64_t base = int64_t(blockIdx.x) * kThreads + threadIdx.x; base < block16; base += stride * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t o = base + u * stride;
      if (o < block16) v[u] = ld_host_stream(src + o);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t o = base + u * stride;
      if (o < block16) {
        const int64_t row = o >> row16_log2;
        const int64_t col = o & (row16 - 1);
        const int64_t hk = row >> C_log2;               // h*2 + kv
        const int64_t tt = (int64_t(c) << C_log2) + (row & (g.C - 1));
        const int64_t page = pages[tt >> S_log2];
        dst_layer[page * page16 + ((hk << S_log2) + (tt & (g.S - 1))) * row16 + col] = v[u];
      }
    }
  }
}

// One 16-byte unit per thread-iteration over [n2][Hkv][d/8] for K and V, then the tail rows.
__global__ void kv_append_kernel(const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                                 uint4* __restrict__ pool, const int32_t* __restrict__ pages, int64_t n1,
                                 int64_t n2, int32_t n_req_pages, int32_t layer, KvGeom g, int32_t row16_log2,
                                 int32_t S_log2) {
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

int ilog2(int64_t x) {
  int r = 0;
  while ((int64_t(1) << r) < x) ++r;
  return r;
}

}  // namespace

cudaError_t launch_kv_gather(const void* store, void* pool, const int32_t* d_slots, const int32_t* d_pages,
                             int32_t n_matched, int32_t layer, const KvGeom& g, int32_t target_ctas,
                             cudaStream_t stream) {
  if (n_matched <= 0) return cudaSuccess;
  const int per_chunk = (target_ctas + n_matched - 1) / n_matched;
  dim3 grid(per_chunk, n_matched);
  kv_gather_kernel<<<grid, kThreads, 0, stream>>>(static_cast<const uint4*>(store), static_cast<uint4*>(pool),
                                                  d_slots, d_pages, layer, g, ilog2(g.d / 8), ilog2(g.C),
                                                  ilog2(g.S));
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
