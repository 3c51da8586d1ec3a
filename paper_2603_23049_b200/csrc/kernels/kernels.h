// Launch interface of the hot-path kernels (internal; the public boundary is include/pcr.h).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace pcr {

// Geometry shared by the copy kernels.  All sizes are in elements (bf16) unless noted.
struct KvGeom {
  int32_t L, Hkv, d, C, S;          // layers, local kv heads, head dim, chunk tokens, page tokens
  int64_t n_pool_pages;             // pages in the pool
  int64_t slot_elems;               // elements of one store slot = L*Hkv*2*C*d
};

// Store slots are page-major: slot[layer][t/S % (C/S)][h][kv][t%S][d] (= the images of the pool
// pages the chunk fills), so a chunk-layer with consecutive pool pages is one contiguous run.
// pcr_store_write/read convert from/to the API layout [L][Hkv][2][C][d].

// Up to kMax linear copies of n16[i] 16-byte units, src[i] -> dst[i] (16-byte aligned), that ride
// in the same gather launch (host_io: the layer's q/k/v from mapped page-locked host memory).
struct LinearCopies {
  static constexpr int kMax = 3;
  int32_t n;
  const uint4* src[kMax];
  uint4* dst[kMax];
  int64_t n16[kMax];
  int64_t src_stride16[kMax], dst_stride16[kMax];   // per-layer advance (streamed gather; 0 otherwise)
};

// a2: pool[layer][pages[t/S]][h][kv][t%S] = store[slots[t/C]][layer][(t%C)/S][h][kv][t%S], t < n_matched*C.
// `store` is the device (UVA) view of the mapped pinned host store; 16-byte loads/stores.
// `lin` (nullable): extra linear copies done by the same launch.
cudaError_t launch_kv_gather(const void* store, void* pool, const int32_t* d_slots, const int32_t* d_pages,
                             int32_t n_matched, int32_t layer, const KvGeom& g, int32_t target_ctas,
                             cudaStream_t stream, const LinearCopies* lin = nullptr);

// a2, streamed: every layer of the request in one launch (layers in order); after its share of
// layer l each warp adds 1 to ready[l] with release semantics, so layer l is complete when
// ready[l] == *warps_out (the attention acquires it).  ready[0..L) must be zero before the launch.
// Linear copy i of layer l: src[i] + l*src_stride16[i] -> dst[i] + l*dst_stride16[i].
cudaError_t launch_kv_gather_stream(const void* store, void* pool, const int32_t* d_slots, const int32_t* d_pages,
                                    int32_t n_matched, const KvGeom& g, int32_t target_ctas, const LinearCopies* lin,
                                    int32_t* ready, cudaStream_t stream, int32_t* warps_out);

// a2 variant (load_mode 3, experiment): same copy with TMA bulk copies (host -> smem -> pool).
cudaError_t launch_kv_gather_tma(const void* store, void* pool, const int32_t* d_slots, const int32_t* d_pages,
                                 int32_t n_matched, int32_t layer, const KvGeom& g, int32_t ctas, cudaStream_t stream);

// f1: store[slots[c]][layer][(t%C)/S][h][kv][t%S] = pool[layer][pages[t/S]][h][kv][t%S] for the chain
// chunks c in [chunk0, chunk0+n_chunks) (the request's reserved chunks), into the mapped store.
cudaError_t launch_kv_scatter(const void* pool, void* store, const int32_t* d_slots, const int32_t* d_pages,
                              int32_t chunk0, int32_t n_chunks, int32_t layer, const KvGeom& g, int32_t target_ctas,
                              cudaStream_t stream);

// a3: suffix token i -> pool token n1+i for K and V; zero-fills rows [n1+n2, n_pages*S) of the
// request's last page so the attention never reads uninitialised (possibly NaN) bits.
cudaError_t launch_kv_append(const void* k_new, const void* v_new, void* pool, const int32_t* d_pages,
                             int64_t n1, int64_t n2, int32_t n_req_pages, int32_t layer, const KvGeom& g,
                             cudaStream_t stream);

struct AttnParams {
  const uint16_t* q;      // [N2][Hq_loc][d]
  uint16_t* out;          // [N2][Hq_loc][d]
  const int32_t* pages;   // [n_req_pages] device page table of the request
  int32_t n1, n2;
  int32_t hq, hkv;        // local heads
  int32_t layer;
  int32_t S;              // page tokens
  int32_t n_req_pages;
  int64_t n_pool_pages;
  float scale_log2;       // log2(e) / sqrt(d)
  int32_t n_splits;       // set by the launcher (split-KV count)
  float* ws_o;            // split-KV workspace [splits][N2*hq][d] fp32 (nullable: no split-KV)
  float* ws_lse;          // [splits][N2*hq] log2-domain LSE
  int64_t ws_bytes;       // bytes available in ws_o
  // Context-split sharding: keys available on this rank = [0, kv_len) of the virtual
  // context (its own prefix chunks, then -- on the rank that holds it -- the suffix); 0 = n1 + n2;
  // < 0 = no key on this rank.
  int32_t kv_len;
  // Non-null: write this rank's partial -- O normalised by its own row sum (fp32, [N2*hq][d]) and
  // the log2-domain LSE ([N2*hq]) -- instead of the bf16 output (merged across ranks later).
  float* part_o;
  float* part_lse;
  // Fused a3 (non-null k_new/v_new, [N2][hkv][d] device): the attention reads the suffix keys
  // straight from k_new/v_new (TMA) instead of the pool, and the CTAs of the last M-block write
  // them into the request's pool pages (TMA stores from the same shared-memory tiles), so no
  // separate append kernel runs.  Rows past N2 in the last page's final 64-row box are written as
  // zeros; rows beyond that box are not touched (the attention never reads them).
  const uint16_t* k_new;
  const uint16_t* v_new;
  int32_t cluster_reduce;   // set by the launcher: split-KV partials reduced over DSMEM in-kernel
  // Streamed gather (non-null): the TMA producer waits until ready[layer] >= ready_target (acquire)
  // before its first load -- the layer's pool pages (and host_io inputs) have landed.
  const int32_t* ready;
  int32_t ready_target;
  // Split-KV reduce inside the attention through L2 (set by the launcher when the whole grid is one
  // wave): spin_ctr = [2][256] uint32 per plan region (arrival counts, generations), zeroed once.
  uint32_t* spin_ctr;
  int32_t spin_reduce;
  // 1: no kernel before this one in the stream writes anything it reads (fused append): PDL's
  // griddepcontrol.wait moves from the prologue to just before the epilogue's global writes.
  int32_t late_dep_wait;
  // Set by the launcher: the epilogue stages O (bf16 out, or the fp32 split-KV / context-split
  // partial) in shared memory and writes it with TMA stores (coalesced, rows past N2 clipped)
  // instead of one row per thread from registers.
  int32_t tma_epilogue;
  // Set by the launcher: fused-append placement (0: the last M-block's CTAs store every suffix box
  // of their range; 1: each suffix box is stored by the CTA whose query tokens contain it).
  int32_t append_owner;
};

// Merge n_parts partials (O normalised per part, log2-domain LSE; part s at o + s*o_stride and
// lse + s*lse_stride, rows x d and rows floats) into bf16 out [rows][d] (the split-KV combine).
cudaError_t launch_merge_partials(const float* o, int64_t o_stride, const float* lse, int64_t lse_stride,
                                  int32_t n_parts, int64_t rows, int32_t d, uint16_t* out, cudaStream_t stream);

// a4: suffix-query causal attention over the request's pool pages (tcgen05 + TMEM + TMA).
// `tmap_pool` is a 2D tensor map over the pool viewed as [rows][d] (rows = L*pages*Hkv*2*S),
// box {64, S}, SWIZZLE_128B.
// Rows of the pool tensor map's TMA box the attention kernel expects (S_pg, or a 64-row part).
int32_t attn_pool_box_rows(int32_t S);
// `launches` is incremented by the number of kernels enqueued (attention [+ split-KV combine]).
cudaError_t launch_suffix_attn(const CUtensorMap* tmap_pool, const AttnParams& p, int32_t d,
                               cudaStream_t stream, int* launches);

}  // namespace pcr
