// a4 — suffix-query causal attention over the paged pool (prefix + suffix KV), sm_100a.
//
// What it computes (R2/R3/R18): for local query head h (kv head g = h / G)
// and suffix row i at absolute position p = n1 + i,
//     out[i][h] = sum_{j<=p} w_j V[j][g] / sum_{j<=p} w_j,   w_j = bf16(exp(s_j - m)),
//     s_j = q[i][h] . K[j][g] / sqrt(d),
// bf16 inputs, fp32 accumulation (TMEM), bf16 output.
//
// B200 design (DESIGN.md §6 "suffix_attn"):
//  * GQA packing: M rows are (token, head-in-group) pairs, r = t*G + gg, so one K/V tile read
//    serves all G query heads of the group.  A CTA owns NQ = 2 Q tiles of 128 rows (256 rows)
//    of one kv head and a range of 64-key tiles (split-KV when the grid is small); CTAs run
//    heaviest causal M-blocks first.
//  * warps 0 / 3 (converged, one elected lane issues): TMA producers -- warp 0 loads Q tile 1
//    (3D tensor map over q [N2][Hq][d], box {64, G, 128/G}, rows past N2 zero-filled) and the K
//    tiles, warp 3 the V tiles (2D map over the pool, boxes {64 dims, min(S_pg, 64) rows},
//    SWIZZLE_128B) into a 4-stage ring.  With the fused append the CTAs of the last M-block (or,
//    in a split-KV grid with a long suffix, each box's owning CTA) also store the suffix K/V boxes
//    they loaded into the pool (TMA stores, two tiles after the load, not blocking the producer).
//  * warp 1 (converged, elected issue, precomputed descriptors): tcgen05.mma kind::f16 --
//        S_t(j) = Q_t K(j)^T  (tile 0: TS, Q_0 in TMEM; tile 1: SS, K-major) into a TMEM S buffer
//        O_t   += P_t(j) V(j) (P from TMEM, V MN-major) into TMEM O_t (d columns)
//    S rotates through three 64-column buffers shared by the two tiles (S_t(j) in buffer
//    (2j + t) % 3; Q_0 64 + S 192 + O 256 = 512 columns), so S_t(j+1) is computed while the softmax
//    works on S_t(j); an S is only ever issued into the buffer the PV just issued has read (tcgen05
//    MMAs of one thread execute in issue order).  (PCR_Q0_TMEM=0: both Q tiles in shared memory,
//    S double-buffered per tile.)
//  * warp 2: tcgen05.alloc of all 512 TMEM columns.
//  * warps 4-7 / 8-11: softmax of Q tile 0 / 1, one thread per M row (= TMEM lane): row max
//    with FMNMX3, x = s*scale - m with FFMA2, 2^x by MUFU.EX2 or (kPolyPairs of every 16 pairs) a
//    polynomial on the FMA pipe, P -> TMEM over the S columns (tcgen05.st), row sum of the fp32
//    weights with FADD2 (R18); the two warpgroups take turns on the exponentials; causal mask
//    only on tiles crossing the diagonal; lazy rescaling of O (only when the running max grows by
//    > 8, log2 units), after waiting for the previous PV.  Epilogue: O / l -> bf16, or the fp32
//    partial + log2-LSE per KV split, staged in shared memory and written with TMA stores.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace pcr {
namespace {

using namespace ptx;

constexpr int kBlockM = 128;   // rows per Q tile (= TMEM lanes)
// Keys per tile: 64, so S fits double-buffered per Q tile in TMEM (2 x 2 x 64 + 2 x 128 O = 512
// columns) and the softmax of S_t(j+1) can start while PV_t(j) runs.  A 128-key variant (S
// single-buffered per Q tile, QK^T with N = 128, each row's scores streamed from TMEM in two
// 64-column halves -- the softmax below is written for any multiple of 64) measured 7% slower on
// the M7 shapes (profiles/r02_block_n_128.txt): the lost S double-buffering costs more than the
// halved barrier round trips and operand traffic save.
#ifndef PCR_BLOCK_N
#define PCR_BLOCK_N 64
#endif
constexpr int kBlockN = PCR_BLOCK_N;
static_assert(kBlockN == 64 || kBlockN == 128, "64- or 128-key tiles");
constexpr int kNQ = 2;         // Q tiles per CTA
#ifndef PCR_KV_STAGES
#define PCR_KV_STAGES (256 / PCR_BLOCK_N)
#endif
constexpr int kStages = PCR_KV_STAGES;  // K/V smem ring depth
constexpr int kThreads = 128 + kNQ * 128;
// Experiment (PCR_Q_TMEM=1): Q lives in TMEM and QK^T runs as a TS MMA (A = Q from TMEM, only K
// is read from shared memory: the 64-key SS QK^T is bound by shared-memory operand bandwidth).
// The 128 TMEM columns for two Q tiles come from single-buffering S per Q tile.
#ifndef PCR_Q_TMEM
#define PCR_Q_TMEM 0
#endif
constexpr int kSBuf = (PCR_Q_TMEM || kBlockN == 128) ? 1 : 2;   // S buffers per Q tile (barrier parity domain)
// PCR_Q0_TMEM=1: Q tile 0 lives in TMEM and its QK^T runs as a TS MMA (A from TMEM: no shared-
// memory traffic for A), Q tile 1 stays in shared memory (SS).  The 64 TMEM columns for Q0 come
// from sharing THREE rotating S buffers between the two tiles instead of two per tile: S_t(j) goes
// to buffer (2j + t) % 3, and the MMA issue order [P0(j)] PV0(j) S1(j+1) [P1(j)] PV1(j) S0(j+2)
// only ever writes the buffer the PV just issued has read (MMAs of one thread run in order).
#ifndef PCR_Q0_TMEM
#define PCR_Q0_TMEM 1
#endif
static_assert(!(PCR_Q0_TMEM && PCR_Q_TMEM), "one Q-in-TMEM mode at a time");
constexpr int kSCols = PCR_Q0_TMEM ? 3 * kBlockN : kSBuf * kNQ * kBlockN;   // TMEM columns of S
// TMEM column (relative) of S_t(it)
__device__ __forceinline__ uint32_t s_buf_col(int t, int it) {
  return PCR_Q0_TMEM ? uint32_t(((2 * it + t) % 3) * kBlockN) : uint32_t((kSBuf * t + it % kSBuf) * kBlockN);
}
constexpr int kMaxBox = kBlockN / 16;   // TMA boxes per key tile (pool boxes are >= 16 rows)
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// Pairs (of 16 per 32-column chunk) whose exp2 runs as a polynomial on the FMA pipe instead of
// MUFU.EX2: at d = 128 the MUFU rate (16/clk/SM) equals the tensor rate per score, so moving some
// exponentials to the FMA pipe helps the softmax keep up with the MMAs.  Round 1 measured 4 of 16
// best; with the row sum on the FMA pipe too (FADD2, R18) 1 of 16 is (+8% on the M7 shape,
// profiles/r02_poly_pairs_sweep.txt).
#ifndef PCR_POLY_PAIRS
#define PCR_POLY_PAIRS 1
#endif
constexpr int kPolyPairs = PCR_POLY_PAIRS;
// Experiment knob (never set by the default build), a bit mask: 1 = skip the softmax arithmetic
// (the warpgroups only hand the S buffers back), 2 = skip the MMAs (only commits), 4 = skip the
// K/V TMA loads (the producer only arrives), 8 = the MMA warp does not wait for P: which side
// bounds the pipeline.
// Split-KV: every split keeps at least this many key tiles (small N2 grids are latency bound:
// fewer tiles per CTA shorten the serial QK -> softmax -> PV chain).
#ifndef PCR_SPLIT_MIN_TILES
#define PCR_SPLIT_MIN_TILES 4
#endif
// Row sum l (reading R18): accumulates the fp32 weights before their bf16 rounding -- one FADD2 per
// pair inside the exponential loop -- rather than the rounded weights (PCR_ROWSUM_F32=0: one
// FHADD.BF16 per weight after P is published).  +4% on the M7 r=0.5 shape, +2.5% on L70, others
// within noise (profiles/r02_rowsum_variant.txt).
#ifndef PCR_ROWSUM_F32
#define PCR_ROWSUM_F32 1
#endif
// Two TMA producer warps (warp 0: Q + K, warp 3: V) instead of one: +5-10% on the long-suffix
// shapes on a typical box, +30% on a box where the default measured 885 TF/s
// (profiles/r02_split_producer.txt).  PCR_SPLIT_PRODUCER=0 restores the single producer.
#ifndef PCR_SPLIT_PRODUCER
#define PCR_SPLIT_PRODUCER 1
#endif
#ifndef PCR_ATTN_TIMING
#define PCR_ATTN_TIMING 0
#endif
#ifndef PCR_ATTN_PROFILE
#define PCR_ATTN_PROFILE 0
#endif
// the two softmax warpgroups alternate their exponential phases (off in the skip-softmax profile)
#ifndef PCR_EXP_PINGPONG
#define PCR_EXP_PINGPONG ((PCR_ATTN_PROFILE & 1) == 0)
#endif

template <int D>
struct Layout {
  static constexpr int kHalves = D / 64;
  static constexpr int kQHalf = kBlockM * 128;                 // 128 rows x 128 B
  static constexpr int kQTile = kHalves * kQHalf;
  static constexpr int kKVHalf = kBlockN * 128;                // 64 keys x 128 B
  static constexpr int kKVTile = kHalves * kKVHalf;
  static constexpr int kQ0 = 0;
  static constexpr int kK0 = kQ0 + (PCR_Q_TMEM ? 0 : (PCR_Q0_TMEM ? kNQ - 1 : kNQ) * kQTile);   // smem Q tiles
  static constexpr int kV0 = kK0 + kStages * kKVTile;
  static constexpr int kBar = kV0 + kStages * kKVTile;
  // split-KV cluster reduce: this CTA's row LSEs and the merged LSEs (kNQ*128 floats each); the
  // weighted partial O of the CTA ([kNQ*128][D] fp32, 16-byte chunks XOR-swizzled by row) reuses
  // the K/V ring once every MMA has completed
  static constexpr int kLse = kBar + 512;
  static constexpr int kBytes = kLse + 2 * kNQ * kBlockM * 4;
  static_assert(2 * kStages * kKVTile >= kNQ * kBlockM * D * 4, "cluster-reduce partials must fit the K/V ring");
  static constexpr int kAlloc = kBytes + 1024;  // slack for 1024-byte alignment
  // TMEM columns: S_{t,b} (Q tile t, buffer b) at (kSBuf*t+b)*64; [Q_t at kColQ + t*D/2 (bf16
  // pairs), PCR_Q_TMEM]; O_t at kColO + t*D.
  static constexpr uint32_t kColQ = kSCols;
  static constexpr uint32_t kColO = kColQ + (PCR_Q_TMEM ? kNQ * D / 2 : PCR_Q0_TMEM ? D / 2 : 0);
  static_assert(kColO + kNQ * D <= kTmemCols, "TMEM columns");
};

struct Bars {
  uint64_t q_full, k_full[kStages], v_full[kStages], k_empty[kStages], v_empty[kStages];
  uint64_t s_full[kNQ][2], p_full[kNQ][2], o_done[kNQ], o_full;
  uint64_t store_done;   // fused append: the producer's pool stores have finished reading smem
  uint32_t tmem_base;
};

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// L2 loads (cache-global: never a stale L1 line of another CTA's partial)
__device__ __forceinline__ float ld_cg_f32(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_cg_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- cluster (DSMEM) helpers
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_dsmem_f32x4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr) : "memory");
  return v;
}
// TMA store of one box from shared memory into the pool (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(smem_u32(smem_src))
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, const void* smem_src, int32_t c0, int32_t c1,
                                             int32_t c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(smem_src))
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* smem_src, int32_t c0, int32_t c1,
                                             int32_t c2, int32_t c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(smem_src))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* m, int32_t c0, int32_t c1,
                                            int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Experiment knob: K/V TMA loads carry an L2 evict_last policy (the pool's layer stays in L2
// while the next layer's load streams in beside the attention).
#ifndef PCR_KV_L2HINT
#define PCR_KV_L2HINT 0
#endif
__device__ __forceinline__ void tma_load_2d_kv(void* smem_dst, const CUtensorMap* m, int32_t c0, int32_t c1,
                                               uint64_t* bar, uint64_t policy) {
#if PCR_KV_L2HINT
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
#else
  (void)policy;
  tma_load_2d(smem_dst, m, c0, c1, bar);
#endif
}

// D[tmem] (+)= A[tmem] * B[smem]  (kind::f16; A is M x K bf16 packed two per 32-bit column).
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Experiment knobs (mbarrier polling): the K/V-landed checks of tile 0's softmax warpgroup by ONE
// thread instead of 128 (PCR_KV_WAIT_ONE; the p_full arrival of that thread still orders the MMA
// warp after the loads), and every other wait of a converged warp by lane 0 + __syncwarp
// (PCR_LANE0_WAIT): 128 threads polling one mbarrier compete with the producers' arrivals.
#ifndef PCR_KV_WAIT_ONE
#define PCR_KV_WAIT_ONE 1
#endif
#ifndef PCR_LANE0_WAIT
#define PCR_LANE0_WAIT 0
#endif
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  if (PCR_LANE0_WAIT) {
    if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
    __syncwarp();
  } else {
    mbar_wait(bar, parity);
  }
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 2^x for a pair of x <= 0 on the FMA pipe (FA4-style MUFU offload): x = n + f with
// n = round(x), f in [-1/2, 1/2]; 2^f by a degree-3 minimax polynomial (max relative error
// 7.5e-5, far below the 2^-9 bf16 rounding P gets next); 2^n added to the exponent bits.
// x is clamped at -126 (result >= 2^-126 instead of 0 for masked keys: < 1e-37 relative).
__device__ __forceinline__ void exp2_poly2(uint64_t x2, float& y0, float& y1) {
  float x0, x1;
  f2_unpack(x2, x0, x1);
  const uint64_t xc = f2_pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t t = fadd2(xc, f2_pack(12582912.f, 12582912.f));      // 1.5 * 2^23: round to int
  const uint64_t r = fadd2(t, f2_pack(-12582912.f, -12582912.f));     // round(x)
  const uint64_t f = ffma2(r, f2_pack(-1.f, -1.f), xc);               // x - round(x)
  uint64_t q = ffma2(f, f2_pack(0.055171095f, 0.055171095f), f2_pack(0.24260999f, 0.24260999f));
  q = ffma2(q, f, f2_pack(0.69326097f, 0.69326097f));
  q = ffma2(q, f, f2_pack(0.99992812f, 0.99992812f));
  float q0, q1, t0, t1;
  f2_unpack(q, q0, q1);
  f2_unpack(t, t0, t1);
  // bits(t) = bits(1.5*2^23) + n and (bits(1.5*2^23) << 23) == 0 mod 2^32, so n << 23 == bits(t) << 23
  y0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23));
  y1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23));
}

#if PCR_ATTN_TIMELINE
// experiment: per-CTA timeline (globaltimer ns: start, first S ready, main loop end, end; SM; key
// tiles) of the last launch of each layer, read back with pcr_debug_attn_timeline
constexpr int kTlLayers = 128, kTlCtas = 2048;
__device__ unsigned long long g_timeline[kTlLayers][kTlCtas][6];
#endif

// 136 registers x 384 threads = 52K of the SM's 64K: a 256-thread gather CTA (10K) still fits
// beside an attention CTA, so layer l+1's host->HBM load never waits for attention SMs.
template <int D>
__global__ void __maxnreg__(136)
    suffix_attn_kernel(const __grid_constant__ CUtensorMap tmap_pool, const __grid_constant__ CUtensorMap tmap_q,
                       const __grid_constant__ CUtensorMap tmap_kn, const __grid_constant__ CUtensorMap tmap_vn,
                       const __grid_constant__ CUtensorMap tmap_out, const AttnParams p) {
  using Lay = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + Lay::kBar);

  // warp index through a shuffle: provably warp-uniform, so role branches are uniform and the MMA
  // and TMA loops keep counters and descriptors in uniform registers (no R2UR per instruction)
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
#ifndef PCR_ATTN_TIMELINE
#define PCR_ATTN_TIMELINE 0
#endif
#if PCR_ATTN_TIMELINE
  // experiment: per-CTA timeline (globaltimer ns) printed by the first softmax thread
  const uint64_t tl_start = globaltimer_ns();
  uint64_t tl_loop0 = 0, tl_loop1 = 0;
#endif
  // Longest-processing-time-first order (causal: the last M-blocks see the most keys)
  const int G = p.hq / p.hkv;
  const int tok_per_tile = kBlockM / G;
  const int n_mblocks = (p.n2 + kNQ * tok_per_tile - 1) / (kNQ * tok_per_tile);
  const int g = blockIdx.x % p.hkv;  // local kv head
  const int mblock = n_mblocks - 1 - blockIdx.x / p.hkv;
  const int i0 = mblock * kNQ * tok_per_tile;
  const int i_end = min(i0 + kNQ * tok_per_tile, p.n2);
  const int kv_len = p.kv_len > 0 ? p.kv_len : (p.kv_len < 0 ? 0 : p.n1 + p.n2);   // keys present here
  const int n_tiles_all = (min(p.n1 + i_end, kv_len) + kBlockN - 1) / kBlockN;
  const int per_split = (n_tiles_all + p.n_splits - 1) / p.n_splits;
  const int j_begin = blockIdx.z * per_split;
  const int j_end = min(j_begin + per_split, n_tiles_all);
  const int n_iter = max(0, j_end - j_begin);
  auto tile_of = [&](int it) { return j_begin + it; };

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, PCR_Q_TMEM ? kNQ * 128 : PCR_Q0_TMEM ? 1 + 128 : 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    for (int t = 0; t < kNQ; ++t) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&bars->s_full[t][b], 1);
        mbar_init(&bars->p_full[t][b], 128);
      }
      mbar_init(&bars->o_done[t], 1);
    }
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->store_done, PCR_SPLIT_PRODUCER ? 2 : 1);   // one arrival per producer warp
    fence_mbar_init();
    tma_prefetch_desc(&tmap_pool);
    tma_prefetch_desc(&tmap_q);
    if (p.k_new) {
      tma_prefetch_desc(&tmap_kn);
      tma_prefetch_desc(&tmap_vn);
    }
  }
  // fused append (every other read of the suffix keys comes from k_new/v_new), two placements
  // chosen by the launcher (p.append_owner):
  //  * 0: the CTAs of the last M-block (they see every key) write every suffix K/V box of their key
  //    range -- best when the grid runs in several waves, which absorb those CTAs' extra work;
  //  * 1: each box is written by the CTA whose own query tokens contain its first key (about one
  //    tile per CTA, on its causal diagonal) -- best for a split-KV grid with a long suffix, where
  //    the last M-block's CTAs would be the critical path (M7 r=0.5 on one kv head: 102 -> 71 us
  //    per layer; 4-6% slower on the multi-wave shapes, profiles/r02_append_owner.txt).
  const bool fold = p.k_new != nullptr;
  const bool owner_mode = p.append_owner != 0;
  const bool writer = fold && (owner_mode || blockIdx.x / p.hkv == 0);
  if (warp == 2) tmem_alloc<kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  // Everything above (barrier init, descriptor prefetch, TMEM alloc) overlaps the tail of the
  // append kernel before it under PDL; q and the pool are read only after it has completed.
  // PDL: the kernel before this one in the stream may still be draining.  Without a separate append
  // kernel (fused append) nothing this kernel READS was written by it -- the prefix arrives through
  // the streamed gather's counters or cross-stream events, q/k_new/v_new from the caller -- so the
  // wait moves to just before the first global WRITE that an earlier kernel may still read (the
  // split-KV workspace a previous combine reads): the main loop overlaps that combine.
  if (!p.late_dep_wait) grid_dep_wait();
  grid_dep_launch();

  float ep_lse = -INFINITY, ep_inv_l = 0.f;   // cluster reduce: this softmax thread's row LSE and 1/l

  if (warp == 0 || (PCR_SPLIT_PRODUCER && warp == 3)) {
    // ---------------------------------------------------------------- TMA producers
    // Converged warps: the lanes hold the page ids of 32 consecutive pages (one coalesced load per
    // 32 pages, read by shuffles), one elected lane issues the TMA copies.  Warp 0 loads Q and the
    // K tiles, warp 3 the V tiles (PCR_SPLIT_PRODUCER; else warp 0 does both): K(j) is needed two
    // iterations before V(j) (S(j+2) is issued right after PV(j)), and a single producer issues
    // K(j) only after V(j-1), which waits for the PV that freed its stage.
    const bool do_k = warp == 0, do_v = warp == 3 || !PCR_SPLIT_PRODUCER;
    if (n_iter > 0) {
      const int lane = threadIdx.x & 31;
      if (p.ready) {
        // streamed gather: wait until every warp of the gather kernel has published this layer,
        // then order the TMA (async-proxy) reads after the generic-proxy writes just acquired
        if (lane == 0) {
          const uint64_t t0 = globaltimer_ns();
          uint32_t ns = 32;
          while (ld_acquire_gpu(p.ready + p.layer) < p.ready_target) {
            __nanosleep(ns);
            ns = min(ns * 2, 1024u);
            if (globaltimer_ns() - t0 > 10ull * 1000 * 1000 * 1000) {   // 10 s: never hang the GPU
              printf("suffix_attn: layer %d load never completed (ready %d of %d)\n", p.layer,
                     ld_acquire_gpu(p.ready + p.layer), p.ready_target);
              __trap();
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
      }
      if (do_k && !PCR_Q_TMEM && elect_one()) {
        constexpr int t0 = PCR_Q0_TMEM ? 1 : 0;   // (Q0 mode: tile 0 goes to TMEM via its softmax warps)
        mbar_arrive_expect_tx(&bars->q_full, (kNQ - t0) * Lay::kQTile);
        for (int t = t0; t < kNQ; ++t)
          for (int hf = 0; hf < Lay::kHalves; ++hf)
            tma_load_3d(smem + Lay::kQ0 + (t - t0) * Lay::kQTile + hf * Lay::kQHalf, &tmap_q, hf * 64, g * G,
                        i0 + t * tok_per_tile, &bars->q_full);
      }
      __syncwarp();
      // pool rows fit in 32 bits (TMA coordinates are int32); S_pg is a power of two
      const int layer_row0 = p.layer * (p.n_pool_pages * p.hkv * 2 * p.S);
      const int s_log2 = 31 - __clz(p.S);
      const int box = min(p.S, kBlockN);  // rows per TMA box (the pool tensor map's box height)
      const int n_box = kBlockN / box;    // 1 .. kMaxBox (S_pg >= 16)
      int pg_base = -64, pg_row = 0;      // lane l: pool row of K of request page pg_base + l
      uint64_t kv_policy = 0;
#if PCR_KV_L2HINT
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(kv_policy));
#endif
      // Pool row of K for box b of tile `tile` (V = + S), and whether the box holds suffix keys
      // (fused append: read from k_new/v_new; `dst` = it has a pool page to be written to).
      auto box_rows = [&](int tile, int b, int& row, bool& sfx, bool& dst) {
        const int key = tile_of(tile) * kBlockN + b * box;
        const bool in_req = (key >> s_log2) < p.n_req_pages;
        const int pidx = in_req ? key >> s_log2 : p.n_req_pages - 1;  // clamp: finite, masked
        if (pidx < pg_base || pidx >= pg_base + 32) {
          pg_base = pidx;
          pg_row = pidx + lane < p.n_req_pages ? layer_row0 + ((p.pages[pidx + lane] * p.hkv + g) << (s_log2 + 1)) : 0;
        }
        row = __shfl_sync(0xffffffffu, pg_row, pidx - pg_base) + (in_req ? key & (p.S - 1) : 0);
        sfx = fold && key >= p.n1;
        // dst: this CTA stores the box (a suffix box of a request page it owns)
        dst = sfx && in_req && (!owner_mode || (key - p.n1 >= i0 && key - p.n1 < i_end));
      };
      // whether tile `tile` holds a box this CTA stores (fused append)
      auto tile_stores = [&](int tile) {
        bool any = false;
#pragma unroll
        for (int b = 0; b < kMaxBox; ++b) {
          if (b < n_box) {
            int row;
            bool sfx, dst;
            box_rows(tile, b, row, sfx, dst);
            any |= dst;
          }
        }
        return any;
      };
      // fused append: write the suffix boxes of tile `tile` (its K or V stage) into the pool
      auto store_tile = [&](int tile, bool v) {
        const int st = tile % kStages;
        const uint8_t* base = smem + (v ? Lay::kV0 : Lay::kK0) + st * Lay::kKVTile;
#pragma unroll
        for (int b = 0; b < kMaxBox; ++b) {
          if (b < n_box) {
            int row;
            bool sfx, dst;
            box_rows(tile, b, row, sfx, dst);
            if (dst && lane == 0) {
#pragma unroll
              for (int hf = 0; hf < Lay::kHalves; ++hf)
                tma_store_2d(&tmap_pool, base + hf * Lay::kKVHalf + b * box * 128, hf * 64, row + (v ? p.S : 0));
            }
          }
        }
        if (lane == 0) bulk_commit();   // one bulk group per stored tile
        __syncwarp();
      };
      // load the K (or V) tile `it` into stage it % kStages (boxes from the pool, or -- suffix keys,
      // fused append -- from k_new / v_new)
      auto load_tile = [&](int it, bool v) {
        const int st = it % kStages;
        int row_k[kMaxBox];
        bool sfx[kMaxBox], dst_unused;
#pragma unroll
        for (int b = 0; b < kMaxBox; ++b)
          if (b < n_box) box_rows(it, b, row_k[b], sfx[b], dst_unused);
        const int sfx_row0 = tile_of(it) * kBlockN - p.n1;   // suffix row of box 0 (fused append)
        uint8_t* dst_s = smem + (v ? Lay::kV0 : Lay::kK0) + st * Lay::kKVTile;
        uint64_t* full = v ? &bars->v_full[st] : &bars->k_full[st];
        if (elect_one()) {
          if (PCR_ATTN_PROFILE & 4) {
            mbar_arrive(full);
          } else {
            mbar_arrive_expect_tx(full, Lay::kKVTile);
#pragma unroll
            for (int b = 0; b < kMaxBox; ++b)
#pragma unroll
              for (int hf = 0; hf < Lay::kHalves; ++hf)
                if (b < n_box) {
                  if (sfx[b])
                    tma_load_3d(dst_s + hf * Lay::kKVHalf + b * box * 128, v ? &tmap_vn : &tmap_kn, hf * 64, g,
                                sfx_row0 + b * box, full);
                  else
                    tma_load_2d_kv(dst_s + hf * Lay::kKVHalf + b * box * 128, &tmap_pool, hf * 64,
                                   row_k[b] + (v ? p.S : 0), full, kv_policy);
                }
          }
        }
        __syncwarp();
      };
      // K(j) and V(j) go into stage j % kStages once their previous occupants are consumed: K after
      // the last QK^T that read it (k_empty), V after the last PV (v_empty).  A tile holding boxes
      // this CTA stores (fused append) is written into the pool from the stage it landed in,
      // kStoreLag tiles later (it has landed by then: the wait is short) and without waiting for
      // the store; before such a stage is refilled the producer waits until its stores have read
      // it (wait_group.read 0: a CTA stores one or two tiles, or -- append_owner = 0, last
      // M-block -- every suffix tile).
#if PCR_ATTN_TIMING
      long long pw_ = 0, pl_ = 0, pc_ = clock64();
#define PCR_PTICK(acc) do { const long long n_ = clock64(); acc += n_ - pc_; pc_ = n_; } while (0)
#else
#define PCR_PTICK(acc) do { } while (0)
#endif
      constexpr int kStoreLag = kStages > 2 ? 2 : 1;
      static_assert(kStoreLag < kStages, "a tile is stored before its stage is refilled");
      uint32_t stored[2] = {0u, 0u};   // per K / V: stages whose tile has pool stores in flight
      bool any_store = false;
      auto produce = [&](int it, bool v) {
        const int st = it % kStages;
        if (it >= kStages) {
          mbar_wait(v ? &bars->v_empty[st] : &bars->k_empty[st], ((it / kStages) - 1) & 1);
          PCR_PTICK(pw_);
          if (writer && ((stored[v] >> st) & 1u)) {
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            stored[v] &= ~(1u << st);
          }
        }
        load_tile(it, v);
        if (writer && it >= kStoreLag && tile_stores(it - kStoreLag)) {
          const int js = it - kStoreLag;
          mbar_wait(v ? &bars->v_full[js % kStages] : &bars->k_full[js % kStages], (js / kStages) & 1);
          store_tile(js, v);
          stored[v] |= 1u << (js % kStages);
          any_store = true;
        }
        PCR_PTICK(pl_);
      };
      for (int it = 0; it < n_iter; ++it) {
        if (do_k) produce(it, false);
        if (do_v) produce(it, true);
      }
#if PCR_ATTN_TIMING
      if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 8 || blockIdx.x == 300) && blockIdx.z == 0)
        printf("PRODTIMING blk %d warp %d iters %d: empty-wait %lld load-issue %lld (clk/iter)\n", blockIdx.x, warp,
               n_iter, pw_ / max(n_iter, 1), pl_ / max(n_iter, 1));
#endif
      if (writer) {
        // the last kStoreLag tiles: store once they have landed, then wait for every pool write
        for (int js = max(0, n_iter - kStoreLag); js < n_iter; ++js) {
          if (!tile_stores(js)) continue;
          if (do_k) {
            mbar_wait(&bars->k_full[js % kStages], (js / kStages) & 1);
            store_tile(js, false);
          }
          if (do_v) {
            mbar_wait(&bars->v_full[js % kStages], (js / kStages) & 1);
            store_tile(js, true);
          }
          any_store = true;
        }
        // the stores have read the ring (the epilogue may stage over it); their global writes
        // complete with the grid, like the epilogue's own TMA stores
#ifndef PCR_TAIL_WAIT_FULL
#define PCR_TAIL_WAIT_FULL 0
#endif
        if (any_store && lane == 0) {
          if (PCR_TAIL_WAIT_FULL) bulk_wait0();
          else bulk_wait_read<0>();
        }
        __syncwarp();
      }
    }
    if (writer && elect_one()) mbar_arrive(&bars->store_done);
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // Converged warp; one elected lane issues each MMA group; descriptor bases precomputed.
    if (n_iter > 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kBlockM, kBlockN, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kBlockM, D, 0, 1);
      mbar_wait(&bars->q_full, 0);
      const uint64_t q_desc0 = smem_desc_sw128(smem_u32(smem + Lay::kQ0), 16, 1024);
      const uint64_t k_desc0 = smem_desc_sw128(smem_u32(smem + Lay::kK0), 16, 1024);
      const uint64_t v_desc0 = smem_desc_sw128(smem_u32(smem + Lay::kV0), Lay::kKVHalf, 1024);
      auto issue_s = [&](int t, int it) {
        const uint64_t qd = q_desc0 + uint64_t((t - (PCR_Q0_TMEM ? 1 : 0)) * Lay::kQTile >> 4);
        const uint64_t kd = k_desc0 + uint64_t((it % kStages) * Lay::kKVTile >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16 && (PCR_ATTN_PROFILE & 2) == 0; ++kk) {
            if (PCR_Q_TMEM || (PCR_Q0_TMEM && t == 0))
              mma_bf16_ts(tmem + s_buf_col(t, it), tmem + Lay::kColQ + (PCR_Q0_TMEM ? 0 : t * (D / 2)) + kk * 8,
                          kd + (((kk >> 2) * Lay::kKVHalf + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
            else
              mma_bf16_ss(tmem + s_buf_col(t, it),
                          qd + (((kk >> 2) * Lay::kQHalf + (kk & 3) * 32) >> 4),
                          kd + (((kk >> 2) * Lay::kKVHalf + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
          }
          mma_commit(&bars->s_full[t][it % kSBuf]);
          if (t == kNQ - 1) mma_commit(&bars->k_empty[it % kStages]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int it) {
        const uint64_t vd = v_desc0 + uint64_t((it % kStages) * Lay::kKVTile >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kBlockN / 16 && (PCR_ATTN_PROFILE & 2) == 0; ++kk)
            mma_bf16_ts(tmem + Lay::kColO + t * D, tmem + s_buf_col(t, it) + kk * 8,
                        vd + (kk * 2048 >> 4), idesc_o, (it > 0 || kk > 0));
          // O_t rescale fence for the last tile only (earlier rescales wait on s_full, below); with
          // one S buffer the wait for S_t(it) already covers PV_t(it-1)
          if (kSBuf == 2 && it == n_iter - 2) mma_commit(&bars->o_done[t]);
          if (t == kNQ - 1) mma_commit(&bars->v_empty[it % kStages]);
        }
        __syncwarp();
      };
      if (PCR_Q0_TMEM) {   // S0(0), S1(0), S0(1): the three rotating S buffers
        mbar_wait(&bars->k_full[0], 0);
        tc_fence_after();
        issue_s(0, 0);
        issue_s(1, 0);
        if (n_iter > 1) {
          mbar_wait(&bars->k_full[1], 0);
          tc_fence_after();
          issue_s(0, 1);
        }
      } else {
        for (int it = 0; it < min(kSBuf, n_iter); ++it) {
          mbar_wait(&bars->k_full[it], 0);
          tc_fence_after();
          for (int t = 0; t < kNQ; ++t) issue_s(t, it);
        }
      }
      // Per Q tile: O_t += P_t(it) V(it), then S_t(it+2) into the buffer P_t(it) just left (MMAs of
      // one thread run in issue order).  Tile 0's next S does not wait for tile 1's P, so the two
      // softmax warpgroups settle out of phase (one in its exponentials while the other waits
      // for S) instead of contending for MUFU in lockstep.
#if PCR_ATTN_TIMING
      long long mt_[5] = {0, 0, 0, 0, 0}, mc_ = clock64();
#define PCR_MTICK(k) do { const long long n_ = clock64(); mt_[k] += n_ - mc_; mc_ = n_; } while (0)
#else
#define PCR_MTICK(k) do { } while (0)
#endif
      // The tensor pipe's instruction queue is shallow (about one MMA group): a pause between
      // groups idles it, and every mbarrier wait costs ~100 clk even when its phase completed long
      // ago.  So the MMA warp waits only for P: tile 0's softmax warpgroup checks that V(it) and
      // K(it+2) have landed before it publishes P_0(it) (it has slack; the MMA warp has none).
      //   [p_full(0,it)] PV_0(it) S_0(it+2) [p_full(1,it)] PV_1(it) S_1(it+2)
      for (int it = 0; it < n_iter; ++it) {
        const bool more = it + kSBuf < n_iter;
        PCR_MTICK(2);
        if ((PCR_ATTN_PROFILE & 8) == 0) mbar_wait_warp(&bars->p_full[0][it % kSBuf], (it / kSBuf) & 1);
        tc_fence_after();
        PCR_MTICK(1);
        issue_pv(0, it);
        if (PCR_Q0_TMEM) {
          if (it + 1 < n_iter) issue_s(1, it + 1);   // into the buffer PV0(it) just read
        } else if (more) {
          issue_s(0, it + kSBuf);
        }
        PCR_MTICK(2);
        if ((PCR_ATTN_PROFILE & 8) == 0) mbar_wait_warp(&bars->p_full[1][it % kSBuf], (it / kSBuf) & 1);
        tc_fence_after();
        PCR_MTICK(1);
        issue_pv(1, it);
        if (PCR_Q0_TMEM) {
          if (it + 2 < n_iter) issue_s(0, it + 2);   // into the buffer PV1(it) just read
        } else if (more) {
          issue_s(1, it + kSBuf);
        }
      }
#if PCR_ATTN_TIMING
      if ((threadIdx.x & 31) == 0 && (blockIdx.x == 0 || blockIdx.x == 300) && blockIdx.z == 0)
        printf("MMATIMING blk %d iters %d: p-wait %lld issue %lld (clk/iter)\n", blockIdx.x, n_iter,
               mt_[1] / max(n_iter, 1), mt_[2] / max(n_iter, 1));
#endif
      if (elect_one()) mma_commit(&bars->o_full);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax / epilogue
    const int t = (warp - 4) >> 2;              // Q tile of this warpgroup
    const int r = threadIdx.x - 128 * (1 + t);   // row within the tile == TMEM lane
    const int i = i0 + t * tok_per_tile + r / G; // suffix token of this row
    const int qh = g * G + (r % G);              // local query head
    const uint32_t lane_base = tmem + (uint32_t((warp & 3) * 32) << 16);
    const uint32_t o_col = lane_base + Lay::kColO + t * D;
    const int kv_len_s = p.kv_len > 0 ? p.kv_len : (p.kv_len < 0 ? 0 : p.n1 + p.n2);
    const int limit = min(p.n1 + i, kv_len_s - 1);  // last visible key of this row
    const int tile_first_key_limit = min(p.n1 + i0 + t * tok_per_tile, kv_len_s - 1);
    // Per tile of 64 keys: (1) row max of S (two 32-column TMEM loads, four FMNMX3 chains);
    // (2) P = bf16(2^(s*scale - m)) via FFMA2 + ex2 (MUFU, or a polynomial on the FMA pipe for
    // kPolyPairs of every 16 pairs), written over the S columns it came from, and the row sum
    // of the fp32 weights via FADD2 (R18).
    float m_raw = -INFINITY, l = 0.f;
#if PCR_Q_TMEM
    if (n_iter > 0) {
      // this row's q (D bf16, zero past N2) -> TMEM columns kColQ + t*D/2 .. (bf16 pairs, lane = row)
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (int64_t(i) * p.hq + qh) * D);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint4 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = i < p.n2 ? src[c * 8 + e] : make_uint4(0, 0, 0, 0);
        tmem_st32(lane_base + Lay::kColQ + t * (D / 2) + c * 32, reinterpret_cast<const float*>(v));
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars->q_full);
    }
#endif
#if PCR_EXP_PINGPONG
    if (t == 1 && n_iter > 0) named_bar_arrive(1, 256);  // tile 0 takes the first turn
#endif
#if PCR_ATTN_TIMING
    long long tm_[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tc_ = clock64();
#define PCR_TICK(k) do { const long long n_ = clock64(); tm_[k] += n_ - tc_; tc_ = n_; } while (0)
#else
#define PCR_TICK(k) do { } while (0)
#endif
    const uint64_t scale2 = f2_pack(p.scale_log2, p.scale_log2);
    // Before publishing P_t(it) the warpgroup checks that the tiles the MMA warp reads right after
    // it have landed (the MMA warp waits only for P): PV_t(it) reads V(it); the S issued next reads
    // K(it+2) (two S buffers per tile), or in the Q0 mode K(it+1) after P0 and K(it+2) after P1.
    auto wait_kv_for_next_mmas = [&](int it) {
      if (PCR_Q0_TMEM) {
        if (PCR_KV_WAIT_ONE && r != 0) return;
        if (t == 0) {
          mbar_wait(&bars->v_full[it % kStages], (it / kStages) & 1);
          if (it + 1 < n_iter) mbar_wait(&bars->k_full[(it + 1) % kStages], ((it + 1) / kStages) & 1);
        } else if (it + 2 < n_iter) {
          mbar_wait(&bars->k_full[(it + 2) % kStages], ((it + 2) / kStages) & 1);
        }
      } else if (t == 0 && (!PCR_KV_WAIT_ONE || r == 0)) {
        mbar_wait(&bars->v_full[it % kStages], (it / kStages) & 1);
        PCR_TICK(8);
        if (it + kSBuf < n_iter) mbar_wait(&bars->k_full[(it + kSBuf) % kStages], ((it + kSBuf) / kStages) & 1);
      }
    };
#if PCR_Q0_TMEM
    if (t == 0 && n_iter > 0) {
      // Q tile 0 -> TMEM columns kColQ.. (bf16 pairs, lane = row; zero past N2).  With the streamed
      // gather (host_io: q itself arrives through the gather) every thread first acquires the layer.
      if (p.ready)
        while (ld_acquire_gpu(p.ready + p.layer) < p.ready_target) __nanosleep(64);
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (int64_t(i) * p.hq + qh) * D);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint4 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = i < p.n2 ? src[c * 8 + e] : make_uint4(0, 0, 0, 0);
        tmem_st32(lane_base + Lay::kColQ + c * 32, reinterpret_cast<const float*>(v));
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars->q_full);
    }
#endif
    for (int it = 0; it < n_iter; ++it) {
      const int key0 = tile_of(it) * kBlockN;
      const bool diag = key0 + kBlockN - 1 > tile_first_key_limit;  // tile crosses this Q tile's diagonal
      const uint32_t s_col = lane_base + s_buf_col(t, it);
      PCR_TICK(5);
      mbar_wait_warp(&bars->s_full[t][it % kSBuf], (it / kSBuf) & 1);
      tc_fence_after();
      PCR_TICK(0);
#if PCR_ATTN_TIMELINE
      if (it == 0) tl_loop0 = globaltimer_ns();
#endif
      if (PCR_ATTN_PROFILE & 1) {
        tc_fence_before();
        wait_kv_for_next_mmas(it);
        mbar_arrive(&bars->p_full[t][it % kSBuf]);
        continue;
      }
      // the tile's scores in 64-column halves (two with 128-key tiles): the row max over all of
      // them first, the last half loaded being half 0, which pass 2 then uses without a reload
      constexpr int kH = kBlockN / 64;
      float va[32], vb[32];
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      auto load_half = [&](int hh) {
        tmem_ld32(s_col + hh * 64, va);
        tmem_ld32(s_col + hh * 64 + 32, vb);
        tmem_ld_wait();
        if (diag) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            va[e] = (key0 + hh * 64 + e <= limit) ? va[e] : -INFINITY;
            vb[e] = (key0 + hh * 64 + 32 + e <= limit) ? vb[e] : -INFINITY;
          }
        }
      };
#pragma unroll 1
      for (int hh = kH - 1; hh >= 0; --hh) {
        load_half(hh);
        if (hh == kH - 1) PCR_TICK(1);
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          mx4[(e >> 2) & 1] = fmax3(mx4[(e >> 2) & 1], va[e], va[e + 1]);
          mx4[((e >> 2) & 1) + 2] = fmax3(mx4[((e >> 2) & 1) + 2], va[e + 2], va[e + 3]);
          mx4[(e >> 2) & 1] = fmax3(mx4[(e >> 2) & 1], vb[e], vb[e + 1]);
          mx4[((e >> 2) & 1) + 2] = fmax3(mx4[((e >> 2) & 1) + 2], vb[e + 2], vb[e + 3]);
        }
      }
      const float rowmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      const float m_new = fmaxf(m_raw, rowmax);
      const bool rescale = (m_new - m_raw) * p.scale_log2 > kRescaleThreshold;
      const float m_use = rescale ? m_new : m_raw;
      // a split-KV range can lie wholly past a row's causal limit: nothing visible yet
      const float neg_m = m_use == -INFINITY ? 0.f : -m_use * p.scale_log2;
      const uint64_t negm2 = f2_pack(neg_m, neg_m);
      // alpha = 2^((m_raw - m_use) * scale) is exactly 1 unless this row rescales: no MUFU op in the
      // common case (it would queue behind the other warpgroup's exponentials)
      const float alpha = rescale ? ex2(fmaf(m_raw, p.scale_log2, neg_m)) : 1.f;
      if (it > 0 && __any_sync(0xffffffffu, rescale)) {
        // O_t must hold PV_t(it-1) before it is rescaled.  S_t(it+1) is issued right after
        // PV_t(it-1) and its commit covers every earlier MMA, so its s_full phase (which this
        // warpgroup waits for next iteration anyway) certifies PV_t(it-1); the last tile has no
        // S_t(it+1) and waits on o_done, committed once after PV_t(n_iter-2).  Every barrier
        // phase thus has a waiter (compute-sanitizer synccheck clean).
        if (kSBuf == 2) {
          if (it + 1 < n_iter) mbar_wait(&bars->s_full[t][(it + 1) & 1], ((it + 1) >> 1) & 1);
          else mbar_wait(&bars->o_done[t], 0);
          tc_fence_after();
        }
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          tmem_ld32(o_col + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] *= alpha;
          tmem_st32(o_col + c * 32, o);
        }
      }
      PCR_TICK(2);
      // P = bf16(2^(s*scale - m)) (MUFU, or the FMA-pipe polynomial for kPolyPairs of every 16
      // pairs), written over the S columns it came from
      uint32_t pk[2][16];
      uint64_t rs2 = 0;   // PCR_ROWSUM_F32: packed fp32 row sum of the unrounded weights
      auto exp_chunk = [&](float* v, int c) {
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const uint64_t x2 = ffma2(f2_pack(v[e], v[e + 1]), scale2, negm2);
          float y0, y1;
          if (e >= 32 - 2 * kPolyPairs) {
            exp2_poly2(x2, y0, y1);       // FMA pipe
          } else {
            float x0, x1;
            f2_unpack(x2, x0, x1);
            y0 = ex2(x0);                 // MUFU
            y1 = ex2(x1);
          }
          __nv_bfloat162 b = __floats2bfloat162_rn(y0, y1);
          pk[c & 1][e / 2] = *reinterpret_cast<uint32_t*>(&b);
          if (PCR_ROWSUM_F32) rs2 = fadd2(rs2, f2_pack(y0, y1));
        }
        // P chunk c -> columns [16c, 16c+16): scores already consumed (128-key tiles: chunks 2, 3
        // land on half 0's columns 32-63, written after half 0 was used and half 1 reloaded)
        tmem_st16(s_col + c * 16, pk[c & 1]);
      };
#if PCR_EXP_PINGPONG
      // The two warpgroups take turns on the exponentials (they share each SMSP's MUFU): wait for
      // the other one to finish its exp phase, run ours, hand the turn back.  Tile 0 first checks
      // that V(it) and K(it+2) have landed (the MMA warp issues PV(it) and S(it+2) on P_0(it) alone);
      // those waits hide inside the wait for the turn.
      wait_kv_for_next_mmas(it);
      PCR_TICK(6);
      named_bar_sync(1 + t, 256);
      PCR_TICK(7);
#endif
#pragma unroll 1
      for (int hh = 0; hh < kH; ++hh) {
        if (hh > 0) load_half(hh);
        exp_chunk(va, 2 * hh);
        exp_chunk(vb, 2 * hh + 1);
      }
#if PCR_EXP_PINGPONG
      if (!(t == 1 && it == n_iter - 1)) named_bar_arrive(2 - t, 256);
#endif
      PCR_TICK(3);
      tmem_st_wait();
      tc_fence_before();
#if !PCR_EXP_PINGPONG
      wait_kv_for_next_mmas(it);
#endif
      mbar_arrive(&bars->p_full[t][it % kSBuf]);
      // row sum of the same bf16-rounded weights (R18), off the MMA warp's critical path:
      // fp32 += bf16 (FHADD.BF16), four independent chains
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (PCR_ROWSUM_F32) {
        f2_unpack(rs2, acc[0], acc[1]);
      } else {
        static_assert(PCR_ROWSUM_F32 || kBlockN == 64, "rounded-weight row sum: 64-key tiles only");
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 16; ++e)
            asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
                "add.rn.f32.bf16 %0, lo, %0;\n\tadd.rn.f32.bf16 %1, hi, %1;\n\t}"
                : "+f"(acc[(e & 1) * 2]), "+f"(acc[(e & 1) * 2 + 1]) : "r"(pk[c][e]));
      }
      l = l * alpha + ((acc[0] + acc[1]) + (acc[2] + acc[3]));
      PCR_TICK(4);
      m_raw = m_use;
    }
#if PCR_ATTN_TIMING
    if ((threadIdx.x & 31) == 0 && (blockIdx.x == 0 || blockIdx.x == 8 || blockIdx.x == 300) && blockIdx.z == 0)
      printf("TIMING blk %d warp %d iters %d: wait %lld ld %lld max %lld vwait %lld kwait %lld turn %lld exp %lld post %lld loop %lld\n",
             blockIdx.x, threadIdx.x >> 5, n_iter, tm_[0] / max(n_iter, 1), tm_[1] / max(n_iter, 1),
             tm_[2] / max(n_iter, 1), tm_[8] / max(n_iter, 1), tm_[6] / max(n_iter, 1), tm_[7] / max(n_iter, 1),
             tm_[3] / max(n_iter, 1), tm_[4] / max(n_iter, 1), tm_[5] / max(n_iter, 1));
#endif
    // ---------------------------------------------------------------- epilogue
#if PCR_ATTN_TIMELINE
    tl_loop1 = globaltimer_ns();
#endif
    if (p.late_dep_wait) grid_dep_wait();
    const bool row_ok = i < p.n2;
    const int64_t row_id = int64_t(i) * p.hq + qh;
    if (n_iter > 0) {
      mbar_wait(&bars->o_full, 0);
      tc_fence_after();
    }
    const float inv_l = (n_iter > 0 && l > 0.f) ? 1.f / l : 0.f;
    if (p.cluster_reduce) {
      // split-KV over a cluster: publish this row's LSE; the O rows are weighted and reduced over
      // DSMEM below, once every CTA of the cluster has published its LSEs
      ep_lse = (n_iter > 0 && l > 0.f) ? m_raw * p.scale_log2 + __log2f(l) : -INFINITY;
      ep_inv_l = inv_l;
      reinterpret_cast<float*>(smem + Lay::kLse)[t * kBlockM + r] = ep_lse;
    } else if (p.tma_epilogue) {
      // O (bf16, or the fp32 partial) -> shared memory in the TMA box layout (128-byte rows,
      // SWIZZLE_128B: 16-byte chunk c of row r at r*128 + ((c ^ r%8) << 4)), then one thread of the
      // warpgroup stores the tile with TMA: coalesced, and rows past N2 are clipped by the map.
      // Staging reuses [0, 64 KB) (bf16) or [0, 128 KB) (fp32) of the Q tiles and K ring, free once
      // o_full certifies every MMA -- and, in a writer CTA, once its pool stores have read the ring.
      const bool f32 = !(p.n_splits == 1 && p.part_o == nullptr);
      if (writer) mbar_wait(&bars->store_done, 0);
      uint8_t* stage = smem + t * (f32 ? kBlockM * D * 4 : Lay::kQTile);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        if (n_iter > 0) {
          tmem_ld32(o_col + c * 32, o);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = 0.f;
        }
        if (f32) {
          uint8_t* box = stage + c * (kBlockM * 128) + r * 128;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            *reinterpret_cast<float4*>(box + ((e ^ (r & 7)) << 4)) =
                make_float4(o[4 * e] * inv_l, o[4 * e + 1] * inv_l, o[4 * e + 2] * inv_l, o[4 * e + 3] * inv_l);
        } else {
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 b = __floats2bfloat162_rn(o[q8 * 8 + 2 * e] * inv_l, o[q8 * 8 + 2 * e + 1] * inv_l);
              w[e] = *reinterpret_cast<uint32_t*>(&b);
            }
            const int chunk = c * 4 + q8;   // 16-byte chunk of the row (8 per 64-column half)
            *reinterpret_cast<uint4*>(stage + (chunk >> 3) * Lay::kQHalf + r * 128 + (((chunk & 7) ^ (r & 7)) << 4)) =
                make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      if (f32 && row_ok)
        (p.ws_lse + int64_t(blockIdx.z) * p.n2 * p.hq)[row_id] =
            (n_iter > 0 && l > 0.f) ? m_raw * p.scale_log2 + __log2f(l) : -INFINITY;
      fence_proxy_async_smem();
      named_bar_sync(3 + t, 128);
      if (r == 0) {
        const int tok0 = i0 + t * tok_per_tile;
        if (f32) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) tma_store_4d(&tmap_out, stage + c * (kBlockM * 128), c * 32, g * G, tok0, blockIdx.z);
        } else {
#pragma unroll
          for (int hf = 0; hf < Lay::kHalves; ++hf) tma_store_3d(&tmap_out, stage + hf * Lay::kQHalf, hf * 64, g * G, tok0);
        }
        bulk_commit();
#ifndef PCR_EPI_WAIT_READ
#define PCR_EPI_WAIT_READ 1
#endif
        // the staging must have been read before the CTA's shared memory is released; the global
        // writes complete with the grid (the kernel boundary -- or the dependent's
        // griddepcontrol.wait -- orders them before any reader)
        if (PCR_EPI_WAIT_READ) bulk_wait_read<0>();
        else bulk_wait0();
      }
    } else if (p.n_splits == 1 && p.part_o == nullptr) {
      uint4* dst = reinterpret_cast<uint4*>(p.out + row_id * D);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(o_col + c * 32, o);
        tmem_ld_wait();
        if (row_ok) {
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 b = __floats2bfloat162_rn(o[q8 * 8 + 2 * e] * inv_l, o[q8 * 8 + 2 * e + 1] * inv_l);
              w[e] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[c * 4 + q8] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    } else {
      // split-KV partial: normalised O of this key range + its log2-domain LSE
      const int64_t rows_total = int64_t(p.n2) * p.hq;
      float4* dst = reinterpret_cast<float4*>(p.ws_o + (int64_t(blockIdx.z) * rows_total + row_id) * D);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        if (n_iter > 0) {
          tmem_ld32(o_col + c * 32, o);
          tmem_ld_wait();
        }
        if (row_ok) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            dst[c * 8 + e] = n_iter > 0 ? make_float4(o[4 * e] * inv_l, o[4 * e + 1] * inv_l, o[4 * e + 2] * inv_l,
                                                      o[4 * e + 3] * inv_l)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      if (row_ok)
        p.ws_lse[int64_t(blockIdx.z) * rows_total + row_id] =
            (n_iter > 0 && l > 0.f) ? m_raw * p.scale_log2 + __log2f(l) : -INFINITY;
    }
    tc_fence_before();
  }
  if (p.spin_reduce) {
    // ---------------------------------------------------------------- split-KV reduce through L2
    // The n_splits CTAs of an (M block, kv head) group wrote their partials (O normalised by their
    // own row sums, log2 LSE) to the workspace above.  The whole grid is resident (one wave, checked
    // by the launcher), so each CTA can wait for its group: thread 0 publishes the CTA's partial
    // (fence + arrival count); the last arrival resets the count and bumps the group's generation
    // (release); the others acquire the generation change.  Then CTA z merges 1/n_splits of the
    // group's (row, 8 columns) units -- out = sum_s 2^(lse_s - M) O_s / sum_s 2^(lse_s - M) -- from
    // L2, so no combine kernel runs.
    const int nsp = p.n_splits;
    if (p.late_dep_wait) grid_dep_wait();
    uint32_t* cnt = p.spin_ctr + blockIdx.x;
    uint32_t* gen = p.spin_ctr + 256 + blockIdx.x;
    __syncthreads();   // every row of this CTA's partial is written
    if (threadIdx.x == 0) {
      const uint32_t my_gen = ld_acquire_gpu_u32(gen);
      __threadfence();
      const uint32_t old = atomicAdd(cnt, 1u);
      if (old == uint32_t(nsp - 1)) {
        *cnt = 0u;
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
      } else {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_gpu_u32(gen) == my_gen) {
          __nanosleep(64);
          if (globaltimer_ns() - t0 > 10ull * 1000 * 1000 * 1000) {   // 10 s: never hang the GPU
            printf("suffix_attn: split group %d never completed\n", blockIdx.x);
            __trap();
          }
        }
      }
    }
    __syncthreads();
    const int64_t rows_total = int64_t(p.n2) * p.hq;
    constexpr int kUnits = kNQ * kBlockM * (D / 8);
    const int per = (kUnits + nsp - 1) / nsp;
    const int u_end = min(kUnits, int(blockIdx.z + 1) * per);
    for (int u = int(blockIdx.z) * per + int(threadIdx.x); u < u_end; u += kThreads) {
      const int row = u / (D / 8), grp = u % (D / 8);
      const int tt = row / kBlockM, rr = row % kBlockM;
      const int ii = i0 + tt * tok_per_tile + rr / G;
      if (ii >= p.n2) continue;
      const int64_t row_id = int64_t(ii) * p.hq + g * G + rr % G;
      float mx = -INFINITY;
      for (int sp = 0; sp < nsp; ++sp) mx = fmaxf(mx, ld_cg_f32(p.ws_lse + sp * rows_total + row_id));
      float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, wsum = 0.f;
      if (mx != -INFINITY) {
        for (int sp = 0; sp < nsp; ++sp) {
          const float w = ex2(ld_cg_f32(p.ws_lse + sp * rows_total + row_id) - mx);
          const float4* src = reinterpret_cast<const float4*>(p.ws_o + (sp * rows_total + row_id) * D + grp * 8);
          const float4 x = ld_cg_f4(src), y = ld_cg_f4(src + 1);
          wsum += w;
          a[0] += w * x.x; a[1] += w * x.y; a[2] += w * x.z; a[3] += w * x.w;
          a[4] += w * y.x; a[5] += w * y.y; a[6] += w * y.z; a[7] += w * y.w;
        }
      }
      const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
      if (p.part_o) {
        float4* dst = reinterpret_cast<float4*>(p.part_o + row_id * D + grp * 8);
        dst[0] = make_float4(a[0] * inv, a[1] * inv, a[2] * inv, a[3] * inv);
        dst[1] = make_float4(a[4] * inv, a[5] * inv, a[6] * inv, a[7] * inv);
        if (grp == 0) p.part_lse[row_id] = wsum > 0.f ? mx + __log2f(wsum) : -INFINITY;
      } else {
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 h2 = __floats2bfloat162_rn(a[2 * e] * inv, a[2 * e + 1] * inv);
          wv[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
        *reinterpret_cast<uint4*>(p.out + row_id * D + grp * 8) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
  }
  if (p.cluster_reduce) {
    // ---------------------------------------------------------------- split-KV cluster reduce
    // The n_splits CTAs of a cluster (cluster dims (1, 1, n_splits): rank == blockIdx.z) hold the
    // partials of the same rows over disjoint key ranges.  (1) every row's merged weights from the
    // n_splits LSEs, (2) each CTA writes its partial O row times its weight 2^(lse_s - M) / Z into
    // its own shared memory, (3) CTA s sums its 1/n_splits share of the (row, 8 columns) units over
    // the cluster's DSMEM and writes the output -- no workspace, no second kernel.
    const int nsp = p.n_splits;
    if (p.late_dep_wait) grid_dep_wait();
    float* lse_own = reinterpret_cast<float*>(smem + Lay::kLse);
    float* lse_merged = lse_own + kNQ * kBlockM;
    cluster_sync_all();   // #1: every CTA's row LSEs are visible cluster-wide
    if (warp >= 4) {
      const int tr = threadIdx.x - 128;   // row of this CTA's kNQ * 128
      float M = -INFINITY;
      for (int sp = 0; sp < nsp; ++sp) M = fmaxf(M, ld_dsmem_f32(dsmem_addr(&lse_own[tr], sp)));
      float Z = 0.f;
      if (M != -INFINITY)
        for (int sp = 0; sp < nsp; ++sp) Z += ex2(ld_dsmem_f32(dsmem_addr(&lse_own[tr], sp)) - M);
      const float w = (M == -INFINITY || ep_lse == -INFINITY) ? 0.f : ex2(ep_lse - M) / Z;
      lse_merged[tr] = M == -INFINITY ? -INFINITY : M + __log2f(Z);
      if (writer) mbar_wait(&bars->store_done, 0);   // the K/V ring is no longer read by pool stores
      float4* part = reinterpret_cast<float4*>(smem + Lay::kK0) + tr * (D / 4);
      const float sc = w * ep_inv_l;
      const uint32_t o_col = tmem + (uint32_t(((warp & 3) * 32)) << 16) + Lay::kColO + ((warp - 4) >> 2) * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        if (n_iter > 0) {
          tmem_ld32(o_col + c * 32, o);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e)
          part[(c * 8 + e) ^ (tr & (D / 4 - 1))] =
              make_float4(o[4 * e] * sc, o[4 * e + 1] * sc, o[4 * e + 2] * sc, o[4 * e + 3] * sc);
      }
    }
    cluster_sync_all();   // #2: every CTA's weighted partials are visible
    constexpr int kUnits = kNQ * kBlockM * (D / 8);
    const int per = (kUnits + nsp - 1) / nsp;
    const int u_end = min(kUnits, int(blockIdx.z + 1) * per);
    const uint32_t part_base = smem_u32(smem + Lay::kK0);
    for (int u = int(blockIdx.z) * per + int(threadIdx.x); u < u_end; u += kThreads) {
      const int row = u / (D / 8), grp = u % (D / 8);
      const int tt = row / kBlockM, rr = row % kBlockM;
      const int ii = i0 + tt * tok_per_tile + rr / G;
      if (ii >= p.n2) continue;
      const int64_t row_id = int64_t(ii) * p.hq + g * G + rr % G;
      const int sw = row & (D / 4 - 1);
      const uint32_t off0 = uint32_t(row * (D / 4) + ((2 * grp) ^ sw)) * 16;
      const uint32_t off1 = uint32_t(row * (D / 4) + ((2 * grp + 1) ^ sw)) * 16;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      for (int sp = 0; sp < nsp; ++sp) {
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(part_base + off0), "r"(sp));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(part_base + off1), "r"(sp));
        const float4 x = ld_dsmem_f32x4(ra), y = ld_dsmem_f32x4(rb);
        a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
        b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
      }
      if (p.part_o) {
        float4* dst = reinterpret_cast<float4*>(p.part_o + row_id * D + grp * 8);
        dst[0] = a;
        dst[1] = b;
        if (grp == 0) p.part_lse[row_id] = lse_merged[row];
      } else {
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
          wv[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
        *reinterpret_cast<uint4*>(p.out + row_id * D + grp * 8) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
    cluster_sync_all();   // #3: no CTA leaves while its shared memory may still be read
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
#if PCR_ATTN_TIMELINE
  if (threadIdx.x == 128) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const uint32_t cta = blockIdx.z * gridDim.x + blockIdx.x;
    if (p.layer < kTlLayers && cta < kTlCtas) {
      unsigned long long* rec = g_timeline[p.layer][cta];
      rec[0] = tl_start;
      rec[1] = tl_loop0;
      rec[2] = tl_loop1;
      rec[3] = globaltimer_ns();
      rec[4] = smid;
      rec[5] = uint64_t(n_iter);
    }
  }
#endif
}

// Merge split-KV partials: out = sum_s 2^(lse_s - M) O_s / sum_s 2^(lse_s - M), M = max_s lse_s.
// Part s lives at ws_o + s*o_stride (rows x D) and ws_lse + s*lse_stride.  part_o != null: write
// the merged fp32 O and log2-domain LSE (this rank's partial, context split) instead of bf16.
template <int D>
__global__ void __launch_bounds__(256) combine_kernel(const float* __restrict__ ws_o, int64_t o_stride,
                                                      const float* __restrict__ ws_lse, int64_t lse_stride,
                                                      uint16_t* __restrict__ out, float* __restrict__ part_o,
                                                      float* __restrict__ part_lse, int64_t rows_total, int n_splits) {
  constexpr int kVec = D / 8;  // 8 outputs (one 16-byte store) per thread
  const int64_t n = rows_total * kVec;
  grid_dep_wait();   // PDL: the partials are complete and visible past this point
  grid_dep_launch(); // the next layer's attention may start its main loop while this merge runs
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = u / kVec;
    const int c8 = int(u % kVec) * 8;
    // The loads of a group of 4 splits are issued before any of them is used (the loop is
    // latency-bound otherwise); the accumulation order over s is unchanged.
    float mx = -INFINITY;
#pragma unroll 8
    for (int s = 0; s < n_splits; ++s) mx = fmaxf(mx, ws_lse[s * lse_stride + row]);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, wsum = 0.f;
    if (mx != -INFINITY) {
      for (int s0 = 0; s0 < n_splits; s0 += 4) {
        float lse[4];
        float4 a[4], b[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (s0 + k < n_splits) {
            const int s = s0 + k;
            lse[k] = ws_lse[s * lse_stride + row];
            const float4* src = reinterpret_cast<const float4*>(ws_o + s * o_stride + row * D + c8);
            a[k] = src[0];
            b[k] = src[1];
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (s0 + k < n_splits) {
            const float w = ex2(lse[k] - mx);
            wsum += w;
            acc[0] += w * a[k].x; acc[1] += w * a[k].y; acc[2] += w * a[k].z; acc[3] += w * a[k].w;
            acc[4] += w * b[k].x; acc[5] += w * b[k].y; acc[6] += w * b[k].z; acc[7] += w * b[k].w;
          }
        }
      }
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    if (part_o) {
      float4* dst = reinterpret_cast<float4*>(part_o + row * D + c8);
      dst[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      dst[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
      if (c8 == 0) part_lse[row] = wsum > 0.f ? mx + __log2f(wsum) : -INFINITY;
      continue;
    }
    uint32_t wv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * e] * inv, acc[2 * e + 1] * inv);
      wv[e] = *reinterpret_cast<uint32_t*>(&b);
    }
    *reinterpret_cast<uint4*>(out + row * D + c8) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

// Programmatic dependent launch (PCR_PDL=0 disables): the grid may be scheduled while the kernel
// before it in the stream drains; its griddepcontrol.wait then orders every dependent read.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, int cluster_z,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_z > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = 1;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = cluster_z;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Experiment (PCR_SPLIT_CLUSTER=1): split-KV partials reduced inside the attention kernel over a
// thread-block cluster (DSMEM) instead of the fp32 workspace + combine kernel.  Measured slower on
// this pool's B200 (profiles/r02_split_cluster.txt): only 15 clusters of 8 fit at once (GPC sizes),
// and the in-kernel epilogue costs more than the combine launch it saves, so it is off by default.
bool split_cluster_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_SPLIT_CLUSTER");
    return e && e[0] == '1';
  }();
  return on;
}

// Experiment (PCR_SPLIT_SPIN=1): split-KV partials merged inside the attention kernel through L2
// when its grid is one wave and no other request is active, instead of the combine kernel.
// Bit-identical output, half the launches, but no faster: the short-suffix layer measured 29.3-29.5
// vs 27.7-27.8 us alone and 10.58 vs 10.66 ms L8 TTFT in the pipeline (profiles/r02_split_spin.txt)
// -- the combine kernel's launch is already hidden by PDL -- so it is off by default.
bool split_spin_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_SPLIT_SPIN");
    return e && e[0] == '1';
  }();
  return on;
}

// TMA-store epilogue (PCR_TMA_EPILOGUE=0 restores the per-thread row stores).
bool tma_epilogue_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_TMA_EPILOGUE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// SMs the split-KV sizing may count on (PCR_ATTN_SMS overrides).  136 of the 148: the split grid
// then leaves ~12 SMs free, where the next layer's attention CTAs (programmatic dependent launch)
// start while this layer's last CTAs and its combine drain.  L8 short-suffix layer (16 M-block x
// head pairs: 8 splits = 128 CTAs instead of 9 = 144): 18.6-18.8 vs 20.8 us, six alternating
// runs each (profiles/r02_short_suffix_split_count.txt); the L70 rank slice at r = 1 +1%.
int attn_sm_budget() {
  static const int n = [] {
    const char* e = std::getenv("PCR_ATTN_SMS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 && v <= 148 ? v : 136;
  }();
  return n;
}

template <int D>
cudaError_t launch_d(const CUtensorMap* tmap_pool, const AttnParams& p0, cudaStream_t stream, int* launches) {
  // act[s] = clusters of s CTAs (one per SM: ~194 KB smem) that can be resident at once, s <= 16.
  // GPCs differ in SM count, so e.g. 16 clusters of 9 may not fit in one wave while 16 of 8 do.
  // (One-time setup behind a thread-safe function-local static.)
  struct Setup {
    int act[17] = {0};
    cudaError_t err = cudaSuccess;
  };
  auto kern = suffix_attn_kernel<D>;
  static const Setup setup = [kern] {
    Setup su;
    su.err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Layout<D>::kAlloc);
    if (su.err != cudaSuccess) return su;
    const bool np = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    for (int cs = 1; cs <= (np ? 16 : 8); ++cs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1, 1, cs);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = Layout<D>::kAlloc;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 1;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = cs;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      su.act[cs] = cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess ? n : 0;
    }
    cudaGetLastError();
    if (const char* dbg = std::getenv("PCR_DEBUG"); dbg && dbg[0] == '1') {
      std::fprintf(stderr, "suffix_attn<%d> max active clusters by size:", D);
      for (int cs = 1; cs <= 16; ++cs) std::fprintf(stderr, " %d:%d", cs, su.act[cs]);
      std::fprintf(stderr, "\n");
    }
    return su;
  }();
  if (setup.err != cudaSuccess) return setup.err;
  const int* act = setup.act;
  AttnParams p = p0;
  const int G = p.hq / p.hkv;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // Q tensor map over q [N2][Hq][D]: box {64, G, 128/G} lands a Q tile as rows r = t*G + gg.
  CUtensorMap tmap_q, tmap_kn, tmap_vn;
  {
    cuuint64_t dims[3] = {cuuint64_t(D), cuuint64_t(p.hq), cuuint64_t(p.n2)};
    cuuint64_t strides[2] = {cuuint64_t(D) * 2, cuuint64_t(p.hq) * D * 2};
    cuuint32_t box[3] = {64, cuuint32_t(G), cuuint32_t(kBlockM / G)};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&tmap_q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(p.q), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  tmap_kn = tmap_vn = tmap_q;   // (unused unless the append is fused)
  if (p.k_new) {
    // suffix K / V [N2][hkv][D]: box {64, 1, pool box rows} lands exactly like a pool box; rows past
    // N2 are zero-filled by the TMA unit
    cuuint64_t dims[3] = {cuuint64_t(D), cuuint64_t(p.hkv), cuuint64_t(p.n2)};
    cuuint64_t strides[2] = {cuuint64_t(D) * 2, cuuint64_t(p.hkv) * D * 2};
    cuuint32_t box[3] = {64, 1, cuuint32_t(std::min(p.S, kBlockN))};
    cuuint32_t estr[3] = {1, 1, 1};
    for (int kv = 0; kv < 2; ++kv)
      if (enc(kv ? &tmap_vn : &tmap_kn, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
              const_cast<uint16_t*>(kv ? p.v_new : p.k_new), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
  }
  const int tok_per_cta = kNQ * kBlockM / G;
  const int n_mblocks = (p.n2 + tok_per_cta - 1) / tok_per_cta;
  // Split-KV when the (m-block x kv-head) grid leaves SMs idle; each split keeps >= 2 key tiles.
  const int ctas = n_mblocks * p.hkv;
  const int max_tiles = (p.n1 + p.n2 + kBlockN - 1) / kBlockN;
  const bool cluster_ok = split_cluster_enabled();
  int splits = 1;
  const int sms = attn_sm_budget();
  // Split only small grids (< 48 CTAs): a split-KV layer ends in a combine that waits for every
  // split, while an unsplit grid of >= ~1/3 of the SMs lets the next layer's CTAs run beside it
  // (programmatic dependent launch) -- M7 r=0.5 per-rank slice at P = 8 (66 CTAs): 2.53 -> 1.70 ms
  // TTFT unsplit; 34 and 18 CTAs (r = 0.75 / 0.875) and L8 (16) stay faster split
  // (profiles/r02_split_threshold.txt).
#ifndef PCR_SPLIT_MAX_CTAS
#define PCR_SPLIT_MAX_CTAS 48
#endif
  constexpr int kSplitMaxCtas = PCR_SPLIT_MAX_CTAS;
  if ((p.ws_o || cluster_ok) && ctas < std::min(sms, kSplitMaxCtas)) {   // (kv_len < n1 + n2 only shortens the key range)
    splits = std::max(1, sms / ctas);
    splits = std::min(splits, std::max(1, max_tiles / PCR_SPLIT_MIN_TILES));
    if (cluster_ok) {
      // the largest cluster size whose clusters all fit in one wave beside each other
      const char* cap = std::getenv("PCR_MAX_CLUSTER");
      splits = std::min(splits, cap ? std::max(1, std::atoi(cap)) : 16);
      while (splits > 1 && act[splits] < ctas) --splits;
    } else {
      const int64_t per_split_bytes = int64_t(p.n2) * p.hq * (D + 1) * 4;
      splits = int(std::min<int64_t>(splits, std::max<int64_t>(1, p.ws_bytes / per_split_bytes)));
    }
  }
  p.n_splits = splits;
  p.cluster_reduce = (splits > 1 && cluster_ok) ? 1 : 0;
  // in-kernel reduce through L2 when the whole grid is one wave (every group's splits resident)
  p.spin_reduce = (splits > 1 && !p.cluster_reduce && p.spin_ctr && split_spin_enabled() && ctas <= 256 &&
                   int64_t(ctas) * splits <= act[1])
                      ? 1 : 0;
  if (p.part_o && splits == 1) {   // one split: the kernel writes the partial itself
    p.ws_o = p.part_o;
    p.ws_lse = p.part_lse;
  }
  // fused-append placement (see the kernel): the owning CTAs when the whole grid is one wave, the
  // suffix spans more than 4 key tiles, and either the grid is split-KV (the combine waits for
  // every split, so the last M-block's CTAs, storing every suffix tile, are the layer's critical
  // path) or the suffix is >= 70% of the keys (those CTAs store nearly every tile they load);
  // otherwise the next layer's CTAs absorb their extra time.  Same-box A/B (M7 per-rank slices,
  // TTFT): P = 8 r = 0.5 (2 splits) 3.71 -> 2.53 ms, r = 0 2.58-2.66 -> 2.08-2.13, r = 0.25
  // 2.18-2.22 -> 1.97; kept on the last M-block: P = 4 r = 0.5 2.97-2.99 (3.07 with the owners),
  // P = 4 r = 0 (two waves) 3.85-3.88 (3.97-3.98).  PCR_APPEND_OWNER=0 / 1 forces either placement.
  {
    static const int force = [] {
      const char* e = std::getenv("PCR_APPEND_OWNER");
      return e ? std::atoi(e) : -1;
    }();
    const bool one_wave = int64_t(ctas) * splits <= 148;
    const bool long_sfx = p.n2 > 4 * kBlockN;
    const bool heavy = splits > 1 || int64_t(p.n2) * 10 >= int64_t(p.n1 + p.n2) * 7;
    p.append_owner = force >= 0 ? (force ? 1 : 0) : (one_wave && long_sfx && heavy ? 1 : 0);
  }
  // TMA-store epilogue (PCR_TMA_EPILOGUE=0: one row per thread from registers): bf16 out as a 3D
  // map like q's, or the fp32 partial [splits][N2][Hq][D] as a 4D map with 32-float (128-byte) boxes
  CUtensorMap tmap_out = tmap_q;
  p.tma_epilogue = 0;
  if (tma_epilogue_enabled() && !p.cluster_reduce && !p.spin_reduce) {
    const bool f32 = !(splits == 1 && p.part_o == nullptr);
    CUresult r;
    if (f32) {
      cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(p.hq), cuuint64_t(p.n2), cuuint64_t(splits)};
      cuuint64_t strides[3] = {cuuint64_t(D) * 4, cuuint64_t(p.hq) * D * 4, cuuint64_t(p.n2) * p.hq * D * 4};
      cuuint32_t box[4] = {32, cuuint32_t(G), cuuint32_t(kBlockM / G), 1};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      r = enc(&tmap_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.ws_o, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[3] = {cuuint64_t(D), cuuint64_t(p.hq), cuuint64_t(p.n2)};
      cuuint64_t strides[2] = {cuuint64_t(D) * 2, cuuint64_t(p.hq) * D * 2};
      cuuint32_t box[3] = {64, cuuint32_t(G), cuuint32_t(kBlockM / G)};
      cuuint32_t estr[3] = {1, 1, 1};
      r = enc(&tmap_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p.out, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    p.tma_epilogue = r == CUDA_SUCCESS ? 1 : 0;
  }
  dim3 grid(n_mblocks * p.hkv, 1, splits);
  cudaError_t e = launch_pdl(kern, grid, dim3(kThreads), Layout<D>::kAlloc, stream, p.cluster_reduce ? splits : 1,
                             *tmap_pool, tmap_q, tmap_kn, tmap_vn, tmap_out, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  *launches += 1;
  if (splits > 1 && !p.cluster_reduce && !p.spin_reduce) {
    const int64_t rows_total = int64_t(p.n2) * p.hq;
    int64_t blocks = (rows_total * (D / 8) + 255) / 256;
    blocks = std::min<int64_t>(blocks, 148 * 8);
    e = launch_pdl(combine_kernel<D>, dim3(int(blocks)), dim3(256), 0, stream, 1, (const float*)p.ws_o,
                   rows_total * D, (const float*)p.ws_lse, rows_total, p.out, p.part_o, p.part_lse, rows_total,
                   splits);
    if (e == cudaSuccess) e = cudaGetLastError();
    *launches += 1;
  }
  return e;
}

}  // namespace

int32_t attn_pool_box_rows(int32_t S) { return std::min(S, kBlockN); }

cudaError_t launch_merge_partials(const float* o, int64_t o_stride, const float* lse, int64_t lse_stride,
                                  int32_t n_parts, int64_t rows, int32_t d, uint16_t* out, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  int64_t blocks = std::min<int64_t>((rows * (d / 8) + 255) / 256, 148 * 8);
  if (d == 128)
    combine_kernel<128><<<int(blocks), 256, 0, stream>>>(o, o_stride, lse, lse_stride, out, nullptr, nullptr, rows,
                                                         n_parts);
  else if (d == 64)
    combine_kernel<64><<<int(blocks), 256, 0, stream>>>(o, o_stride, lse, lse_stride, out, nullptr, nullptr, rows,
                                                        n_parts);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_suffix_attn(const CUtensorMap* tmap_pool, const AttnParams& p, int32_t d, cudaStream_t stream,
                               int* launches) {
  if (p.n2 <= 0) return cudaSuccess;
  if (d == 128) return launch_d<128>(tmap_pool, p, stream, launches);
  if (d == 64) return launch_d<64>(tmap_pool, p, stream, launches);
  return cudaErrorInvalidValue;
}

}  // namespace pcr

#if PCR_ATTN_TIMELINE
extern "C" int pcr_debug_attn_timeline(void* host_dst, long long bytes) {
  const long long n = sizeof(pcr::g_timeline) < (unsigned long long)bytes ? (long long)sizeof(pcr::g_timeline) : bytes;
  if (cudaMemcpyFromSymbol(host_dst, pcr::g_timeline, size_t(n)) != cudaSuccess) return -1;
  return 0;
}
extern "C" int pcr_debug_attn_timeline_clear() {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, pcr::g_timeline) != cudaSuccess) return -1;
  return cudaMemset(p, 0, sizeof(pcr::g_timeline)) == cudaSuccess ? 0 : -1;
}
#endif
