// a4 — suffix-query causal attention over the paged pool (prefix + suffix KV), sm_100a.
//
// What it computes (R2/R3): for local query head h (kv head g = h / G) and
// suffix row i at absolute position p = n1 + i,
//     out[i][h] = sum_{j<=p} exp(s_j - m) V[j][g] / sum_{j<=p} exp(s_j - m),  s_j = q[i][h].K[j][g]/sqrt(d)
// with bf16 inputs, fp32 accumulation and bf16 output.
//
// B200 design: one CTA per (128-row M tile, kv head).  M rows pack
// (token, head-in-group) pairs, row r = t*G + gg, so one K/V tile read serves all G query heads
// of the group.  Keys are processed in tiles of 128:
//   warp 0  TMA producer: K and V pages of the tile -> smem (2D tensor map over the pool,
//           one box of {64 dims, S_pg rows} per page-half, SWIZZLE_128B), 2-stage ring;
//   warp 1  MMA issuer (one thread): S = Q K^T into TMEM (double-buffered, 2 x 128 columns),
//           then O += P V into TMEM (D columns), tcgen05.commit -> mbarriers;
//   warp 2  TMEM allocator (512 columns);
//   warps 4-7 softmax / correction / epilogue, one thread per M row (TMEM lane): tcgen05.ld of
//           its S row, causal mask on the diagonal tiles only, online softmax in the log2
//           domain with lazy rescaling of O (only when the running max grows by > 8, so P <= 256),
//           P as bf16 into smem in the UMMA K-major SWIZZLE_128B layout, final O / l -> bf16.
#include <cuda_bf16.h>

#include <cstdio>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace pcr {
namespace {

using namespace ptx;

constexpr int kBlockM = 128;
constexpr int kBlockN = 128;
constexpr int kThreads = 256;
constexpr int kHalfBytes = 128 * 128;  // 128 rows x 128 bytes (64 bf16) per swizzle column block
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int D>
struct Layout {
  static constexpr int kHalves = D / 64;
  static constexpr int kQ = 0;
  static constexpr int kQBytes = kHalves * kHalfBytes;
  static constexpr int kTileBytes = kHalves * kHalfBytes;  // one K or V tile of 128 keys
  static constexpr int kK0 = kQ + kQBytes;
  static constexpr int kV0 = kK0 + 2 * kTileBytes;
  static constexpr int kP = kV0 + 2 * kTileBytes;
  static constexpr int kPBytes = 2 * kHalfBytes;           // 128 rows x 128 keys
  static constexpr int kBar = kP + kPBytes;
  static constexpr int kBytes = kBar + 256;
  static constexpr int kAlloc = kBytes + 1024;              // slack for 1024-byte alignment
};

struct Bars {
  uint64_t k_full[2], v_full[2], kv_empty[2], s_full[2], s_empty[2], p_full, o_done, q_full;
  uint32_t tmem_base;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    suffix_attn_kernel(const __grid_constant__ CUtensorMap tmap, const AttnParams p) {
  using Lay = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + Lay::kBar);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.y;                 // local kv head
  const int G = p.hq / p.hkv;
  const int tok_per_tile = kBlockM / G;
  const int i0 = blockIdx.x * tok_per_tile;
  const int i_end = min(i0 + tok_per_tile, p.n2);
  const int n_tiles = (p.n1 + i_end + kBlockN - 1) / kBlockN;
  const int pages_per_tile = kBlockN / p.S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->kv_empty[s], 1);
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->s_empty[s], 128);
    }
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->o_done, 1);
    mbar_init(&bars->q_full, 128);
    fence_mbar_init();
    tma_prefetch_desc(&tmap);
  }
  if (warp == 2) tmem_alloc<kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      const int64_t layer_rows = p.n_pool_pages * p.hkv * 2 * p.S;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&bars->kv_empty[st], ((j >> 1) - 1) & 1);
        uint8_t* ks = smem + Lay::kK0 + st * Lay::kTileBytes;
        uint8_t* vs = smem + Lay::kV0 + st * Lay::kTileBytes;
        mbar_arrive_expect_tx(&bars->k_full[st], Lay::kTileBytes);
        mbar_arrive_expect_tx(&bars->v_full[st], Lay::kTileBytes);
        for (int pp = 0; pp < pages_per_tile; ++pp) {
          const int pidx = min(j * pages_per_tile + pp, p.n_req_pages - 1);  // clamp: finite, masked
          const int64_t page = p.pages[pidx];
          const int64_t row_k = int64_t(p.layer) * layer_rows + ((page * p.hkv + g) * 2 + 0) * p.S;
          const int64_t row_v = row_k + p.S;
#pragma unroll
          for (int hf = 0; hf < Lay::kHalves; ++hf) {
            tma_load_2d(ks + hf * kHalfBytes + pp * p.S * 128, &tmap, hf * 64, int32_t(row_k), &bars->k_full[st]);
            tma_load_2d(vs + hf * kHalfBytes + pp * p.S * 128, &tmap, hf * 64, int32_t(row_v), &bars->v_full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kBlockM, kBlockN, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kBlockM, D, 0, 1);
      const uint32_t q_addr = smem_u32(smem + Lay::kQ);
      const uint32_t p_addr = smem_u32(smem + Lay::kP);
      mbar_wait(&bars->q_full, 0);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&bars->k_full[st], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&bars->s_empty[st], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + Lay::kK0 + st * Lay::kTileBytes);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
          mma_bf16_ss(tmem + st * kBlockN, smem_desc_sw128(q_addr + off, 16, 1024),
                      smem_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0);
        }
        mma_commit(&bars->s_full[st]);
      };
      issue_s(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) issue_s(j + 1);
        const int st = j & 1;
        mbar_wait(&bars->p_full, j & 1);
        mbar_wait(&bars->v_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(smem + Lay::kV0 + st * Lay::kTileBytes);
#pragma unroll
        for (int kk = 0; kk < kBlockN / 16; ++kk) {
          const uint32_t poff = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
          mma_bf16_ss(tmem + 2 * kBlockN, smem_desc_sw128(p_addr + poff, 16, 1024),
                      smem_desc_sw128(v_addr + kk * 2048, kHalfBytes, 1024), idesc_o, (j > 0 || kk > 0));
        }
        mma_commit(&bars->o_done);
        mma_commit(&bars->kv_empty[st]);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax / epilogue
    const int r = threadIdx.x - 128;             // M row == TMEM lane
    const int i = i0 + r / G;                     // suffix token of this row
    const int qh = g * G + (r % G);               // local query head
    const uint32_t lane_addr = tmem + (uint32_t((warp & 3) * 32) << 16);
    {
      uint8_t* qs = smem + Lay::kQ;
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (int64_t(i) * p.hq + qh) * D);
#pragma unroll
      for (int c16 = 0; c16 < D / 8; ++c16) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (i < p.n2) v = src[c16];
        const int hf = c16 >> 3, cc = c16 & 7;
        *reinterpret_cast<uint4*>(qs + hf * kHalfBytes + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
      }
      fence_proxy_async_smem();
      mbar_arrive(&bars->q_full);
    }
    const int limit = p.n1 + i;                   // last visible key of this row
    float m = -INFINITY, l = 0.f;
    uint8_t* ps = smem + Lay::kP;
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      mbar_wait(&bars->s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[kBlockN];
#pragma unroll
      for (int c = 0; c < kBlockN / 32; ++c) tmem_ld32(lane_addr + st * kBlockN + c * 32, s + c * 32);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars->s_empty[st]);
      const int key0 = j * kBlockN;
      float rowmax = -INFINITY;
      if (key0 + kBlockN - 1 > p.n1 + i0) {       // diagonal tile(s): causal mask
#pragma unroll
        for (int c = 0; c < kBlockN; ++c) {
          s[c] = (key0 + c <= limit) ? s[c] * p.scale_log2 : -INFINITY;
          rowmax = fmaxf(rowmax, s[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < kBlockN; ++c) {
          s[c] *= p.scale_log2;
          rowmax = fmaxf(rowmax, s[c]);
        }
      }
      const float m_new = fmaxf(m, rowmax);
      const float m_use = (m_new > m + kRescaleThreshold) ? m_new : m;
      const float alpha = ex2(m - m_use);
      float rowsum = 0.f;
      uint32_t pk[kBlockN / 2];
#pragma unroll
      for (int c = 0; c < kBlockN; c += 2) {
        const float e0 = ex2(s[c] - m_use), e1 = ex2(s[c + 1] - m_use);
        __nv_bfloat162 b = __floats2bfloat162_rn(e0, e1);
        // l sums the SAME bf16-rounded weights the PV product uses, so out = sum(w v)/sum(w)
        // is an exact convex combination of V rows (no numerator/denominator mismatch).
        rowsum += __low2float(b) + __high2float(b);
        pk[c / 2] = *reinterpret_cast<uint32_t*>(&b);
      }
      l = l * alpha + rowsum;
      if (j > 0) {
        mbar_wait(&bars->o_done, (j - 1) & 1);   // PV(j-1) done: O stable, P buffer free
        tc_fence_after();
        if (__any_sync(0xffffffffu, m_use != m)) {
          float o[32];
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            tmem_ld32(lane_addr + 2 * kBlockN + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= alpha;
            tmem_st32(lane_addr + 2 * kBlockN + c * 32, o);
          }
          tmem_st_wait();
        }
      }
#pragma unroll
      for (int c16 = 0; c16 < kBlockN / 8; ++c16) {
        const int hf = c16 >> 3, cc = c16 & 7;
        *reinterpret_cast<uint4*>(ps + hf * kHalfBytes + r * 128 + ((cc ^ (r & 7)) << 4)) =
            make_uint4(pk[c16 * 4 + 0], pk[c16 * 4 + 1], pk[c16 * 4 + 2], pk[c16 * 4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->p_full);
      m = m_use;
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(&bars->o_done, (n_tiles - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l;
    uint4* dst = reinterpret_cast<uint4*>(p.out + (int64_t(i) * p.hq + qh) * D);
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      tmem_ld32(lane_addr + 2 * kBlockN + c * 32, o);
      tmem_ld_wait();
      if (i < p.n2) {
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
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

template <int D>
cudaError_t launch_d(const CUtensorMap* tmap, const AttnParams& p, cudaStream_t stream) {
  static bool configured = false;
  auto kern = suffix_attn_kernel<D>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Layout<D>::kAlloc);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int G = p.hq / p.hkv;
  const int tok_per_tile = kBlockM / G;
  dim3 grid((p.n2 + tok_per_tile - 1) / tok_per_tile, p.hkv);
  kern<<<grid, kThreads, Layout<D>::kAlloc, stream>>>(*tmap, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_suffix_attn(const CUtensorMap* tmap, const AttnParams& p, int32_t d, cudaStream_t stream) {
  if (p.n2 <= 0) return cudaSuccess;
  if (d == 128) return launch_d<128>(tmap, p, stream);
  if (d == 64) return launch_d<64>(tmap, p, stream);
  return cudaErrorInvalidValue;
}

}  // namespace pcr
