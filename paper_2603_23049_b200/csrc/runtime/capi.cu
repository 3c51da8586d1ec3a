// libpcr.so — the C-ABI of include/pcr.h: context, pinned DRAM store, device plan tables,
// TMA descriptor over the pool, and the per-layer stream/event pipeline.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../../include/pcr.h"
#include "../host/blake2b.h"
#include "../host/planner.h"
#include "../kernels/kernels.h"
#include "nccl_dl.h"
#include "ssd_io.h"

using pcr::Planner;
using pcr::Request;

struct pcr_ctx {
  pcr_config cfg{};
  int32_t hkv = 0, hq = 0, G = 0;
  bool ctx_split = false;          // shard_mode 1
  int64_t chunk_cap = 0;           // chunk entries per plan region
  float* part_scratch = nullptr;   // shard_mode 1 + all-gather: [L][block] partials (grown on demand)
  int64_t part_scratch_floats = 0;
  int64_t slot_elems = 0, slot_bytes = 0, page_elems_all_layers = 0, n_pool_pages = 0;
  std::unique_ptr<Planner> planner;
  bool device = false;
  // pinned DRAM store (library-owned)
  void* store = nullptr;
  size_t store_bytes = 0;
  bool registered = false;
  void* store_dev = nullptr;
  // device plan arena: max_inflight regions of [pages | slots] int32
  int32_t max_regions = 0;
  int64_t region_words = 0, region_page_cap = 0;
  int32_t* h_arena = nullptr;
  int32_t* d_arena = nullptr;
  std::vector<cudaEvent_t> region_ev;
  CUtensorMap tmap{};
  std::vector<cudaEvent_t> ev_load;
  cudaEvent_t ev_join = nullptr;
  std::vector<cudaEvent_t> ev_t;  // timing: 4 per layer
  std::string err;
  int64_t launches = 0;
  int64_t ce_copies = 0, ce_layer_loads = 0, sm_layer_loads = 0;   // a2 load-path counters (pcr_stats)
  pcr::KvGeom geom{};
  int32_t gather_ctas = 8;   // (profiles/r02_sm_partition.txt: 8 CTAs load as fast as 16, and slow the attention beside them less)
  // split-KV workspace, one slice of ws_region_floats per plan region: ws_floats partial-O
  // floats followed by the LSE floats
  float* ws = nullptr;
  int64_t ws_floats = 0, ws_region_floats = 0;
  int32_t device_active = 0;       // planned requests whose device work has been issued (not released)
  // multi-GPU output re-assembly (§8(e))
  void* nccl_comm = nullptr;
  std::unique_ptr<pcr::SsdIo> ssd;    // SSD tier I/O thread (f2)
  std::vector<int64_t> slot_write_seq; // per DRAM slot: last write-back task reading it
  std::vector<int64_t> slot_read_seq;  // per DRAM slot: last SSD read task filling it
  std::unordered_map<int64_t, int64_t> req_load_seq;  // request -> last SSD load it started
  std::vector<void*> ce_dst, ce_src;  // copy-engine baseline runs (load_mode 1/2/4)
  std::vector<size_t> ce_size;
  std::vector<cudaEvent_t> ev_attn;
  cudaEvent_t ev_comm = nullptr;
  cudaEvent_t ev_off = nullptr;
  // host_io staging (pcr_run_opts.host_io): [2][q | k | v | out] of one layer, grown on demand
  uint16_t* io_buf = nullptr;
  int64_t io_buf_elems = 0;
  cudaStream_t io_d2h = nullptr;
  std::vector<cudaEvent_t> ev_outdone;   // per layer: output copied back
  // load_mode 4: the copy-engine share of the gather runs on this stream, forked/joined per layer
  cudaStream_t ce_stream = nullptr;
  cudaEvent_t ev_ce_fork = nullptr, ev_ce_join = nullptr;
  cudaEvent_t ev_io_join = nullptr;
  // streamed gather: per plan region, L per-layer completion counters (device); the ones the
  // attention launches of the current pcr_run_prefill call wait on (null outside such a call)
  int32_t* d_ready = nullptr;
  cudaEvent_t ev_ready_zero = nullptr;
  // The streamed gather runs on a library-owned stream of the device's greatest priority, forked
  // from and joined back into the caller's load stream: its CTAs are dispatched ahead of the
  // attention grid's pending CTAs, which wait in-kernel for its per-layer counters (without the
  // priority a full attention grid queued first could keep the gather from ever being scheduled).
  cudaStream_t gather_hi = nullptr;
  cudaEvent_t ev_gather_fork = nullptr, ev_gather_join = nullptr;
  const int32_t* cur_ready = nullptr;
  int32_t cur_ready_target = 0;
};

namespace {

pcr_status fail(const pcr_ctx* c, pcr_status s, const std::string& msg) {
  if (c) const_cast<pcr_ctx*>(c)->err = msg;
  return s;
}

pcr_status cuda_fail(const pcr_ctx* c, cudaError_t e, const char* what) {
  return fail(c, PCR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(ctx, call)                                   \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);  \
  } while (0)

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

// NUMA node of the GPU from sysfs (-1 if unknown) and MPOL_PREFERRED placement of the store.
int gpu_numa_node(int dev) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) return -1;
  for (char* p = bus; *p; ++p) *p = static_cast<char>(tolower(*p));
  std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = fopen(path.c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node;
}

void bind_to_node(void* p, size_t bytes, int node) {
  if (node < 0 || node >= 64) return;
  unsigned long mask = 1UL << node;
  const int kMpolPreferred = 1;
  syscall(SYS_mbind, p, bytes, kMpolPreferred, &mask, 64, 0);
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

pcr_status make_pool_tmap(pcr_ctx* c) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(c, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(c, PCR_E_CUDA, "cuTensorMapEncodeTiled not found");
  const int64_t rows = int64_t(c->cfg.n_layers) * c->n_pool_pages * c->hkv * 2 * c->cfg.page_tokens;
  if (rows >= (int64_t(1) << 31)) return fail(c, PCR_E_INVAL, "pool too large for 32-bit TMA row coordinates");
  cuuint64_t dims[2] = {cuuint64_t(c->cfg.head_dim), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(c->cfg.head_dim) * 2};
  cuuint32_t box[2] = {64, cuuint32_t(pcr::attn_pool_box_rows(c->cfg.page_tokens))};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(
      &c->tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c->cfg.pool, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, PCR_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return PCR_OK;
}

Request* planned_request(pcr_ctx* c, int64_t id, pcr_status* st) {
  Request* r = c->planner->find(id);
  if (!r) { *st = fail(c, PCR_E_NOREQ, "unknown request"); return nullptr; }
  if (!r->planned) { *st = fail(c, PCR_E_STATE, "request not planned (call pcr_match_prefix first)"); return nullptr; }
  *st = PCR_OK;
  return r;
}

int32_t* d_pages_of(pcr_ctx* c, const Request* r) { return c->d_arena + r->plan.region * c->region_words; }
int32_t* d_slots_of(pcr_ctx* c, const Request* r) { return d_pages_of(c, r) + c->region_page_cap; }
// shard_mode 1 region tail: [own_slots | vpages | own_res_slots | own_res_pages]
int32_t* d_own_slots_of(pcr_ctx* c, const Request* r) { return d_slots_of(c, r) + c->chunk_cap; }
int32_t* d_vpages_of(pcr_ctx* c, const Request* r) { return d_own_slots_of(c, r) + c->chunk_cap; }
int32_t* d_own_res_slots_of(pcr_ctx* c, const Request* r) { return d_vpages_of(c, r) + c->region_page_cap; }
int32_t* d_own_res_pages_of(pcr_ctx* c, const Request* r) { return d_own_res_slots_of(c, r) + c->chunk_cap; }
bool stream_gather_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_STREAM_GATHER");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool late_dep_wait_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_LATE_DEP_WAIT");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool fused_append_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_FUSED_APPEND");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool owns_chunk(const pcr_ctx* c, int32_t depth) { return !c->ctx_split || depth % c->cfg.world == c->cfg.rank; }

// First device call of a request uploads its page/slot tables; later calls (on any stream)
// are ordered after that upload by an event.
pcr_status ensure_tables(pcr_ctx* c, Request* r, cudaStream_t s) {
  const int32_t reg = r->plan.region;
  if (!r->tables_uploaded) {
    int32_t* h = c->h_arena + reg * c->region_words;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_arena + reg * c->region_words, h, sizeof(int32_t) * c->region_words,
                                cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaEventRecord(c->region_ev[reg], s));
    r->tables_uploaded = true;
    c->device_active += 1;   // (a request with device work issued; until its release)
  } else {
    CUDA_TRY(c, cudaStreamWaitEvent(s, c->region_ev[reg], 0));
  }
  return PCR_OK;
}

pcr_status device_ready(pcr_ctx* c) {
  if (!c->device) return fail(c, PCR_E_STATE, "device call on a host-control-only context (device = -1)");
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  return PCR_OK;
}

// Copy-engine baselines of a2 (f4; the paper's copy path, fig:api).  Each matched chunk's
// layer-l image is C/S pool-page images in the page-major store slot; a page image maps to one pool
// page.  load_mode 1 merges adjacent images whose pool pages are also adjacent into one run (a chunk
// whose pages are consecutive is one Hkv*2*C*d*2-byte copy, 1 MiB for L8) and issues one
// cudaMemcpyAsync per run; load_mode 2 issues one cudaMemcpyAsync per page image (the paper's
// block-by-block baseline).
int64_t build_ce_runs(pcr_ctx* c, const Request* r, int32_t layer, int32_t ch0, int32_t ch1, bool merge) {
  const pcr_config& k = c->cfg;
  const int32_t ppc = k.chunk_tokens / k.page_tokens;
  const size_t page_img = static_cast<size_t>(c->hkv) * 2 * k.page_tokens * k.head_dim * 2;
  c->ce_dst.clear();
  c->ce_src.clear();
  c->ce_size.clear();
  uint8_t* pool = static_cast<uint8_t*>(k.pool);
  uint8_t* store = static_cast<uint8_t*>(c->store);
  for (int32_t ch = ch0; ch < ch1; ++ch)
    for (int32_t pp = 0; pp < ppc && owns_chunk(c, ch); ++pp) {
      uint8_t* src = store + r->plan.slots[ch] * c->slot_bytes + (int64_t(layer) * ppc + pp) * page_img;
      uint8_t* dst = pool + (int64_t(layer) * c->n_pool_pages + r->plan.pages[ch * ppc + pp]) * page_img;
      if (merge && !c->ce_src.empty() && static_cast<uint8_t*>(c->ce_src.back()) + c->ce_size.back() == src &&
          static_cast<uint8_t*>(c->ce_dst.back()) + c->ce_size.back() == dst) {
        c->ce_size.back() += page_img;
      } else {
        c->ce_src.push_back(src);
        c->ce_dst.push_back(dst);
        c->ce_size.push_back(page_img);
      }
    }
  return static_cast<int64_t>(c->ce_src.size());
}

pcr_status enqueue_ce_copy(pcr_ctx* c, Request* r, int32_t layer, cudaStream_t s, int32_t ch0, int32_t ch1,
                           bool merge) {
  const int64_t n = build_ce_runs(c, r, layer, ch0, ch1, merge);
  for (int64_t j = 0; j < n; ++j)
    CUDA_TRY(c, cudaMemcpyAsync(c->ce_dst[j], c->ce_src[j], c->ce_size[j], cudaMemcpyHostToDevice, s));
  c->ce_copies += n;
  return PCR_OK;
}

bool use_copy_engines(const pcr_ctx* c) { return c->cfg.load_mode == 1 || c->cfg.load_mode == 2; }

// Linear host->device copies that ride along with a layer's KV load (host_io: the layer's q/k/v
// inputs).  With device-mapped sources and the SM gather they are folded into the gather launch
// (one kernel per layer, one FIFO over the host link); otherwise one cudaMemcpyAsync each.
struct H2dCopies {
  int32_t n = 0;
  void* dst[3];
  const void* src[3];        // host pointers
  const void* src_dev[3];    // their device-mapped views (nullptr: not mapped)
  size_t bytes[3];
};

pcr_status enqueue_gather(pcr_ctx* c, Request* r, int32_t layer, cudaStream_t s, const H2dCopies* extra = nullptr) {
  pcr::LinearCopies lin{};
  const bool gather_kernel = !use_copy_engines(c) && c->cfg.load_mode != 3;
  if (extra && extra->n > 0) {
    bool fold = gather_kernel;
    for (int32_t i = 0; i < extra->n; ++i)
      fold = fold && extra->src_dev[i] && extra->bytes[i] % 16 == 0 &&
             (reinterpret_cast<uintptr_t>(extra->src_dev[i]) & 15) == 0 &&
             (reinterpret_cast<uintptr_t>(extra->dst[i]) & 15) == 0;
    if (fold) {
      lin.n = extra->n;
      for (int32_t i = 0; i < extra->n; ++i) {
        lin.src[i] = static_cast<const uint4*>(extra->src_dev[i]);
        lin.dst[i] = static_cast<uint4*>(extra->dst[i]);
        lin.n16[i] = static_cast<int64_t>(extra->bytes[i] / 16);
      }
    } else {
      for (int32_t i = 0; i < extra->n; ++i)
        CUDA_TRY(c, cudaMemcpyAsync(extra->dst[i], extra->src[i], extra->bytes[i], cudaMemcpyHostToDevice, s));
    }
  }
  if (r->plan.n_matched == 0 && lin.n == 0) return PCR_OK;
  if (use_copy_engines(c)) {
    c->ce_layer_loads += 1;
    return enqueue_ce_copy(c, r, layer, s, 0, r->plan.n_matched, c->cfg.load_mode == 1);
  }
  if (c->ctx_split) {   // this rank's chunks only (compacted tables)
    if (r->ctx_n_own == 0 && lin.n == 0) return PCR_OK;
    c->sm_layer_loads += r->ctx_n_own > 0;
    if (c->cfg.load_mode == 3)
      CUDA_TRY(c, pcr::launch_kv_gather_tma(c->store_dev, c->cfg.pool, d_own_slots_of(c, r), d_vpages_of(c, r),
                                            r->ctx_n_own, layer, c->geom, 4 * c->gather_ctas, s));
    else
      CUDA_TRY(c, pcr::launch_kv_gather(c->store_dev, c->cfg.pool, d_own_slots_of(c, r), d_vpages_of(c, r),
                                        r->ctx_n_own, layer, c->geom, c->gather_ctas, s, &lin));
    c->launches += 1;
    return PCR_OK;
  }
  if (c->cfg.load_mode == 3) {
    if (r->plan.n_matched == 0) return PCR_OK;
    CUDA_TRY(c, pcr::launch_kv_gather_tma(c->store_dev, c->cfg.pool, d_slots_of(c, r), d_pages_of(c, r),
                                          r->plan.n_matched, layer, c->geom, 4 * c->gather_ctas, s));
    c->launches += 1;
    c->sm_layer_loads += 1;
    return PCR_OK;
  }
  c->sm_layer_loads += r->plan.n_matched > 0;
  int32_t n_ce = 0;
  if (c->cfg.load_mode == 4 && r->plan.n_matched > 0) {
    // hybrid: chunks [0, n_ce) by the copy engines (one cudaMemcpyAsync per merged run) on
    // ce_stream, the rest by the gather kernel on s
    n_ce = std::min(r->plan.n_matched, std::max(0, static_cast<int32_t>(std::lround(
                                                       c->cfg.load_ce_fraction * r->plan.n_matched))));
    if (n_ce > 0) {
      if (!c->ce_stream) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->ce_stream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_ce_fork, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_ce_join, cudaEventDisableTiming));
      }
      CUDA_TRY(c, cudaEventRecord(c->ev_ce_fork, s));
      CUDA_TRY(c, cudaStreamWaitEvent(c->ce_stream, c->ev_ce_fork, 0));
      pcr_status st = enqueue_ce_copy(c, r, layer, c->ce_stream, 0, n_ce, true);
      if (st != PCR_OK) return st;
    }
  }
  if (n_ce < r->plan.n_matched || lin.n > 0) {
    const int32_t ppc = c->cfg.chunk_tokens / c->cfg.page_tokens;
    CUDA_TRY(c, pcr::launch_kv_gather(c->store_dev, c->cfg.pool, d_slots_of(c, r) + n_ce, d_pages_of(c, r) + n_ce * ppc,
                                      r->plan.n_matched - n_ce, layer, c->geom, c->gather_ctas, s, &lin));
    c->launches += 1;
  }
  if (n_ce > 0) {
    CUDA_TRY(c, cudaEventRecord(c->ev_ce_join, c->ce_stream));
    CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_ce_join, 0));
  }
  return PCR_OK;
}

pcr_status enqueue_attn(pcr_ctx* c, Request* r, int32_t layer, const void* q, const void* k, const void* v,
                        void* out, cudaStream_t s, float* part = nullptr) {
  // shard_mode 1: the virtual context of this rank = its own prefix chunks, then the suffix
  // (every rank appends the suffix: its reserved chunks are offloaded from there)
  const int64_t n1 = c->ctx_split ? int64_t(r->ctx_n_own) * c->cfg.chunk_tokens : r->plan.n1, n2 = r->plan.n2;
  const int32_t n_pages = c->ctx_split ? r->ctx_n_vpages : static_cast<int32_t>(r->plan.pages.size());
  const int32_t* pages = c->ctx_split ? d_vpages_of(c, r) : d_pages_of(c, r);
  // a3: fused into the attention (its last M-block's CTAs store the suffix K/V tiles they read into
  // the pool) -- except under the context split, where every rank appends the suffix (its reserved
  // chunks are offloaded from there) but only one attends to it, and with PCR_FUSED_APPEND=0
  const bool fused = !c->ctx_split && fused_append_enabled();
  if (!fused) {
    CUDA_TRY(c, pcr::launch_kv_append(k, v, c->cfg.pool, pages, n1, n2, n_pages, layer, c->geom, s));
    c->launches += 1;
  }
  pcr::AttnParams p{};
  p.ready = c->cur_ready;
  p.ready_target = c->cur_ready_target;
  if (fused) {
    p.k_new = static_cast<const uint16_t*>(k);
    p.v_new = static_cast<const uint16_t*>(v);
    p.late_dep_wait = late_dep_wait_enabled() ? 1 : 0;
  }
  p.q = static_cast<const uint16_t*>(q);
  p.out = static_cast<uint16_t*>(out);
  p.pages = pages;
  if (c->ctx_split) {
    const int64_t len = n1 + (r->ctx_suffix ? n2 : 0);
    p.kv_len = len > 0 ? static_cast<int32_t>(len) : -1;   // -1: no key here (O = 0, LSE = -inf)
    p.part_o = part;
    p.part_lse = part + n2 * c->hq * c->cfg.head_dim;
  }
  p.n1 = static_cast<int32_t>(n1);
  p.n2 = static_cast<int32_t>(n2);
  p.hq = c->hq;
  p.hkv = c->hkv;
  p.layer = layer;
  p.S = c->cfg.page_tokens;
  p.n_req_pages = n_pages;
  p.n_pool_pages = c->n_pool_pages;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(c->cfg.head_dim));
  // each plan region has its own split-KV workspace slice, so requests in flight on different
  // streams never share partials
  float* ws = c->ws ? c->ws + r->plan.region * c->ws_region_floats : nullptr;
  p.ws_o = ws;
  p.ws_lse = ws ? ws + c->ws_floats : nullptr;
  p.ws_bytes = c->ws_floats * 4;
  // The in-kernel split reduce waits for every split of a group, so it needs the whole grid resident:
  // only when no other request's device work can be running beside this one (its kernels could
  // hold the SMs a waiting group needs); otherwise the combine kernel merges the splits.
  p.spin_ctr = (ws && c->device_active <= 1) ? reinterpret_cast<uint32_t*>(ws + c->ws_floats + c->ws_floats / 64 + 64)
                                             : nullptr;
  int n = 0;
  cudaError_t e = pcr::launch_suffix_attn(&c->tmap, p, c->cfg.head_dim, s, &n);
  c->launches += n;
  if (e != cudaSuccess) return cuda_fail(c, e, "launch_suffix_attn");
  return PCR_OK;
}


pcr_status enqueue_offload(pcr_ctx* c, Request* r, int32_t layer, cudaStream_t s) {
  if (r->plan.n_reserved == 0) return PCR_OK;
  if (c->ctx_split) {
    if (r->ctx_n_res_own == 0) return PCR_OK;
    CUDA_TRY(c, pcr::launch_kv_scatter(c->cfg.pool, c->store_dev, d_own_res_slots_of(c, r), d_own_res_pages_of(c, r),
                                       0, r->ctx_n_res_own, layer, c->geom, c->gather_ctas, s));
    c->launches += 1;
    return PCR_OK;
  }
  CUDA_TRY(c, pcr::launch_kv_scatter(c->cfg.pool, c->store_dev, d_slots_of(c, r), d_pages_of(c, r),
                                     r->plan.n_matched, r->plan.n_reserved, layer, c->geom, c->gather_ctas, s));
  c->launches += 1;
  return PCR_OK;
}

// Page-locked host memory: true, with its device-mapped view in *dev (nullptr when the allocation
// is not mapped into the device address space).
bool pinned_host(const void* p, const void** dev) {
  cudaPointerAttributes a{};
  *dev = nullptr;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();   // clear the sticky-free error of an unknown pointer
    return false;
  }
  if (a.type != cudaMemoryTypeHost) return false;
  *dev = a.devicePointer;
  return true;
}

// host_io: the D2H stream, per-layer events and a ring of R staging buffers [q | k | v | out] of one
// layer each.  R = as many layers as fit kIoRingBytes (at least 2, at most L), so the inputs of
// layer l+R-1 can already be crossing the link while layer l computes.
constexpr int64_t kIoRingBytes = int64_t(512) << 20;

pcr_status ensure_host_io(pcr_ctx* c, int64_t layer_elems, int32_t want, int32_t* ring) {
  if (!c->io_d2h) {
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->io_d2h, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_io_join, cudaEventDisableTiming));
    for (int32_t l = 0; l < c->cfg.n_layers; ++l) {
      cudaEvent_t b;
      CUDA_TRY(c, cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      c->ev_outdone.push_back(b);
    }
  }
  const int64_t fit = want > 0 ? want : kIoRingBytes / std::max<int64_t>(1, 2 * layer_elems);
  const int64_t r = std::max<int64_t>(2, std::min<int64_t>(c->cfg.n_layers, fit));
  *ring = static_cast<int32_t>(r);
  if (r * layer_elems > c->io_buf_elems) {
    if (c->io_buf) {
      CUDA_TRY(c, cudaDeviceSynchronize());   // rare: the staging area grows to the largest N2 seen
      CUDA_TRY(c, cudaFree(c->io_buf));
      c->io_buf = nullptr;
    }
    CUDA_TRY(c, cudaMalloc(reinterpret_cast<void**>(&c->io_buf), r * layer_elems * sizeof(uint16_t)));
    c->io_buf_elems = r * layer_elems;
  }
  return PCR_OK;
}

pcr_status run_prefill_impl(pcr_ctx* c, int64_t req_id, const void* q_all, const void* k_all, const void* v_all,
                            void* out_all, const pcr_run_opts& o, int times_stride) {
  if (!c) return PCR_E_INVAL;
  pcr_status st = device_ready(c);
  if (st != PCR_OK) return st;
  Request* r = planned_request(c, req_id, &st);
  if (!r) return st;
  if (!q_all || !k_all || !v_all || (!out_all && !(c->ctx_split && !o.gathered_all)))
    return fail(c, PCR_E_INVAL, "null q/k/v/out");
  if (c->ctx_split && !o.gathered_all && !o.partial_all)
    return fail(c, PCR_E_INVAL, "shard_mode 1 needs partial_all (or gathered_all with pcr_run_prefill_sharded)");
  if (!c->ctx_split && o.partial_all) return fail(c, PCR_E_INVAL, "partial_all is for shard_mode 1");
  if (c->ctx_split && o.host_io) return fail(c, PCR_E_INVAL, "host_io is implemented for shard_mode 0 only");
  if (o.mode < 0 || o.mode > 3)
    return fail(c, PCR_E_INVAL, "mode must be 0 (OVERLAP), 1 (SYNC), 2 (ONLY_UP) or 3 (ONLY_DOWN)");
  // layer-wise loading (up) and offloading (down) overlapped or in order on the compute stream
  // (Only-Up, Only-Down, Up-Down)
  const bool up = o.mode == 0 || o.mode == 2, down = o.mode == 0 || o.mode == 3;
  if (!o.compute_stream) return fail(c, PCR_E_INVAL, "null compute stream");
  if (up && (!o.load_stream || o.load_stream == o.compute_stream))
    return fail(c, PCR_E_INVAL, "OVERLAP mode needs a load stream distinct from the compute stream");
  if (o.gathered_all && (!o.comm_stream || !c->nccl_comm))
    return fail(c, o.comm_stream ? PCR_E_STATE : PCR_E_INVAL, "all-gather needs pcr_comm_init and a comm stream");
  if (o.host_io != 0 && o.host_io != 1) return fail(c, PCR_E_INVAL, "host_io must be 0 or 1");
  if (o.host_io && o.gathered_all) return fail(c, PCR_E_INVAL, "host_io cannot be combined with gathered_all");
  const void *q_dev = nullptr, *k_dev = nullptr, *v_dev = nullptr, *o_dev = nullptr;
  if (o.host_io && !(pinned_host(q_all, &q_dev) && pinned_host(k_all, &k_dev) && pinned_host(v_all, &v_dev) &&
                     pinned_host(out_all, &o_dev)))
    return fail(c, PCR_E_INVAL, "host_io needs page-locked host q/k/v/out buffers");
  cudaStream_t cs = static_cast<cudaStream_t>(o.compute_stream);
  cudaStream_t ls = up ? static_cast<cudaStream_t>(o.load_stream) : cs;
  cudaStream_t os = o.offload_stream ? (down ? static_cast<cudaStream_t>(o.offload_stream) : cs) : nullptr;
  cudaStream_t xs = static_cast<cudaStream_t>(o.comm_stream);
  const int64_t n2 = r->plan.n2;
  const int64_t q_layer = n2 * c->hq * c->cfg.head_dim, kv_layer = n2 * c->hkv * c->cfg.head_dim;
  float* times = o.layer_times_ms;
  const pcr::NcclApi* api = o.gathered_all ? pcr::nccl_api() : nullptr;
  if (o.gathered_all && !api) return fail(c, PCR_E_UNSUPPORTED, "libnccl.so.2 not loadable");
  if ((st = ensure_tables(c, r, ls)) != PCR_OK) return st;
  if (up) CUDA_TRY(c, cudaStreamWaitEvent(cs, c->region_ev[r->plan.region], 0));
  // host_io: layer l's inputs/outputs go through staging buffer l % R (q | k | v | out).  In
  // OVERLAP mode the inputs are copied on the LOAD stream by layer l's gather launch itself (16-byte
  // loads from the mapped host buffers, like the KV) -- one FIFO of host->device traffic in the
  // order the layers need it, so the link never splits between streams (tools/bidir_probe.cu);
  // layer l+R's inputs wait for attention(l) to release the buffer.  Outputs return on the D2H
  // stream (the other direction of the link) with one cudaMemcpyAsync per layer.
  const int64_t io_layer = 2 * q_layer + 2 * kv_layer;
  int32_t ring = 2;
  cudaStream_t ds = cs;
  if (o.host_io) {
    if ((st = ensure_host_io(c, io_layer, o.io_ring_layers, &ring)) != PCR_OK) return st;
    if (up) {
      ds = c->io_d2h;
      CUDA_TRY(c, cudaEventRecord(c->ev_io_join, cs));    // staging may still be read by earlier work
      CUDA_TRY(c, cudaStreamWaitEvent(ls, c->ev_io_join, 0));
      CUDA_TRY(c, cudaStreamWaitEvent(ds, c->ev_io_join, 0));
    }
  }
  auto buf_of = [&](int32_t l) { return c->io_buf + (l % ring) * io_layer; };
  // shard_mode 1: per-layer partial block = O [N2*Hq][d] + LSE [N2*Hq] floats
  const int64_t part_block = n2 * c->hq * (c->cfg.head_dim + 1);
  if (c->ctx_split && !o.partial_all && part_block * c->cfg.n_layers > c->part_scratch_floats) {
    if (c->part_scratch) {
      CUDA_TRY(c, cudaDeviceSynchronize());   // rare: grows to the largest N2 seen
      CUDA_TRY(c, cudaFree(c->part_scratch));
      c->part_scratch = nullptr;
    }
    CUDA_TRY(c, cudaMalloc(reinterpret_cast<void**>(&c->part_scratch), part_block * c->cfg.n_layers * sizeof(float)));
    c->part_scratch_floats = part_block * c->cfg.n_layers;
  }
  auto stage = [&](int32_t l) -> pcr_status {   // SYNC mode: H2D of layer l's q/k/v into buffer l % R
    uint16_t* b = buf_of(l);
    CUDA_TRY(c, cudaMemcpyAsync(b, static_cast<const uint16_t*>(q_all) + l * q_layer, q_layer * 2,
                                cudaMemcpyHostToDevice, cs));
    CUDA_TRY(c, cudaMemcpyAsync(b + q_layer, static_cast<const uint16_t*>(k_all) + l * kv_layer, kv_layer * 2,
                                cudaMemcpyHostToDevice, cs));
    CUDA_TRY(c, cudaMemcpyAsync(b + q_layer + kv_layer, static_cast<const uint16_t*>(v_all) + l * kv_layer,
                                kv_layer * 2, cudaMemcpyHostToDevice, cs));
    return PCR_OK;
  };
  // Streamed gather (OVERLAP loads, SM gather, head sharding): ONE gather launch moves every layer
  // in order and publishes each layer through a per-layer counter that the attention of that layer
  // acquires in-kernel -- no per-layer launch, event or ramp-up on the load stream.  With host_io
  // the inputs ride along when the staging ring holds every layer (no buffer reuse to wait for).
  const int32_t L = c->cfg.n_layers;
  const bool host_io_mapped = o.host_io && q_dev && k_dev && v_dev && (q_layer * 2) % 16 == 0 && (kv_layer * 2) % 16 == 0;
  const bool streamed = up && !c->ctx_split && c->cfg.load_mode == 0 && stream_gather_enabled() &&
                        (r->plan.n_matched > 0 || o.host_io) && (!o.host_io || (host_io_mapped && ring >= L));
  struct ReadyReset {   // the counters belong to this call only (also on an early error return)
    pcr_ctx* c;
    ~ReadyReset() { c->cur_ready = nullptr; c->cur_ready_target = 0; }
  } ready_reset{c};
  if (streamed) {
    int32_t* ready = c->d_ready + int64_t(r->plan.region) * L;
    if (!c->gather_hi) {
      int lo = 0, hi = 0;
      CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CUDA_TRY(c, cudaStreamCreateWithPriority(&c->gather_hi, cudaStreamNonBlocking, hi));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_gather_fork, cudaEventDisableTiming));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_gather_join, cudaEventDisableTiming));
    }
    cudaStream_t gs = c->gather_hi;
    CUDA_TRY(c, cudaEventRecord(c->ev_gather_fork, ls));
    CUDA_TRY(c, cudaStreamWaitEvent(gs, c->ev_gather_fork, 0));
    CUDA_TRY(c, cudaMemsetAsync(ready, 0, sizeof(int32_t) * L, gs));
    CUDA_TRY(c, cudaEventRecord(c->ev_ready_zero, gs));
    CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_ready_zero, 0));   // (not the gather itself)
    pcr::LinearCopies lin{};
    if (o.host_io) {
      const void* srcs[3] = {q_dev, k_dev, v_dev};
      const int64_t off[3] = {0, q_layer, q_layer + kv_layer}, n[3] = {q_layer, kv_layer, kv_layer};
      lin.n = 3;
      for (int i = 0; i < 3; ++i) {
        lin.src[i] = static_cast<const uint4*>(srcs[i]);
        lin.dst[i] = reinterpret_cast<uint4*>(c->io_buf + off[i]);
        lin.n16[i] = n[i] * 2 / 16;
        lin.src_stride16[i] = n[i] * 2 / 16;
        lin.dst_stride16[i] = io_layer * 2 / 16;
      }
    }
    if (times) CUDA_TRY(c, cudaEventRecord(c->ev_t[0], gs));
    int32_t warps = 0;
    CUDA_TRY(c, pcr::launch_kv_gather_stream(c->store_dev, c->cfg.pool, d_slots_of(c, r), d_pages_of(c, r),
                                             r->plan.n_matched, c->geom, c->gather_ctas, &lin, ready, gs, &warps));
    if (times) CUDA_TRY(c, cudaEventRecord(c->ev_t[1], gs));
    CUDA_TRY(c, cudaEventRecord(c->ev_gather_join, gs));
    CUDA_TRY(c, cudaStreamWaitEvent(ls, c->ev_gather_join, 0));
    c->launches += 1;
    if (r->plan.n_matched > 0) c->sm_layer_loads += L;
    c->cur_ready = ready;
    c->cur_ready_target = warps;
  }
  for (int32_t l = 0; l < c->cfg.n_layers; ++l) {
    cudaEvent_t* et = &c->ev_t[6 * l];
    H2dCopies in;
    if (o.host_io && up && !streamed) {   // layer l's inputs join its KV load batch
      uint16_t* b = buf_of(l);
      if (l >= ring) CUDA_TRY(c, cudaStreamWaitEvent(ls, c->ev_attn[l - ring], 0));  // buffer free
      auto at = [](const void* base, int64_t elems) -> const void* {
        return base ? static_cast<const uint16_t*>(base) + elems : nullptr;
      };
      in.n = 3;
      in.dst[0] = b;
      in.src[0] = at(q_all, l * q_layer);
      in.src_dev[0] = at(q_dev, l * q_layer);
      in.bytes[0] = q_layer * 2;
      in.dst[1] = b + q_layer;
      in.src[1] = at(k_all, l * kv_layer);
      in.src_dev[1] = at(k_dev, l * kv_layer);
      in.bytes[1] = kv_layer * 2;
      in.dst[2] = b + q_layer + kv_layer;
      in.src[2] = at(v_all, l * kv_layer);
      in.src_dev[2] = at(v_dev, l * kv_layer);
      in.bytes[2] = kv_layer * 2;
    }
    if (!streamed) {
      if (times) CUDA_TRY(c, cudaEventRecord(et[0], ls));
      if ((st = enqueue_gather(c, r, l, ls, &in)) != PCR_OK) return st;
      if (times) CUDA_TRY(c, cudaEventRecord(et[1], ls));
      if (up) {
        CUDA_TRY(c, cudaEventRecord(c->ev_load[l], ls));
        CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_load[l], 0));
      }
    }
    const uint16_t *q_l = static_cast<const uint16_t*>(q_all) + l * q_layer,
                   *k_l = static_cast<const uint16_t*>(k_all) + l * kv_layer,
                   *v_l = static_cast<const uint16_t*>(v_all) + l * kv_layer;
    uint16_t* out_l = out_all ? static_cast<uint16_t*>(out_all) + l * q_layer : nullptr;
    if (o.host_io) {
      uint16_t* b = buf_of(l);
      if (!up && (st = stage(l)) != PCR_OK) return st;
      if (up) {   // (the inputs precede the load on ls, whose event cs already waits for)
        if (l >= ring) CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_outdone[l - ring], 0));  // out buffer drained
      }
      q_l = b;
      k_l = b + q_layer;
      v_l = b + q_layer + kv_layer;
      out_l = b + q_layer + 2 * kv_layer;
    }
    float* part_l = nullptr;   // shard_mode 1: this rank's partial of layer l
    if (c->ctx_split) part_l = (o.partial_all ? o.partial_all : c->part_scratch) + l * part_block;
    if (times) CUDA_TRY(c, cudaEventRecord(et[2], cs));
    st = enqueue_attn(c, r, l, q_l, k_l, v_l, out_l, cs, part_l);
    if (st != PCR_OK) return st;
    if (times) CUDA_TRY(c, cudaEventRecord(et[3], cs));
    if (os || o.gathered_all || o.host_io) CUDA_TRY(c, cudaEventRecord(c->ev_attn[l], cs));
    if (o.host_io) {
      // D2H of this layer's output while the next layers run; then stage layer l+2's inputs
      if (ds != cs) CUDA_TRY(c, cudaStreamWaitEvent(ds, c->ev_attn[l], 0));
      CUDA_TRY(c, cudaMemcpyAsync(static_cast<uint16_t*>(out_all) + l * q_layer, out_l, q_layer * 2,
                                  cudaMemcpyDeviceToHost, ds));
      if (up) CUDA_TRY(c, cudaEventRecord(c->ev_outdone[l], ds));
    }
    if (os) {
      // layer-wise offload of the new chunks right after this layer's KV exists
      if (os != cs) CUDA_TRY(c, cudaStreamWaitEvent(os, c->ev_attn[l], 0));
      if (times) CUDA_TRY(c, cudaEventRecord(et[4], os));
      if ((st = enqueue_offload(c, r, l, os)) != PCR_OK) return st;
      if (times) CUDA_TRY(c, cudaEventRecord(et[5], os));
    }
    if (o.gathered_all && c->ctx_split) {
      // context split: all-gather the ranks' partials of layer l, merge them into out_all[l]
      CUDA_TRY(c, cudaStreamWaitEvent(xs, c->ev_attn[l], 0));
      float* g = static_cast<float*>(o.gathered_all) + l * c->cfg.world * part_block;
      int rr = api->all_gather(part_l, g, static_cast<size_t>(part_block) * 4, /*ncclInt8*/ 0, c->nccl_comm, xs);
      if (rr != 0) return fail(c, PCR_E_CUDA, "ncclAllGather failed");
      const int64_t rows = n2 * c->hq;
      CUDA_TRY(c, pcr::launch_merge_partials(g, part_block, g + rows * c->cfg.head_dim, part_block, c->cfg.world, rows,
                                             c->cfg.head_dim, static_cast<uint16_t*>(out_all) + l * q_layer, xs));
      c->launches += 1;
    } else if (o.gathered_all) {
      // re-assemble this layer's head-sharded output on the comm stream while layer l+1 runs
      CUDA_TRY(c, cudaStreamWaitEvent(xs, c->ev_attn[l], 0));
      const size_t bytes = static_cast<size_t>(q_layer) * 2;
      int rr = api->all_gather(out_l, static_cast<uint8_t*>(o.gathered_all) + bytes * c->cfg.world * l, bytes,
                               /*ncclInt8*/ 0, c->nccl_comm, xs);
      if (rr != 0) return fail(c, PCR_E_CUDA, "ncclAllGather failed");
    }
  }
  if (o.prefill_done_event)
    CUDA_TRY(c, cudaEventRecord(static_cast<cudaEvent_t>(o.prefill_done_event), cs));
  if (up) {
    CUDA_TRY(c, cudaEventRecord(c->ev_join, ls));
    CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_join, 0));
  }
  if (os && os != cs) {
    CUDA_TRY(c, cudaEventRecord(c->ev_off, os));
    CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_off, 0));
  }
  if (o.gathered_all) {
    CUDA_TRY(c, cudaEventRecord(c->ev_comm, xs));
    CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_comm, 0));
  }
  if (o.host_io && up) {   // the last outputs have reached the host buffer
    CUDA_TRY(c, cudaEventRecord(c->ev_io_join, ds));
    CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_io_join, 0));
  }
  if (times) {
    CUDA_TRY(c, cudaStreamSynchronize(cs));
    float streamed_ms = 0.f;   // streamed gather: one launch for all layers, reported as its mean per layer
    if (streamed) CUDA_TRY(c, cudaEventElapsedTime(&streamed_ms, c->ev_t[0], c->ev_t[1]));
    for (int32_t l = 0; l < c->cfg.n_layers; ++l) {
      cudaEvent_t* et = &c->ev_t[6 * l];
      if (streamed) times[times_stride * l] = streamed_ms / L;
      else CUDA_TRY(c, cudaEventElapsedTime(&times[times_stride * l], et[0], et[1]));
      CUDA_TRY(c, cudaEventElapsedTime(&times[times_stride * l + 1], et[2], et[3]));
      if (times_stride > 2) {
        times[times_stride * l + 2] = 0.f;
        if (os) CUDA_TRY(c, cudaEventElapsedTime(&times[times_stride * l + 2], et[4], et[5]));
      }
    }
  }
  return PCR_OK;
}

}  // namespace

extern "C" {

int32_t pcr_abi_version(void) { return PCR_ABI_VERSION; }

const char* pcr_last_error(const pcr_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t pcr_pool_pages(const pcr_ctx* ctx) { return ctx ? ctx->n_pool_pages : -1; }
int64_t pcr_slot_bytes(const pcr_ctx* ctx) { return ctx ? ctx->slot_bytes : -1; }
int64_t pcr_kernel_launches(const pcr_ctx* ctx) { return ctx ? ctx->launches : -1; }

pcr_status pcr_merge_partials(pcr_ctx* c, const float* gathered, int32_t n_parts, int64_t n2, void* out,
                              void* stream) {
  if (!c) return PCR_E_INVAL;
  pcr_status st = device_ready(c);
  if (st != PCR_OK) return st;
  if (!gathered || !out || n_parts < 1 || n2 < 0) return fail(c, PCR_E_INVAL, "pcr_merge_partials: bad argument");
  const int64_t rows = n2 * c->hq, block = rows * (c->cfg.head_dim + 1);
  CUDA_TRY(c, pcr::launch_merge_partials(gathered, block, gathered + rows * c->cfg.head_dim, block, n_parts, rows,
                                         c->cfg.head_dim, static_cast<uint16_t*>(out), static_cast<cudaStream_t>(stream)));
  c->launches += 1;
  return PCR_OK;
}

pcr_status pcr_set_load_mode(pcr_ctx* c, int32_t load_mode, float load_ce_fraction) {
  if (!c) return PCR_E_INVAL;
  if (load_mode < 0 || load_mode > 4 || !(load_ce_fraction >= 0.f && load_ce_fraction <= 1.f))
    return fail(c, PCR_E_INVAL, "pcr_set_load_mode: load_mode in [0, 4], load_ce_fraction in [0, 1]");
  c->cfg.load_mode = load_mode;
  c->cfg.load_ce_fraction = load_ce_fraction;
  return PCR_OK;
}

pcr_status pcr_create(const pcr_config* cfg, pcr_ctx** out) {
  if (!cfg || !out) return PCR_E_INVAL;
  *out = nullptr;
  const pcr_config& k = *cfg;
  if (k.n_layers < 1 || k.n_q_heads < 1 || k.n_kv_heads < 1 || k.n_q_heads % k.n_kv_heads ||
      k.head_dim < 8 || k.head_dim % 8 || k.world < 1 || k.rank < 0 || k.rank >= k.world ||
      (k.shard_mode == 0 && k.n_kv_heads % k.world) || k.shard_mode < 0 || k.shard_mode > 1 ||
      k.chunk_tokens < 1 || k.page_tokens < 1 || k.chunk_tokens % k.page_tokens ||
      k.store_chunks < 1 || k.window < 0 || k.pool_bytes < 0 || k.max_inflight < 0 || k.max_tokens < 0 ||
      k.gather_ctas < 0 || k.load_mode < 0 || k.load_mode > 4 || k.ssd_chunks < 0 ||
      !(k.load_ce_fraction >= 0.f && k.load_ce_fraction <= 1.f) ||
      (k.ssd_chunks > 0 && !k.ssd_path))
    return PCR_E_INVAL;
  auto c = std::make_unique<pcr_ctx>();
  c->cfg = k;
  c->device = k.device >= 0;
  c->ctx_split = k.shard_mode == 1;
  c->hkv = c->ctx_split ? k.n_kv_heads : k.n_kv_heads / k.world;   // context split: all heads per rank
  c->hq = c->ctx_split ? k.n_q_heads : k.n_q_heads / k.world;
  c->G = c->hq / c->hkv;
  c->slot_elems = int64_t(k.n_layers) * c->hkv * 2 * k.chunk_tokens * k.head_dim;
  c->slot_bytes = c->slot_elems * 2;
  c->page_elems_all_layers = int64_t(k.n_layers) * c->hkv * 2 * k.page_tokens * k.head_dim;
  c->n_pool_pages = k.pool_bytes / (c->page_elems_all_layers * 2);
  if (c->device) {
    if (!(k.head_dim == 64 || k.head_dim == 128) ||
        !(k.page_tokens == 16 || k.page_tokens == 32 || k.page_tokens == 64 || k.page_tokens == 128) ||
        !is_pow2(k.chunk_tokens) || 128 % c->G != 0)
      return PCR_E_UNSUPPORTED;
    if (!k.pool || c->n_pool_pages < 1 || (reinterpret_cast<uintptr_t>(k.pool) & 255)) return PCR_E_INVAL;
  }
  const int64_t max_tokens = k.max_tokens > 0 ? k.max_tokens : std::max<int64_t>(1, c->n_pool_pages * k.page_tokens);
  c->max_regions = k.max_inflight > 0 ? k.max_inflight : 4;
  c->region_page_cap = (max_tokens + k.page_tokens - 1) / k.page_tokens;
  c->chunk_cap = (max_tokens + k.chunk_tokens - 1) / k.chunk_tokens;
  // [pages | slots], + context split: [own_slots | vpages | own_res_slots | own_res_pages]
  // (own_res_pages holds <= region_page_cap entries): 3 * (page_cap + chunk_cap) words in all
  c->region_words = (c->ctx_split ? 3 : 1) * (c->region_page_cap + c->chunk_cap);
  c->region_words = (c->region_words + 63) / 64 * 64;
  c->planner = std::make_unique<Planner>(k.chunk_tokens, k.page_tokens, k.store_chunks, c->n_pool_pages, k.window,
                                         c->max_regions, k.ssd_chunks);
  c->geom = pcr::KvGeom{k.n_layers, c->hkv, k.head_dim, k.chunk_tokens, k.page_tokens, c->n_pool_pages,
                        c->slot_elems};
  if (k.gather_ctas > 0) c->gather_ctas = k.gather_ctas;

  // DRAM store: anonymous mapping, NUMA-local to the GPU, pinned + mapped for zero-copy reads.
  c->store_bytes = static_cast<size_t>(k.store_chunks) * static_cast<size_t>(c->slot_bytes);
  void* p = mmap(nullptr, c->store_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  if (p == MAP_FAILED) return PCR_E_NOMEM;
  c->store = p;
  madvise(p, c->store_bytes, MADV_HUGEPAGE);
  c->h_arena = nullptr;
  if (k.ssd_chunks > 0) {
    c->ssd = std::make_unique<pcr::SsdIo>(k.ssd_path, k.ssd_chunks, c->slot_bytes);
    if (!c->ssd->ok()) {
      std::fprintf(stderr, "pcr_create: SSD tier: %s\n", c->ssd->error().c_str());
      pcr_destroy(c.release());
      return PCR_E_NOMEM;
    }
    c->slot_write_seq.assign(k.store_chunks, 0);
    c->slot_read_seq.assign(k.store_chunks, 0);
  }
  if (c->device) {
    pcr_ctx* cp = c.get();
    cudaError_t e = cudaSetDevice(k.device);
    if (e == cudaSuccess) bind_to_node(p, c->store_bytes, gpu_numa_node(k.device));
    if (e == cudaSuccess) e = cudaHostRegister(p, c->store_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e == cudaSuccess) { cp->registered = true; e = cudaHostGetDevicePointer(&cp->store_dev, p, 0); }
    if (e == cudaSuccess)
      e = cudaHostAlloc(reinterpret_cast<void**>(&cp->h_arena), sizeof(int32_t) * c->region_words * c->max_regions,
                        cudaHostAllocDefault);
    if (e == cudaSuccess)
      e = cudaMalloc(reinterpret_cast<void**>(&cp->d_arena), sizeof(int32_t) * c->region_words * c->max_regions);
    for (int i = 0; e == cudaSuccess && i < c->max_regions; ++i) {
      cudaEvent_t ev;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e == cudaSuccess) cp->region_ev.push_back(ev);
    }
    for (int l = 0; e == cudaSuccess && l < k.n_layers; ++l) {
      cudaEvent_t ev;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e == cudaSuccess) cp->ev_load.push_back(ev);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cp->ev_join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cp->ev_ready_zero, cudaEventDisableTiming);
    if (e == cudaSuccess)
      e = cudaMalloc(reinterpret_cast<void**>(&cp->d_ready), sizeof(int32_t) * k.n_layers * c->max_regions);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cp->ev_comm, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cp->ev_off, cudaEventDisableTiming);
    for (int l = 0; e == cudaSuccess && l < k.n_layers; ++l) {
      cudaEvent_t ev;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e == cudaSuccess) cp->ev_attn.push_back(ev);
    }
    if (e == cudaSuccess) {
      cp->ws_floats = (int64_t(32) << 20) / 4;  // 32 MiB of partial O (+ LSE) per region
      // + 512 words: the in-kernel split reduce's per-group arrival counts and generations
      cp->ws_region_floats = cp->ws_floats + cp->ws_floats / 64 + 64 + 512;
      e = cudaMalloc(reinterpret_cast<void**>(&cp->ws), cp->ws_region_floats * c->max_regions * 4);
      if (e == cudaSuccess) e = cudaMemset(cp->ws, 0, cp->ws_region_floats * c->max_regions * 4);
    }
    for (int l = 0; e == cudaSuccess && l < 6 * k.n_layers; ++l) {
      cudaEvent_t ev;
      e = cudaEventCreate(&ev);
      if (e == cudaSuccess) cp->ev_t.push_back(ev);
    }
    if (e != cudaSuccess) {
      std::fprintf(stderr, "pcr_create: %s\n", cudaGetErrorString(e));
      pcr_destroy(c.release());
      return PCR_E_CUDA;
    }
    if (make_pool_tmap(cp) != PCR_OK) {
      std::fprintf(stderr, "pcr_create: %s\n", cp->err.c_str());
      pcr_destroy(c.release());
      return PCR_E_CUDA;
    }
  } else {
    c->h_arena = static_cast<int32_t*>(std::calloc(c->region_words * c->max_regions, sizeof(int32_t)));
    if (!c->h_arena) { pcr_destroy(c.release()); return PCR_E_NOMEM; }
  }
  *out = c.release();
  return PCR_OK;
}

void pcr_destroy(pcr_ctx* c) {
  if (!c) return;
  if (c->device) {
    cudaSetDevice(c->cfg.device);
    cudaDeviceSynchronize();
    for (auto e : c->region_ev) cudaEventDestroy(e);
    for (auto e : c->ev_load) cudaEventDestroy(e);
    for (auto e : c->ev_t) cudaEventDestroy(e);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_ready_zero) cudaEventDestroy(c->ev_ready_zero);
    if (c->ev_gather_fork) cudaEventDestroy(c->ev_gather_fork);
    if (c->ev_gather_join) cudaEventDestroy(c->ev_gather_join);
    if (c->gather_hi) cudaStreamDestroy(c->gather_hi);
    if (c->d_ready) cudaFree(c->d_ready);
    if (c->ev_comm) cudaEventDestroy(c->ev_comm);
    if (c->ev_off) cudaEventDestroy(c->ev_off);
    for (auto e : c->ev_attn) cudaEventDestroy(e);
    for (auto e : c->ev_outdone) cudaEventDestroy(e);
    if (c->ev_io_join) cudaEventDestroy(c->ev_io_join);
    if (c->io_d2h) cudaStreamDestroy(c->io_d2h);
    if (c->part_scratch) cudaFree(c->part_scratch);
    if (c->io_buf) cudaFree(c->io_buf);
    if (c->ev_ce_fork) cudaEventDestroy(c->ev_ce_fork);
    if (c->ev_ce_join) cudaEventDestroy(c->ev_ce_join);
    if (c->ce_stream) cudaStreamDestroy(c->ce_stream);
    if (c->nccl_comm) {
      if (const pcr::NcclApi* api = pcr::nccl_api()) api->comm_destroy(c->nccl_comm);
    }
    if (c->d_arena) cudaFree(c->d_arena);
    if (c->ws) cudaFree(c->ws);
    if (c->h_arena) cudaFreeHost(c->h_arena);
    if (c->registered) cudaHostUnregister(c->store);
  } else {
    std::free(c->h_arena);
  }
  c->ssd.reset();  // drains queued I/O before the store goes away
  if (c->store) munmap(c->store, c->store_bytes);
  delete c;
}

pcr_status pcr_submit(pcr_ctx* c, int64_t req_id, const uint32_t* tokens, int64_t n_tokens, int64_t n_cacheable) {
  if (!c) return PCR_E_INVAL;
  std::string err;
  int32_t s = c->planner->submit(req_id, tokens, n_tokens, n_cacheable, &err);
  if (s != 0) return fail(c, static_cast<pcr_status>(s), err);
  return PCR_OK;
}

pcr_status pcr_match_prefix(pcr_ctx* c, int64_t req_id, const int64_t* pending, int32_t n_pending, pcr_plan* out) {
  if (!c || !out) return c ? fail(c, PCR_E_INVAL, "pcr_match_prefix: null plan") : PCR_E_INVAL;
  Request* r = c->planner->find(req_id);
  if (r && !r->planned) {
    const int64_t need_pages = (static_cast<int64_t>(r->tokens.size()) + c->cfg.page_tokens - 1) / c->cfg.page_tokens;
    if (need_pages > c->region_page_cap)
      return fail(c, PCR_E_NOMEM, "pcr_match_prefix: request longer than pcr_config.max_tokens");
  }
  if ((out->cap_slots > 0 && !out->slots) || (out->cap_pages > 0 && !out->pages) ||
      (out->cap_evicted > 0 && (!out->evicted_keys || !out->evicted_slots)))
    return fail(c, PCR_E_INVAL, "pcr_match_prefix: null output array with nonzero capacity");
  std::string err;
  int32_t s = c->planner->match_prefix(req_id, pending, n_pending, out->cap_slots, out->cap_pages,
                                       out->cap_evicted, &err);
  if (s != 0) return fail(c, static_cast<pcr_status>(s), err);
  const pcr::Plan& pl = r->plan;
  if (c->ssd) {
    // SSD -> DRAM loads (prefetch + on demand); reserved slots must not be overwritten while an
    // earlier write-back still reads them; the chain's own loads complete before returning.
    int64_t wait_seq = 0, last = 0;
    uint8_t* store = static_cast<uint8_t*>(c->store);
    for (const pcr::IoOp& op : pl.loads) {
      last = c->ssd->read(op.ssd_slot, store + static_cast<size_t>(op.dram_slot) * c->slot_bytes);
      c->slot_read_seq[op.dram_slot] = last;
      if (op.wait_now) wait_seq = last;
    }
    for (int32_t slot : pl.new_slots) wait_seq = std::max(wait_seq, c->slot_write_seq[slot]);
    // a matched chunk may still be LOADING from an earlier request's look-ahead prefetch: its read
    // must have landed before this request's gather reads the slot
    for (int32_t i = 0; i < pl.n_matched; ++i) wait_seq = std::max(wait_seq, c->slot_read_seq[pl.slots[i]]);
    if (last) c->req_load_seq[req_id] = last;
    if (wait_seq && !c->ssd->wait(wait_seq)) return fail(c, PCR_E_INTERNAL, "SSD I/O failed");
  }
  out->n_matched = pl.n_matched;
  out->n_reserved = pl.n_reserved;
  out->n1_tokens = pl.n1;
  out->n2_tokens = pl.n2;
  out->n_pages = static_cast<int32_t>(pl.pages.size());
  out->n_evicted = static_cast<int32_t>(pl.evicted.size());
  out->n_from_ssd = pl.n_from_ssd;
  std::copy(pl.slots.begin(), pl.slots.end(), out->slots);
  std::copy(pl.pages.begin(), pl.pages.end(), out->pages);
  for (size_t i = 0; i < pl.evicted.size(); ++i) {
    std::memcpy(out->evicted_keys + 16 * i, pl.evicted[i].first.data(), 16);
    out->evicted_slots[i] = pl.evicted[i].second;
  }
  // Stage the device tables (host memory only; uploaded by the first device call).
  int32_t* h = c->h_arena + pl.region * c->region_words;
  std::copy(pl.pages.begin(), pl.pages.end(), h);
  std::copy(pl.slots.begin(), pl.slots.end(), h + c->region_page_cap);
  if (c->ctx_split) {
    // [own_slots | vpages | own_res_slots | own_res_pages]: chunks at depth c % world == rank;
    // vpages = their pages, then the pages of the suffix tokens [n1, N)
    const int32_t ppc = c->cfg.chunk_tokens / c->cfg.page_tokens;
    int32_t* own_slots = h + c->region_page_cap + c->chunk_cap;
    int32_t* vpages = own_slots + c->chunk_cap;
    int32_t* res_slots = vpages + c->region_page_cap;
    int32_t* res_pages = res_slots + c->chunk_cap;
    int32_t n_own = 0, n_res = 0, nv = 0;
    for (int32_t ch = 0; ch < pl.n_matched; ++ch)
      if (owns_chunk(c, ch)) {
        own_slots[n_own++] = pl.slots[ch];
        for (int32_t pp = 0; pp < ppc; ++pp) vpages[nv++] = pl.pages[ch * ppc + pp];
      }
    for (size_t pg = static_cast<size_t>(pl.n_matched) * ppc; pg < pl.pages.size(); ++pg) vpages[nv++] = pl.pages[pg];
    for (int32_t ch = pl.n_matched; ch < pl.n_matched + pl.n_reserved; ++ch)
      if (owns_chunk(c, ch)) {
        for (int32_t pp = 0; pp < ppc; ++pp) res_pages[n_res * ppc + pp] = pl.pages[ch * ppc + pp];
        res_slots[n_res++] = pl.slots[ch];
      }
    r->ctx_n_own = n_own;
    r->ctx_n_res_own = n_res;
    r->ctx_n_vpages = nv;
    r->ctx_suffix = pl.n_matched % c->cfg.world == c->cfg.rank;
  }
  return PCR_OK;
}

pcr_status pcr_release(pcr_ctx* c, int64_t req_id, int32_t commit) {
  if (!c) return PCR_E_INVAL;
  if (c->ssd) {  // DrainCompletedSSDLoads (Alg.1): loads this request's match started
    auto it = c->req_load_seq.find(req_id);
    if (it != c->req_load_seq.end()) {
      if (c->planner->find(req_id) && !c->ssd->wait(it->second)) return fail(c, PCR_E_INTERNAL, "SSD I/O failed");
    }
  }
  std::string err;
  std::vector<pcr::IoOp> writes;
  const Request* rel = c->planner->find(req_id);
  const bool had_device_work = rel && rel->tables_uploaded;
  int32_t s = c->planner->release(req_id, commit != 0, &err, &writes);
  if (s == 0 && had_device_work) c->device_active -= 1;
  if (s != 0) return fail(c, static_cast<pcr_status>(s), err);
  c->req_load_seq.erase(req_id);
  uint8_t* store = static_cast<uint8_t*>(c->store);
  for (const pcr::IoOp& op : writes)  // asynchronous write-back
    c->slot_write_seq[op.dram_slot] = c->ssd->write(op.ssd_slot, store + static_cast<size_t>(op.dram_slot) * c->slot_bytes);
  return PCR_OK;
}

pcr_status pcr_get_stats(const pcr_ctx* c, pcr_stats* out) {
  if (!c || !out) return PCR_E_INVAL;
  const pcr::TierStats& t = c->planner->stats();
  out->prefetch_loads = t.prefetch;
  out->ondemand_loads = t.ondemand;
  out->writebacks = t.writeback;
  out->ssd_evictions = t.ssd_evict;
  out->dram_evictions = t.dram_evict;
  out->ssd_bytes_read = c->ssd ? c->ssd->bytes_read() : 0;
  out->ssd_bytes_written = c->ssd ? c->ssd->bytes_written() : 0;
  out->ce_copies = c->ce_copies;
  out->ce_layer_loads = c->ce_layer_loads;
  out->sm_layer_loads = c->sm_layer_loads;
  return PCR_OK;
}

// API slot layout [L][Hkv][2][C][d] <-> the store's page-major layout [L][C/S][Hkv][2][S][d].
void slot_permute(const pcr_ctx* c, uint8_t* dst, const uint8_t* src, bool to_store) {
  const pcr_config& k = c->cfg;
  const int32_t ppc = k.chunk_tokens / k.page_tokens;
  const size_t seg = static_cast<size_t>(k.page_tokens) * k.head_dim * 2;
  for (int32_t l = 0; l < k.n_layers; ++l)
    for (int32_t h = 0; h < c->hkv; ++h)
      for (int32_t kv = 0; kv < 2; ++kv)
        for (int32_t pp = 0; pp < ppc; ++pp) {
          const size_t api = ((static_cast<size_t>(l) * c->hkv + h) * 2 + kv) * ppc + pp;
          const size_t sto = ((static_cast<size_t>(l) * ppc + pp) * c->hkv + h) * 2 + kv;
          if (to_store) std::memcpy(dst + sto * seg, src + api * seg, seg);
          else std::memcpy(dst + api * seg, src + sto * seg, seg);
        }
}

pcr_status pcr_store_write(pcr_ctx* c, int32_t slot, const void* src) {
  if (!c || !src) return c ? fail(c, PCR_E_INVAL, "pcr_store_write: null source") : PCR_E_INVAL;
  if (slot < 0 || slot >= c->cfg.store_chunks) return fail(c, PCR_E_INVAL, "pcr_store_write: slot out of range");
  slot_permute(c, static_cast<uint8_t*>(c->store) + static_cast<size_t>(slot) * c->slot_bytes,
               static_cast<const uint8_t*>(src), true);
  return PCR_OK;
}

pcr_status pcr_store_read(const pcr_ctx* c, int32_t slot, void* dst) {
  if (!c || !dst) return c ? fail(c, PCR_E_INVAL, "pcr_store_read: null destination") : PCR_E_INVAL;
  if (slot < 0 || slot >= c->cfg.store_chunks) return fail(c, PCR_E_INVAL, "pcr_store_read: slot out of range");
  slot_permute(c, static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(c->store) + static_cast<size_t>(slot) * c->slot_bytes,
               false);
  return PCR_OK;
}

pcr_status pcr_leaf_list(const pcr_ctx* c, uint8_t* keys, int32_t cap, int32_t* n_out) {
  if (!c || !n_out || (cap > 0 && !keys)) return PCR_E_INVAL;
  auto leaves = c->planner->leaf_list();
  *n_out = static_cast<int32_t>(leaves.size());
  if (static_cast<int64_t>(leaves.size()) > cap) return fail(c, PCR_E_INVAL, "pcr_leaf_list: capacity too small");
  for (size_t i = 0; i < leaves.size(); ++i) std::memcpy(keys + 16 * i, leaves[i].data(), 16);
  return PCR_OK;
}

pcr_status pcr_blake2b(const void* data, int64_t n, const void* key, int32_t keylen, int32_t digest_len,
                       uint8_t* out) {
  if ((n > 0 && !data) || !out || n < 0 || keylen < 0 || (keylen > 0 && !key)) return PCR_E_INVAL;
  return pcr::blake2b(out, static_cast<size_t>(digest_len), key, static_cast<size_t>(keylen), data,
                      static_cast<size_t>(n))
             ? PCR_OK
             : PCR_E_INVAL;
}

pcr_status pcr_load_layer_kv(pcr_ctx* c, int64_t req_id, int32_t layer, void* load_stream) {
  if (!c) return PCR_E_INVAL;
  pcr_status st = device_ready(c);
  if (st != PCR_OK) return st;
  Request* r = planned_request(c, req_id, &st);
  if (!r) return st;
  if (layer < 0 || layer >= c->cfg.n_layers) return fail(c, PCR_E_INVAL, "layer out of range");
  cudaStream_t s = static_cast<cudaStream_t>(load_stream);
  if ((st = ensure_tables(c, r, s)) != PCR_OK) return st;
  return enqueue_gather(c, r, layer, s);
}

pcr_status pcr_prefill_attn_layer(pcr_ctx* c, int64_t req_id, int32_t layer, const void* q, const void* k_new,
                                  const void* v_new, void* out, void* compute_stream) {
  if (!c) return PCR_E_INVAL;
  pcr_status st = device_ready(c);
  if (st != PCR_OK) return st;
  Request* r = planned_request(c, req_id, &st);
  if (!r) return st;
  if (layer < 0 || layer >= c->cfg.n_layers) return fail(c, PCR_E_INVAL, "layer out of range");
  if (!q || !k_new || !v_new || !out) return fail(c, PCR_E_INVAL, "null q/k/v/out");
  if (c->ctx_split)   // a rank's attention is a partial there: pcr_run_prefill_ex(partial_all)
    return fail(c, PCR_E_INVAL, "pcr_prefill_attn_layer: shard_mode 1 returns partials (pcr_run_prefill_ex)");
  cudaStream_t s = static_cast<cudaStream_t>(compute_stream);
  if ((st = ensure_tables(c, r, s)) != PCR_OK) return st;
  return enqueue_attn(c, r, layer, q, k_new, v_new, out, s);
}

pcr_status pcr_run_prefill(pcr_ctx* c, int64_t req_id, const void* q_all, const void* k_all, const void* v_all,
                           void* out_all, void* compute_stream, void* load_stream, int32_t mode,
                           float* layer_times_ms) {
  pcr_run_opts o{};
  o.compute_stream = compute_stream;
  o.load_stream = load_stream;
  o.mode = mode;
  o.layer_times_ms = layer_times_ms;
  return run_prefill_impl(c, req_id, q_all, k_all, v_all, out_all, o, 2);
}

pcr_status pcr_run_prefill_sharded(pcr_ctx* c, int64_t req_id, const void* q_all, const void* k_all,
                                   const void* v_all, void* out_all, void* gathered_all, void* compute_stream,
                                   void* load_stream, void* comm_stream, int32_t mode, float* layer_times_ms) {
  if (!c) return PCR_E_INVAL;
  if (!c->nccl_comm) return fail(c, PCR_E_STATE, "pcr_run_prefill_sharded: call pcr_comm_init first");
  if (!gathered_all || !comm_stream) return fail(c, PCR_E_INVAL, "null gathered_all or comm_stream");
  pcr_run_opts o{};
  o.compute_stream = compute_stream;
  o.load_stream = load_stream;
  o.comm_stream = comm_stream;
  o.gathered_all = gathered_all;
  o.mode = mode;
  o.layer_times_ms = layer_times_ms;
  return run_prefill_impl(c, req_id, q_all, k_all, v_all, out_all, o, 2);
}

pcr_status pcr_run_prefill_ex(pcr_ctx* c, int64_t req_id, const void* q_all, const void* k_all, const void* v_all,
                              void* out_all, const pcr_run_opts* opts) {
  if (!c || !opts) return c ? fail(c, PCR_E_INVAL, "null options") : PCR_E_INVAL;
  return run_prefill_impl(c, req_id, q_all, k_all, v_all, out_all, *opts, 3);
}

pcr_status pcr_offload_layer_kv(pcr_ctx* c, int64_t req_id, int32_t layer, void* offload_stream) {
  if (!c) return PCR_E_INVAL;
  pcr_status st = device_ready(c);
  if (st != PCR_OK) return st;
  Request* r = planned_request(c, req_id, &st);
  if (!r) return st;
  if (layer < 0 || layer >= c->cfg.n_layers) return fail(c, PCR_E_INVAL, "layer out of range");
  cudaStream_t s = static_cast<cudaStream_t>(offload_stream);
  if ((st = ensure_tables(c, r, s)) != PCR_OK) return st;
  return enqueue_offload(c, r, layer, s);
}

pcr_status pcr_comm_unique_id(uint8_t* out) {
  if (!out) return PCR_E_INVAL;
  const pcr::NcclApi* api = pcr::nccl_api();
  if (!api) return PCR_E_UNSUPPORTED;
  pcr::NcclApi::UniqueId id;
  if (api->get_unique_id(&id) != 0) return PCR_E_CUDA;
  std::memcpy(out, id.internal, 128);
  return PCR_OK;
}

pcr_status pcr_comm_init(pcr_ctx* c, const uint8_t* id) {
  if (!c || !id) return c ? fail(c, PCR_E_INVAL, "pcr_comm_init: null id") : PCR_E_INVAL;
  pcr_status st = device_ready(c);
  if (st != PCR_OK) return st;
  if (c->nccl_comm) return fail(c, PCR_E_STATE, "pcr_comm_init: communicator already attached");
  const pcr::NcclApi* api = pcr::nccl_api();
  if (!api) return fail(c, PCR_E_UNSUPPORTED, "pcr_comm_init: libnccl.so.2 not loadable");
  pcr::NcclApi::UniqueId uid;
  std::memcpy(uid.internal, id, 128);
  void* comm = nullptr;
  int r = api->comm_init_rank(&comm, c->cfg.world, uid, c->cfg.rank);
  if (r != 0)
    return fail(c, PCR_E_CUDA, std::string("ncclCommInitRank: ") + (api->get_error_string ? api->get_error_string(r) : "error"));
  c->nccl_comm = comm;
  return PCR_OK;
}

}  // extern "C"
