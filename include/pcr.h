/*
 * pcr.h — C-ABI of libpcr.so, the B200-native reuse-prefill hot path of PCR
 * (arXiv 2603.23049, "prefetch-enhanced KV-cache reuse for RAG serving").
 *
 * Cites: P:<n> = /root/reference/PAPER.md line n; S:<n> = SPEC.md line n.
 *
 * The problem statement the calls follow (Alg. 1): the executor
 * "interacts with the Cache Engine to identify reusable prefixes" (pcr_match_prefix),
 * loads the matched KV from CPU memory layer by layer (pcr_load_layer_kv), computes
 * the remaining tokens (pcr_prefill_attn_layer), overlapping load(l+1) with compute(l)
 * on separate CUDA streams (pcr_run_prefill), and commits or drops
 * the new chunks at the end of the step (pcr_release).
 *
 * Conventions
 *  - C99; no C++/CUDA/torch types cross the ABI. Streams are cudaStream_t passed as void*.
 *  - Every call returns pcr_status; the message of the last failure is pcr_last_error().
 *    No exception or abort crosses the ABI.
 *  - Host-control calls (pcr_submit, pcr_match_prefix, pcr_release) make NO CUDA calls
 *    and give the strong guarantee: on error nothing changed.
 *  - Device calls only ENQUEUE work on the given streams and never synchronise (except
 *    pcr_run_prefill with a non-NULL layer_times_ms, see there). Launch errors return
 *    PCR_E_CUDA; asynchronous faults surface at the caller's stream synchronisation.
 *  - A ctx is not thread-safe: one owner thread.
 *  - Ownership: the library owns the pinned host store, the prefix tree and the per-
 *    request plan (including its device-side page/slot tables). The caller owns the
 *    HBM pool, all Q/K/V/out buffers and the streams; the library borrows raw pointers.
 *  - Lifecycle per request: pcr_submit -> (may appear in other requests' pending ids)
 *    -> pcr_match_prefix -> device calls -> [caller synchronises] -> pcr_release.
 *    Calls out of order return PCR_E_STATE; unknown ids PCR_E_NOREQ.
 *    pcr_release frees the request's pool pages and table region for reuse, so the
 *    caller must make sure the request's device work has completed before releasing.
 *
 * Data layouts (all bf16, row-major, innermost last; "loc" = this rank's slice):
 *   store slot (one chunk, all layers)  [L][Hkv_loc][2][C][d]       2 = {K, V}
 *   HBM pool                            [L][n_pages][Hkv_loc][2][S_pg][d]
 *     token t of a request lives in pool page pages[t / S_pg], row t % S_pg.
 *   q    (one layer)                    [N2][Hq_loc][d]
 *   k_new, v_new (one layer)            [N2][Hkv_loc][d]   (post-RoPE)
 *   out  (one layer)                    [N2][Hq_loc][d]
 *   *_all (pcr_run_prefill)             [L][...] of the per-layer layouts above
 * Query head h (local index) uses KV head h / G, G = Hq / Hkv (GQA, HF repeat_kv).
 * Rank r of `world` owns KV heads [r*Hkv/world, (r+1)*Hkv/world) and the matching Q heads.
 */
#ifndef PCR_H_
#define PCR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCR_ABI_VERSION 7

typedef struct pcr_ctx pcr_ctx;

typedef enum pcr_status {
  PCR_OK = 0,
  PCR_E_INVAL = -1,      /* bad argument (null pointer, out-of-range id/layer, short capacity) */
  PCR_E_NOMEM = -2,      /* pool pages, plan regions or host memory exhausted */
  PCR_E_CUDA = -3,       /* a CUDA runtime call or kernel launch failed */
  PCR_E_STATE = -4,      /* call out of lifecycle order, or device call on a host-only ctx */
  PCR_E_NOREQ = -5,      /* unknown request id */
  PCR_E_INTERNAL = -6,   /* invariant violated (S:145 InconsistentDrop); a bug */
  PCR_E_UNSUPPORTED = -7 /* shape the kernels do not implement (see pcr_create) */
} pcr_status;

/* Model geometry and cache configuration.  Every rank passes the same struct except
 * `rank`, `device` and `pool`; host decisions are deterministic, so every rank computes
 * identical slots, pages and evictions without any control traffic. */
typedef struct pcr_config {
  int32_t n_layers;      /* L */
  int32_t n_q_heads;     /* Hq (full model); Hq % Hkv == 0 */
  int32_t n_kv_heads;    /* Hkv (full model); world divides Hkv */
  int32_t head_dim;      /* d; the device path implements d in {64, 128} */
  int32_t rank, world;   /* KV-head sharding */
  int32_t chunk_tokens;  /* C: tree/store granularity (paper 256) */
  int32_t page_tokens;   /* S_pg: pool page tokens (paper's vLLM block 16);
                            S_pg in {16, 32, 64, 128} and S_pg divides C */
  int64_t store_chunks;  /* DRAM store capacity in chunks (reading R13: capacity unit) */
  int32_t window;        /* look-ahead window W (paper 4; best 6) */
  int32_t device;        /* CUDA ordinal; -1 = host-control only (no CUDA calls at all;
                            the store is ordinary memory; device calls return PCR_E_STATE) */
  void* pool;            /* caller-owned HBM pool (device pointer, 256-byte aligned) */
  int64_t pool_bytes;    /* n_pages = pool_bytes / (L*Hkv_loc*2*S_pg*d*2) */
  int32_t max_inflight;  /* requests planned but not yet released; 0 -> 4 */
  int32_t max_tokens;    /* max tokens of one request; 0 -> pool capacity in tokens */
  int32_t gather_ctas;   /* CTAs of the host->HBM gather kernel; 0 -> library default */
  int32_t load_mode;     /* a2 implementation: 0 = sm_100a 16-byte gather kernel (default; the
                            north_star mover: coalesced 16-byte loads from the mapped host store).
                            f4 baselines of the paper's copy path (fig:api), no SMs used:
                            1 = copy engines, one cudaMemcpyAsync per run (adjacent page images of
                            a chunk whose pool pages are also adjacent merge into one run);
                            2 = copy engines, one cudaMemcpyAsync per page image (block by block);
                            3 = experiment: TMA bulk copies host -> smem -> pool page;
                            4 = hybrid: the copy engines (one cudaMemcpyAsync per run, on a library
                            stream) move the first load_ce_fraction of the matched chunks while
                            the gather kernel moves the rest, both over the same host link.
                            The f1 offload always uses the SM scatter kernel. */
  float load_ce_fraction;  /* load_mode 4 only: share of the chunks for the copy engines, [0, 1] */
  /* SSD tier (§8 f2): a file of ssd_chunks chunk records behind the DRAM store.
   * Committed chunks are written back asynchronously; chunks of requests in the
   * look-ahead window that are only on the SSD are prefetched into DRAM by an I/O thread
   * (P:456); a scheduled request's SSD-only chunks are loaded on demand.  NULL / 0 = no SSD.
   * The library creates (truncates) the file at pcr_create and removes it at pcr_destroy: the
   * records are meaningless without the context's in-memory index. */
  const char* ssd_path;
  int64_t ssd_chunks;
  /* How `world` ranks share a request.  0 = KV-head sharding: rank r owns KV
   * heads [r*Hkv/world, (r+1)*Hkv/world) and their query heads, of every chunk.
   * 1 = context split (the §8(e) variant for world > Hkv, or to spread the prefix load): every
   * rank holds all heads; a chunk at chain depth c belongs to rank c % world (its store holds
   * and loads only those; the planner stays replicated, so the store is still sized
   * store_chunks slots per rank), and the suffix keys to rank (n_matched % world).  Each rank
   * attends all suffix rows to its own keys and returns a partial (O normalised by its own row
   * sum, log2-domain LSE: pcr_run_opts.partial_all); the partials of all ranks merge into the
   * output (pcr_merge_partials, or the per-layer NCCL all-gather + merge of
   * pcr_run_prefill_sharded).  Every rank receives all heads' q/k_new/v_new. */
  int32_t shard_mode;
} pcr_config;

/* Create a context.  Allocates the pinned store (mmap + NUMA-local mbind to the GPU's
 * node + cudaHostRegister, mapped), the device plan arena, events and TMA descriptors
 * over `pool`.  PCR_E_INVAL: inconsistent geometry; PCR_E_UNSUPPORTED: head_dim or
 * page_tokens outside what the kernels implement; PCR_E_NOMEM / PCR_E_CUDA: allocation. */
pcr_status pcr_create(const pcr_config* cfg, pcr_ctx** out);
void pcr_destroy(pcr_ctx* ctx);                 /* NULL is a no-op */
const char* pcr_last_error(const pcr_ctx* ctx); /* never NULL; "" if no error */
int32_t pcr_abi_version(void);

/* Derived geometry: pool pages, bytes of one store slot, bytes of one pool page (all layers). */
int64_t pcr_pool_pages(const pcr_ctx* ctx);
int64_t pcr_slot_bytes(const pcr_ctx* ctx);

/* ---------------------------------------------------------------- host control ------ */

/* Register a request (it may now appear in pending windows).  tokens[n_tokens] are copied;
 * chunks are hashed once here (Alg.1 Chunkify/HashPrefix):
 *   key_i = BLAKE2b-128(key_{i-1} || tokens_i as little-endian uint32), key_{-1} = 0^16,
 * for the min(n_cacheable / C, (n_tokens-1) / C) cacheable chunks (reading R5: at least
 * one token is always recomputed).  PCR_E_INVAL: n_tokens < 1 or n_cacheable outside
 * [0, n_tokens] or null tokens; PCR_E_STATE: id already registered. */
pcr_status pcr_submit(pcr_ctx* ctx, int64_t req_id, const uint32_t* tokens, int64_t n_tokens,
                      int64_t n_cacheable);

/* The movement plan of one request (Alg.1: cpu_to_gpu = the n_matched chunks,
 * gpu_to_cpu = the n_reserved new chunks; AdjustTokens = n1/n2).  Caller-owned arrays
 * with capacities; if a capacity is short the call fails with PCR_E_INVAL and nothing
 * changes.  Arrays may be NULL when their capacity is 0 and no entries are produced. */
typedef struct pcr_plan {
  int32_t n_matched;     /* chunks reused from the DRAM store (pinned until release) */
  int32_t n_reserved;    /* new chunks given a store slot (PENDING until release/commit) */
  int64_t n1_tokens;     /* n_matched * C */
  int64_t n2_tokens;     /* n_tokens - n1_tokens (>= 1) */
  int32_t* slots;        /* [n_matched + n_reserved] store slots in chain order */
  int32_t cap_slots;
  int32_t* pages;        /* [ceil(n_tokens / S_pg)] pool pages, logical order */
  int32_t cap_pages;
  int32_t n_pages;
  int32_t n_evicted;
  uint8_t* evicted_keys; /* [n_evicted][16] keys evicted to make room, in eviction order */
  int32_t* evicted_slots;/* [n_evicted] their freed slots */
  int32_t cap_evicted;
  int32_t n_from_ssd;    /* chunks of this chain loaded from the SSD on demand (ssd_to_gpu) */
} pcr_plan;

/* Plan one request (§4.2; Alg.1), in this order:
 *  1. look-ahead bump: for each id in Reverse(pending_ids[0 : min(n_pending, window)]),
 *     walk its chunk chain root-first, touching (moving to MRU) every RESIDENT chunk
 *     that is a leaf; stop at the first chunk that is not RESIDENT;
 *  2. match: walk this request's chain while the chunk is RESIDENT (key, parent and
 *     tokens equal); touch and pin each matched chunk ("until a mismatch occurs");
 *  3. reserve: for each remaining cacheable chunk: the lowest free slot, else evict the
 *     first unpinned RESIDENT leaf in LRU order (its parent becomes a leaf at MRU when
 *     this was its last child); insert a PENDING pinned node at MRU (its parent
 *     leaves the leaf list).  Stop at the first chunk that cannot get a slot (all leaves
 *     pinned: SPEC's EvictionStarved is not an error) or whose key exists;
 *  4. pool pages: ceil(n_tokens / S_pg), lowest free first.
 * Ids beyond the window are ignored.  PCR_E_NOREQ: unknown req_id or pending id;
 * PCR_E_STATE: already planned; PCR_E_INVAL: pending ids contain req_id or duplicates,
 * or a short capacity (slots and evicted need >= the request's cacheable chunk count, pages
 * >= ceil(n_tokens / S_pg)); PCR_E_NOMEM: not enough free pages or plan regions, or the
 * request is longer than pcr_config.max_tokens. */
pcr_status pcr_match_prefix(pcr_ctx* ctx, int64_t req_id, const int64_t* pending_ids,
                            int32_t n_pending, pcr_plan* out);

/* End of the step (Alg.1).  commit != 0: reserved chunks become RESIDENT
 * (their slot data must have been written: by offload, or by pcr_store_write) and, with an
 * SSD tier, are queued for asynchronous write-back to the SSD;
 * commit == 0: reserved chunks are dropped deepest-first.  All pins are released and the
 * pool pages returned.  SSD loads started by this request's match are drained first
 * (DrainCompletedSSDLoads, Alg.1).  The request id is then forgotten. */
pcr_status pcr_release(pcr_ctx* ctx, int64_t req_id, int32_t commit);

/* Copy one chunk record ([L][Hkv_loc][2][C][d] bf16, pcr_slot_bytes bytes) into / out of
 * the pinned DRAM store.  Host memcpy; PCR_E_INVAL on a bad slot or null pointer.  The store
 * keeps slots page-major internally ([L][C/S_pg][Hkv_loc][2][S_pg][d]: the images of the pool
 * pages the chunk fills) and converts here, so the record layout callers see is unchanged. */
pcr_status pcr_store_write(pcr_ctx* ctx, int32_t slot, const void* src);
pcr_status pcr_store_read(const pcr_ctx* ctx, int32_t slot, void* dst);

/* Cache-engine counters since creation (SSD tier and evictions). */
typedef struct pcr_stats {
  int64_t prefetch_loads;   /* SSD->DRAM loads submitted by the look-ahead prefetch phase */
  int64_t ondemand_loads;   /* SSD->DRAM loads of a scheduled request's own chain */
  int64_t writebacks;       /* DRAM->SSD write-backs of committed chunks */
  int64_t ssd_evictions;    /* SSD records overwritten (LRU) */
  int64_t dram_evictions;   /* DRAM leaves evicted */
  int64_t ssd_bytes_read, ssd_bytes_written;
  int64_t ce_copies;        /* copy-engine copies (cudaMemcpyAsync) enqueued for a2 loads (load_mode 1/2/4) */
  int64_t ce_layer_loads;   /* layer loads done by the copy engines alone (load_mode 1/2) */
  int64_t sm_layer_loads;   /* layer loads with a kernel moving prefix KV (load_mode 0/3/4) */
} pcr_stats;
pcr_status pcr_get_stats(const pcr_ctx* ctx, pcr_stats* out);

/* Inspection for tests: the leaf list in LRU->MRU order as 16-byte keys. */
pcr_status pcr_leaf_list(const pcr_ctx* ctx, uint8_t* keys, int32_t cap, int32_t* n_out);
/* RFC 7693 BLAKE2b (unkeyed when keylen == 0), digest_len in [1, 64]; used by tests to pin
 * the library's hash against the RFC vectors. */
pcr_status pcr_blake2b(const void* data, int64_t n, const void* key, int32_t keylen,
                       int32_t digest_len, uint8_t* out);

/* ---------------------------------------------------------------- device path ------- */

/* a2 — enqueue on load_stream the copy of layer `layer` of every matched chunk from the
 * pinned host store into the request's pool pages:
 *   pool[layer][pages[t/S_pg]][h][kv][t%S_pg][:] = store[slots[t/C]][layer][h][kv][t%C][:]
 * for t < n1.  An sm_100a kernel reads the mapped host memory over PCIe with 16-byte
 * loads and writes 16-byte stores into the pool pages, or (load_mode 1/2) the copy engines.
 * The first device call of a request also uploads its page/slot tables on its stream. */
pcr_status pcr_load_layer_kv(pcr_ctx* ctx, int64_t req_id, int32_t layer, void* load_stream);

/* a3 + a4 — enqueue on compute_stream: append k_new/v_new ([N2][Hkv_loc][d]) at tokens
 * n1..n1+N2-1 of the pool, then suffix-query causal attention:
 *   out[i][h] = softmax_j( q[i][h] . K[j][h/G] / sqrt(d) ) V[j][h/G],  j <= n1 + i,
 * bf16 inputs, fp32 accumulation (tcgen05/TMEM), bf16 output.  The caller orders this
 * after pcr_load_layer_kv(layer) (pcr_run_prefill does so with events).  PCR_E_INVAL under
 * shard_mode 1 (a rank's result there is a partial: pcr_run_prefill_ex with partial_all). */
pcr_status pcr_prefill_attn_layer(pcr_ctx* ctx, int64_t req_id, int32_t layer, const void* q,
                                  const void* k_new, const void* v_new, void* out,
                                  void* compute_stream);

/* a5 — the whole layer pipeline for one planned request (Alg.1):
 *   mode 0 OVERLAP: load_stream: ONE streamed gather launch moves every layer in order and
 *                   publishes layer l through a per-layer completion counter (release); the
 *                   launch runs on a library-owned stream of the device's greatest priority,
 *                   forked from and joined back into load_stream, so its CTAs are dispatched
 *                   ahead of any attention CTA waiting for them (no caller priority needed);
 *                   compute_stream: attn(0), attn(1), ... each acquiring its layer's counter
 *                   in-kernel before its first load (the suffix append is fused into the
 *                   attention), so gather(l+1) overlaps attn(l).  With the copy-engine / TMA
 *                   baselines, the context split or a wrapping host_io ring: gather(l) -> record
 *                   ev_load[l] on load_stream, wait ev_load[l] -> attn(l) on compute_stream.
 *   mode 1 SYNC:    everything in order on compute_stream (load(l), attn(l)).
 * compute_stream is the stream the caller synchronises on (load_stream is joined into it
 * at the end).  layer_times_ms (nullable) = [2L] floats: per-layer gather and attention
 * durations from CUDA events (streamed gather: its busy time / L for every layer, and each
 * attention's time includes its in-kernel wait for the layer's load); when non-NULL the call
 * blocks until the request's device work has completed. */
pcr_status pcr_run_prefill(pcr_ctx* ctx, int64_t req_id, const void* q_all, const void* k_all,
                           const void* v_all, void* out_all, void* compute_stream,
                           void* load_stream, int32_t mode, float* layer_times_ms);

/* ---------------------------------------------------------------- multi-GPU (§8(e)) - */

/* KV-head sharding: every rank runs the same request on its head slice (pcr_config.rank /
 * world) and the attention outputs are re-assembled with one NCCL all-gather per layer
 * (north_star: "NCCL is used only where outputs must be re-assembled").  NCCL is loaded
 * at run time (dlopen "libnccl.so.2"); nothing else in the library depends on it.
 * pcr_comm_unique_id: ncclGetUniqueId into out[128] (call on one rank, broadcast the bytes).
 * pcr_comm_init: ncclCommInitRank(world, id, rank) for this ctx (collective over ranks).
 * PCR_E_UNSUPPORTED if NCCL cannot be loaded; PCR_E_CUDA on an NCCL error. */
pcr_status pcr_comm_unique_id(uint8_t* out);
pcr_status pcr_comm_init(pcr_ctx* ctx, const uint8_t* id);

/* pcr_run_prefill plus, per layer, after attn(l): comm_stream waits for it and runs
 * ncclAllGather(out_l -> gathered_l), so the gather of layer l overlaps the work of layer l+1.
 * gathered_all = [L][world][N2][Hq_loc][d] (rank-major; rank r's block holds query heads
 * [r*Hq/world, (r+1)*Hq/world)).  compute_stream is joined after the last all-gather.
 * shard_mode 1: `out_all` receives the merged bf16 output [L][N2][Hq][d] and gathered_all is a
 * device fp32 scratch [L][world][N2*Hq*(d+1)]: after attn(l) the comm stream all-gathers this
 * rank's partial of layer l (library-owned) and merges the world partials into out_all[l].
 * PCR_E_STATE if pcr_comm_init has not been called. */
pcr_status pcr_run_prefill_sharded(pcr_ctx* ctx, int64_t req_id, const void* q_all, const void* k_all,
                                   const void* v_all, void* out_all, void* gathered_all,
                                   void* compute_stream, void* load_stream, void* comm_stream,
                                   int32_t mode, float* layer_times_ms);

/* ---------------------------------------------------------------- offload (§8 f1) --- */

/* f1 — layer-wise offload of the request's new chunks (gpu_to_cpu, Alg.1; P:166,
 * P:400 "offloading can commence immediately after each layer's computation"): enqueue on
 * offload_stream the copy of layer `layer` of every reserved chunk from its pool pages into its
 * store slot (16-byte SM loads from HBM, 16-byte stores over PCIe into the mapped store).  The
 * caller orders it after pcr_prefill_attn_layer(layer) (which appended the suffix K/V).  Once
 * all layers' copies have completed, pcr_release(commit=1) makes the chunks RESIDENT. */
pcr_status pcr_offload_layer_kv(pcr_ctx* ctx, int64_t req_id, int32_t layer, void* offload_stream);

/* Options of pcr_run_prefill_ex: the paper's three streams + the optional all-gather. */
typedef struct pcr_run_opts {
  void* compute_stream;    /* required; joined with every other stream at the end */
  void* load_stream;       /* required in OVERLAP / ONLY_UP mode (distinct from compute_stream) */
  void* offload_stream;    /* nullable: offload reserved chunks layer by layer on this stream */
  void* comm_stream;       /* required iff gathered_all != NULL */
  void* gathered_all;      /* nullable: per-layer NCCL all-gather target (pcr_run_prefill_sharded) */
  float* layer_times_ms;   /* nullable: [3L] per-layer gather, append+attention, offload (ms); blocks */
  int32_t mode;            /* 0 OVERLAP (layer-wise loading and offloading both overlapped: the
                            * paper's Up-Down), 1 SYNC (everything in order on compute_stream),
                            * 2 ONLY_UP (loads overlapped, offload in order after each layer's
                            * attention on compute_stream), 3 ONLY_DOWN (loads in order on
                            * compute_stream, offload overlapped) — P:703, fig:breakdown.
                            * Without an offload stream 2 == 0 and 3 == 1. */
  int32_t host_io;         /* 1: q_all/k_all/v_all/out_all are PAGE-LOCKED HOST buffers (cudaHostAlloc /
                            * cudaHostRegister; PCR_E_INVAL otherwise).  Layer l's q/k/v are copied
                            * into a library-owned ring of device staging buffers (as many layers
                            * as fit 512 MiB, >= 2) on the load stream by layer l's gather launch
                            * itself when the buffers are device-mapped (else one cudaMemcpyAsync
                            * each, just ahead of the load), and its output is copied back on an
                            * internal stream right after its attention, so the host I/O overlaps
                            * the layer pipeline.  Not combinable with gathered_all.  The staging
                            * ring is per context: host_io calls of one ctx must not overlap in
                            * time (synchronise the compute stream between them). */
  int32_t io_ring_layers;  /* host_io staging ring depth in layers: 0 = as many as fit 512 MiB
                            * (clamped to [2, L]); otherwise clamped to [2, L]. */
  float* partial_all;      /* shard_mode 1 (required there, NULL otherwise): device fp32
                            * [L][N2*Hq*(d+1)]; layer l's block holds this rank's partial O
                            * ([N2][Hq][d], normalised by its own row sums) followed by its
                            * log2-domain LSE ([N2][Hq]; -inf for rows that see no key here).
                            * out_all is not written (may be NULL) unless gathered_all is set. */
  void* prefill_done_event; /* nullable cudaEvent_t: recorded on compute_stream right after the last
                            * layer's attention, before the offload / all-gather / host_io streams are
                            * joined -- the request's prefill (its first token) is complete when it
                            * completes, while layer-wise offloads may still be running */
} pcr_run_opts;

/* The full per-request pipeline: pcr_run_prefill + (optional) offload on a third stream, the
 * per-layer event chain being load(l) -> append+attn(l) -> offload(l) (and -> all-gather(l));
 * with host_io, [H2D q/k/v(l) -> load(l)] -> append+attn(l) -> [D2H out(l)] (internal stream). */
pcr_status pcr_run_prefill_ex(pcr_ctx* ctx, int64_t req_id, const void* q_all, const void* k_all,
                              const void* v_all, void* out_all, const pcr_run_opts* opts);

/* Count of kernels launched by this ctx since creation (bench `gpu_launches`). */
int64_t pcr_kernel_launches(const pcr_ctx* ctx);

/* shard_mode 1: merge n_parts partial blocks (gathered [n_parts][N2*Hq*(d+1)], device, each
 * laid out as pcr_run_opts.partial_all's per-layer block) into bf16 out [N2][Hq][d] on stream:
 * out = sum_p 2^(lse_p - M) O_p / sum_p 2^(lse_p - M), M = max_p lse_p (the split-KV combine). */
pcr_status pcr_merge_partials(pcr_ctx* ctx, const float* gathered, int32_t n_parts, int64_t n2, void* out,
                              void* stream);

/* Switch the a2 load path (pcr_config.load_mode / load_ce_fraction, same ranges) for layer loads
 * enqueued after this call; call it between requests.  PCR_E_INVAL on an out-of-range value
 * (nothing changes). */
pcr_status pcr_set_load_mode(pcr_ctx* ctx, int32_t load_mode, float load_ce_fraction);

#ifdef __cplusplus
}
#endif
#endif /* PCR_H_ */
