// Host control of the hot path: chunk keys, the prefix tree with a
// look-ahead leaf-LRU list, store-slot and pool-page allocation.  No CUDA here.
//
// Paper: §4.2 P:362-364 (prefix tree, leaf-only LRU eviction, look-ahead priority bump),
// §5 P:480 (window of waiting requests "update the recency for matched chunks"),
// Alg.1 P:487-507 (bump over Reverse(prefetch_reqs), then plan cpu_to_gpu/gpu_to_cpu,
// AdjustTokens), P:518 (computation only on confirmed-present chunks).
// Policy readings R1-R3, R5, R7-R12 are listed in DESIGN.md.
#pragma once

#include <array>
#include <cstdint>
#include <list>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

namespace pcr {

using Key = std::array<uint8_t, 16>;

struct KeyHash {
  size_t operator()(const Key& k) const noexcept {
    uint64_t a;
    __builtin_memcpy(&a, k.data(), 8);
    return static_cast<size_t>(a);
  }
};

enum : int32_t { kPending = 0, kResident = 1, kLoading = 2 };

// Status codes mirror pcr_status (include/pcr.h).
enum : int32_t { kOk = 0, kInval = -1, kNoMem = -2, kState = -4, kNoReq = -5, kInternal = -6 };

struct Node {
  Key key;
  int32_t parent = -1;     // node index, -1 = root
  int32_t slot = -1;
  int32_t state = kPending;
  int32_t pins = 0;
  int32_t n_children = 0;
  int32_t prev = -1, next = -1;  // intrusive leaf-list links
  bool in_list = false;
  bool live = false;
  std::vector<uint32_t> tokens;
};

// An SSD<->DRAM transfer the runtime must execute (the planner itself does no I/O).
struct IoOp {
  int32_t dram_slot, ssd_slot;
  bool wait_now;           // loads: the call must not return before it completes (own chain)
};

struct Plan {
  int32_t n_matched = 0, n_reserved = 0;
  int64_t n1 = 0, n2 = 0;
  std::vector<int32_t> slots, pages;
  std::vector<std::pair<Key, int32_t>> evicted;
  int32_t region = -1;     // device plan-table region
  int32_t n_from_ssd = 0;  // chunks of this chain loaded from SSD on demand (ssd_to_gpu)
  std::vector<IoOp> loads; // SSD -> DRAM reads submitted by this match (prefetch + on demand)
  std::vector<int32_t> new_slots;  // DRAM slots (re)assigned by this match
};

struct TierStats {
  int64_t prefetch = 0, ondemand = 0, writeback = 0, ssd_evict = 0, dram_evict = 0;
};

struct Request {
  std::vector<uint32_t> tokens;
  std::vector<Key> keys;   // cacheable chunk chain
  bool planned = false;
  std::vector<int32_t> matched, reserved;  // node indices
  Plan plan;
  bool tables_uploaded = false;
  // shard_mode 1 (context split), runtime-owned: this rank's matched / reserved chunks, virtual
  // page-table length, and whether it holds the suffix keys
  int32_t ctx_n_own = 0, ctx_n_res_own = 0, ctx_n_vpages = 0;
  bool ctx_suffix = true;
  std::vector<int32_t> loads;      // LOADING nodes this request's match started (drained at release)
};

class Planner {
 public:
  Planner(int32_t chunk_tokens, int32_t page_tokens, int64_t store_chunks, int64_t n_pages,
          int32_t window, int32_t max_regions, int64_t ssd_chunks = 0);

  int32_t submit(int64_t id, const uint32_t* tokens, int64_t n, int64_t n_cacheable, std::string* err);
  // Validates first (strong guarantee); `cap_*` are the caller's capacities (-1 = unchecked).
  int32_t match_prefix(int64_t id, const int64_t* pending, int32_t n_pending, int64_t cap_slots,
                       int64_t cap_pages, int64_t cap_evicted, std::string* err);
  // `writes` receives the SSD write-backs of committed chunks (runtime executes them).
  int32_t release(int64_t id, bool commit, std::string* err, std::vector<IoOp>* writes = nullptr);
  const TierStats& stats() const { return stats_; }

  Request* find(int64_t id) {
    auto it = reqs_.find(id);
    return it == reqs_.end() ? nullptr : &it->second;
  }
  std::vector<Key> leaf_list() const;
  int32_t chunk_tokens() const { return C_; }
  int32_t page_tokens() const { return S_; }

  static Key chunk_key(const Key& parent, const uint32_t* tokens, int32_t n);

 private:
  int32_t C_, S_, window_;
  int64_t n_slots_, n_pages_;
  std::vector<Node> nodes_;
  std::vector<int32_t> free_nodes_;
  std::unordered_map<Key, int32_t, KeyHash> index_;
  int32_t head_ = -1, tail_ = -1;          // leaf list: head = LRU, tail = MRU
  std::set<int32_t> free_slots_, free_pages_, free_regions_;
  std::unordered_map<int64_t, Request> reqs_;
  // SSD tier (oracle/tiers.py readings R19-R24): flat LRU key -> record store.
  struct SsdEntry {
    int32_t slot;
    Key parent;
    std::vector<uint32_t> tokens;
    std::list<Key>::iterator lru;
  };
  int64_t ssd_cap_ = 0;
  std::unordered_map<Key, SsdEntry, KeyHash> ssd_;
  std::list<Key> ssd_lru_;  // front = least recently used
  std::set<int32_t> free_ssd_;
  TierStats stats_;
  Plan* cur_ = nullptr;     // plan being built (eviction log)

  bool on_ssd(const Key& key, const Key& parent, const uint32_t* toks) const;
  int32_t take_slot();                        // lowest free DRAM slot, else evict; -1 = starved
  int32_t insert(const Key& key, int32_t parent, const uint32_t* toks, int32_t state, int32_t pins);
  int32_t start_load(Request& r, const Key& key, int32_t parent, const uint32_t* toks, bool ondemand);
  Key key_of(int32_t n) const { return n < 0 ? Key{} : nodes_[n].key; }

  void list_append(int32_t n);
  void list_remove(int32_t n);
  void touch(int32_t n);
  int32_t valid_child(const Key& key, int32_t parent, const uint32_t* toks) const;
  int32_t new_node();
  void remove_node(int32_t n);  // unlink from parent/list/index; parent may become a leaf
};

}  // namespace pcr
