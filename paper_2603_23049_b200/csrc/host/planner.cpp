// Prefix tree + look-ahead leaf-LRU planner (see planner.h for the paper passages).
#include "planner.h"

#include <algorithm>
#include <cstring>

#include "blake2b.h"

namespace pcr {

Planner::Planner(int32_t C, int32_t S, int64_t store_chunks, int64_t n_pages, int32_t window,
                 int32_t max_regions, int64_t ssd_chunks)
    : C_(C), S_(S), window_(window), n_slots_(store_chunks), n_pages_(n_pages), ssd_cap_(ssd_chunks) {
  for (int64_t i = 0; i < ssd_chunks; ++i) free_ssd_.insert(static_cast<int32_t>(i));
  for (int64_t i = 0; i < store_chunks; ++i) free_slots_.insert(static_cast<int32_t>(i));
  for (int64_t i = 0; i < n_pages; ++i) free_pages_.insert(static_cast<int32_t>(i));
  for (int32_t i = 0; i < max_regions; ++i) free_regions_.insert(i);
}

// HashPrefix(chunk, parent) (Alg.1): BLAKE2b-128(parent || tokens as LE uint32).
Key Planner::chunk_key(const Key& parent, const uint32_t* tokens, int32_t n) {
  Blake2b s;
  blake2b_init(&s, 16, nullptr, 0);
  blake2b_update(&s, parent.data(), 16);
  uint8_t le[4];
  for (int32_t i = 0; i < n; ++i) {  // explicit little-endian serialisation
    le[0] = static_cast<uint8_t>(tokens[i]);
    le[1] = static_cast<uint8_t>(tokens[i] >> 8);
    le[2] = static_cast<uint8_t>(tokens[i] >> 16);
    le[3] = static_cast<uint8_t>(tokens[i] >> 24);
    blake2b_update(&s, le, 4);
  }
  Key k;
  blake2b_final(&s, k.data());
  return k;
}

// ---- leaf list: R1 append at MRU, R2 remove, R3 touch ------------------------------
void Planner::list_append(int32_t n) {
  Node& x = nodes_[n];
  x.prev = tail_;
  x.next = -1;
  if (tail_ >= 0) nodes_[tail_].next = n; else head_ = n;
  tail_ = n;
  x.in_list = true;
}

void Planner::list_remove(int32_t n) {
  Node& x = nodes_[n];
  if (!x.in_list) return;
  if (x.prev >= 0) nodes_[x.prev].next = x.next; else head_ = x.next;
  if (x.next >= 0) nodes_[x.next].prev = x.prev; else tail_ = x.prev;
  x.prev = x.next = -1;
  x.in_list = false;
}

void Planner::touch(int32_t n) {
  if (!nodes_[n].in_list) return;  // R3: internal nodes are not in the LRU order
  list_remove(n);
  list_append(n);
}

int32_t Planner::valid_child(const Key& key, int32_t parent, const uint32_t* toks) const {
  auto it = index_.find(key);
  if (it == index_.end()) return -1;
  const Node& x = nodes_[it->second];
  if (x.parent != parent) return -1;
  if (std::memcmp(x.tokens.data(), toks, sizeof(uint32_t) * C_) != 0) return -1;
  return it->second;
}

int32_t Planner::new_node() {
  int32_t n;
  if (!free_nodes_.empty()) {
    n = free_nodes_.back();
    free_nodes_.pop_back();
  } else {
    n = static_cast<int32_t>(nodes_.size());
    nodes_.emplace_back();
  }
  nodes_[n] = Node();
  nodes_[n].live = true;
  return n;
}

void Planner::remove_node(int32_t n) {
  Node& x = nodes_[n];
  list_remove(n);
  index_.erase(x.key);
  free_slots_.insert(x.slot);
  if (x.parent >= 0) {
    Node& p = nodes_[x.parent];
    if (--p.n_children == 0) list_append(x.parent);  // "its parent becomes a new leaf"
  }
  x.live = false;
  x.tokens.clear();
  free_nodes_.push_back(n);
}

// ---- API ------------------------------------------------------------------------------
int32_t Planner::submit(int64_t id, const uint32_t* tokens, int64_t n, int64_t n_cacheable,
                        std::string* err) {
  if (tokens == nullptr || n < 1 || n_cacheable < 0 || n_cacheable > n) {
    *err = "pcr_submit: need n_tokens >= 1, 0 <= n_cacheable <= n_tokens, tokens != NULL";
    return kInval;
  }
  if (reqs_.count(id)) {
    *err = "pcr_submit: request id already registered";
    return kState;
  }
  Request r;
  r.tokens.assign(tokens, tokens + n);
  // Reading R5: min(n_cacheable / C, (n - 1) / C) chunks, so that N2 >= 1.
  const int64_t m = std::min<int64_t>(n_cacheable / C_, (n - 1) / C_);
  Key parent{};
  for (int64_t i = 0; i < m; ++i) {
    parent = chunk_key(parent, tokens + i * C_, C_);
    r.keys.push_back(parent);
  }
  reqs_.emplace(id, std::move(r));
  return kOk;
}

int32_t Planner::match_prefix(int64_t id, const int64_t* pending, int32_t n_pending,
                              int64_t cap_slots, int64_t cap_pages, int64_t cap_evicted,
                              std::string* err) {
  auto it = reqs_.find(id);
  if (it == reqs_.end()) { *err = "pcr_match_prefix: unknown request"; return kNoReq; }
  Request& r = it->second;
  if (r.planned) { *err = "pcr_match_prefix: request already planned"; return kState; }
  if (n_pending < 0 || (n_pending > 0 && pending == nullptr)) {
    *err = "pcr_match_prefix: bad pending list"; return kInval;
  }
  const int32_t w = std::min(n_pending, window_);
  for (int32_t i = 0; i < w; ++i) {
    if (pending[i] == id) { *err = "pcr_match_prefix: pending ids contain the request"; return kInval; }
    for (int32_t j = 0; j < i; ++j)
      if (pending[j] == pending[i]) { *err = "pcr_match_prefix: duplicate pending id"; return kInval; }
  }
  for (int32_t i = 0; i < w; ++i)
    if (!reqs_.count(pending[i])) { *err = "pcr_match_prefix: unknown pending request"; return kNoReq; }
  const int64_t N = static_cast<int64_t>(r.tokens.size());
  const int64_t need_pages = (N + S_ - 1) / S_;
  if (need_pages > static_cast<int64_t>(free_pages_.size())) {
    *err = "pcr_match_prefix: pool pages exhausted"; return kNoMem;
  }
  if (free_regions_.empty()) { *err = "pcr_match_prefix: too many requests in flight"; return kNoMem; }
  // Capacity checks need the outcome; simulate-free upper bounds keep the strong guarantee.
  const int64_t n_chain = static_cast<int64_t>(r.keys.size());
  if ((cap_slots >= 0 && cap_slots < n_chain) || (cap_pages >= 0 && cap_pages < need_pages) ||
      (cap_evicted >= 0 && cap_evicted < n_chain)) {
    *err = "pcr_match_prefix: output capacity too small (need slots >= chain chunks, "
           "pages >= ceil(N/S_pg), evicted >= chain chunks)";
    return kInval;
  }

  Plan& pl = r.plan;
  pl = Plan();
  cur_ = &pl;
  r.matched.clear();
  r.reserved.clear();
  r.loads.clear();

  // 0. protect the scheduled request's resident chain during the prefetch phase (R24)
  std::vector<int32_t> guard;
  {
    int32_t parent = -1;
    for (size_t c = 0; c < r.keys.size(); ++c) {
      int32_t n = valid_child(r.keys[c], parent, r.tokens.data() + c * C_);
      if (n < 0 || nodes_[n].state != kResident) break;
      nodes_[n].pins++;
      guard.push_back(n);
      parent = n;
    }
  }
  // 1. prefetch phase over Reverse(pending window) (Alg.1): in CPU -> BumpPriority
  //    (recency touch); on SSD -> SubmitSSDToCPULoad; else break.
  std::vector<int32_t> walked;
  for (int32_t i = w - 1; i >= 0; --i) {
    const Request& pr = reqs_.at(pending[i]);
    int32_t parent = -1;
    walked.clear();
    for (size_t c = 0; c < pr.keys.size(); ++c) {
      const uint32_t* toks = pr.tokens.data() + c * C_;
      int32_t n = valid_child(pr.keys[c], parent, toks);
      if (n >= 0 && (nodes_[n].state == kResident || nodes_[n].state == kLoading)) {
        touch(n);
      } else if (n < 0 && !index_.count(pr.keys[c]) && on_ssd(pr.keys[c], key_of(parent), toks)) {
        n = start_load(r, pr.keys[c], parent, toks, false);
        if (n < 0) break;
      } else {
        break;
      }
      nodes_[n].pins++;  // R25: the walked prefix is protected until this walk ends
      walked.push_back(n);
      parent = n;
    }
    for (int32_t n : walked) nodes_[n].pins--;
  }
  for (int32_t n : guard) nodes_[n].pins--;

  // 2. match + pin ("until a mismatch occurs"; P:480 recency update); SSD-only chunks of
  //    this chain are loaded on demand (ssd_to_gpu, Alg.1).
  int32_t parent = -1;
  size_t c = 0;
  for (; c < r.keys.size(); ++c) {
    const uint32_t* toks = r.tokens.data() + c * C_;
    int32_t n = valid_child(r.keys[c], parent, toks);
    if (n >= 0 && (nodes_[n].state == kResident || nodes_[n].state == kLoading)) {
      touch(n);
    } else if (n < 0 && !index_.count(r.keys[c]) && on_ssd(r.keys[c], key_of(parent), toks)) {
      n = start_load(r, r.keys[c], parent, toks, true);
      if (n < 0) break;
      pl.n_from_ssd++;
    } else {
      break;
    }
    nodes_[n].pins++;
    r.matched.push_back(n);
    parent = n;
  }
  // 3. reserve slots for the new chunks (gpu_to_cpu, Alg.1), evicting leaves; never for a
  //    chunk that exists (PENDING elsewhere, or on the SSD: R17, R23).
  for (; c < r.keys.size(); ++c) {
    if (index_.count(r.keys[c]) || ssd_.count(r.keys[c])) break;
    const int32_t n = insert(r.keys[c], parent, r.tokens.data() + c * C_, kPending, 1);
    if (n < 0) break;  // starvation: stop reserving (reading R11)
    r.reserved.push_back(n);
    pl.new_slots.push_back(nodes_[n].slot);
    parent = n;
  }
  // 4. pool pages, lowest free first; the chain's loads must complete before returning (R21).
  auto pit = free_pages_.begin();
  for (int64_t i = 0; i < need_pages; ++i) {
    pl.pages.push_back(*pit);
    pit = free_pages_.erase(pit);
  }
  for (int32_t n : r.matched) {
    if (nodes_[n].state != kLoading) continue;
    nodes_[n].state = kResident;
    nodes_[n].pins--;
    for (IoOp& op : pl.loads)
      if (op.dram_slot == nodes_[n].slot) op.wait_now = true;
  }
  pl.region = *free_regions_.begin();
  free_regions_.erase(free_regions_.begin());
  pl.n_matched = static_cast<int32_t>(r.matched.size());
  pl.n_reserved = static_cast<int32_t>(r.reserved.size());
  pl.n1 = static_cast<int64_t>(pl.n_matched) * C_;
  pl.n2 = N - pl.n1;
  for (int32_t n : r.matched) pl.slots.push_back(nodes_[n].slot);
  for (int32_t n : r.reserved) pl.slots.push_back(nodes_[n].slot);
  r.planned = true;
  r.tables_uploaded = false;
  cur_ = nullptr;
  return kOk;
}

bool Planner::on_ssd(const Key& key, const Key& parent, const uint32_t* toks) const {
  auto it = ssd_.find(key);
  return it != ssd_.end() && it->second.parent == parent &&
         std::memcmp(it->second.tokens.data(), toks, sizeof(uint32_t) * C_) == 0;
}

int32_t Planner::take_slot() {
  if (free_slots_.empty()) {
    int32_t victim = -1;
    for (int32_t n = head_; n >= 0; n = nodes_[n].next)
      if (nodes_[n].pins == 0 && nodes_[n].state == kResident) { victim = n; break; }
    if (victim < 0) return -1;
    if (cur_) cur_->evicted.emplace_back(nodes_[victim].key, nodes_[victim].slot);
    stats_.dram_evict++;
    remove_node(victim);
  }
  const int32_t slot = *free_slots_.begin();
  free_slots_.erase(free_slots_.begin());
  return slot;
}

int32_t Planner::insert(const Key& key, int32_t parent, const uint32_t* toks, int32_t state, int32_t pins) {
  const int32_t slot = take_slot();
  if (slot < 0) return -1;
  const int32_t n = new_node();
  Node& x = nodes_[n];
  x.key = key;
  x.parent = parent;
  x.slot = slot;
  x.state = state;
  x.pins = pins;
  x.tokens.assign(toks, toks + C_);
  if (parent >= 0) {
    if (nodes_[parent].n_children++ == 0) list_remove(parent);  // R2
  }
  index_.emplace(key, n);
  list_append(n);  // R1
  return n;
}

// SSD -> DRAM load of one chunk (P:456 SubmitSSDToCPULoad / on-demand ssd_to_gpu): the node is
// LOADING and holds an io pin until drained (R20-R22).
int32_t Planner::start_load(Request& r, const Key& key, int32_t parent, const uint32_t* toks, bool ondemand) {
  const int32_t n = insert(key, parent, toks, kLoading, 1);
  if (n < 0) return -1;
  SsdEntry& e = ssd_.at(key);
  ssd_lru_.splice(ssd_lru_.end(), ssd_lru_, e.lru);
  cur_->loads.push_back(IoOp{nodes_[n].slot, e.slot, false});
  cur_->new_slots.push_back(nodes_[n].slot);
  r.loads.push_back(n);
  if (ondemand) stats_.ondemand++; else stats_.prefetch++;
  return n;
}

int32_t Planner::release(int64_t id, bool commit, std::string* err, std::vector<IoOp>* writes) {
  auto it = reqs_.find(id);
  if (it == reqs_.end()) { *err = "pcr_release: unknown request"; return kNoReq; }
  Request& r = it->second;
  if (!r.planned) { *err = "pcr_release: request not planned"; return kState; }
  for (int32_t n : r.matched) {
    if (!nodes_[n].live || nodes_[n].pins <= 0) { *err = "pcr_release: pin underflow"; return kInternal; }
  }
  // DrainCompletedSSDLoads (Alg.1; R22): this request's prefetches are now in DRAM.
  for (int32_t n : r.loads) {
    if (nodes_[n].live && nodes_[n].state == kLoading) {
      nodes_[n].state = kResident;
      nodes_[n].pins--;
    }
  }
  for (int32_t n : r.matched) nodes_[n].pins--;
  for (int32_t n : r.reserved) nodes_[n].pins--;
  if (commit) {
    for (int32_t n : r.reserved) nodes_[n].state = kResident;
    // asynchronous write-back of the new chunks to the SSD (R19)
    if (ssd_cap_ > 0) {
      for (int32_t n : r.reserved) {
        const Node& x = nodes_[n];
        auto e = ssd_.find(x.key);
        if (e != ssd_.end()) {
          ssd_lru_.splice(ssd_lru_.end(), ssd_lru_, e->second.lru);
          continue;
        }
        if (free_ssd_.empty()) {
          auto old = ssd_.find(ssd_lru_.front());
          free_ssd_.insert(old->second.slot);
          ssd_.erase(old);
          ssd_lru_.pop_front();
          stats_.ssd_evict++;
        }
        const int32_t slot = *free_ssd_.begin();
        free_ssd_.erase(free_ssd_.begin());
        ssd_lru_.push_back(x.key);
        ssd_.emplace(x.key, SsdEntry{slot, key_of(x.parent), x.tokens, std::prev(ssd_lru_.end())});
        stats_.writeback++;
        if (writes) writes->push_back(IoOp{x.slot, slot, false});
      }
    }
  } else {
    for (auto rit = r.reserved.rbegin(); rit != r.reserved.rend(); ++rit) {
      if (nodes_[*rit].n_children != 0) { *err = "pcr_release: InconsistentDrop"; return kInternal; }
      remove_node(*rit);  // deepest first
    }
  }
  for (int32_t p : r.plan.pages) free_pages_.insert(p);
  free_regions_.insert(r.plan.region);
  reqs_.erase(it);
  return kOk;
}

std::vector<Key> Planner::leaf_list() const {
  std::vector<Key> out;
  for (int32_t n = head_; n >= 0; n = nodes_[n].next) out.push_back(nodes_[n].key);
  return out;
}

}  // namespace pcr
