"""O2 extension — the SSD tier: queue-based SSD->DRAM prefetch and asynchronous
write-back.  (Oracle: test infrastructure only.)

Paper passages, in the paper's order:
  P:456   "the prefetcher maintains a look-ahead window ... checks the KV-cache status of these
          requests in both DRAM and SSD. If a KV cache is found on the SSD but not yet in DRAM,
          the prefetcher launches asynchronous loading tasks to transfer it into DRAM" (R1 in
          DRAM -> nothing; R2, R4 on SSD -> tasks; R3 in neither -> recompute).
  P:458   "after completing one forward pass, the system must write all KV caches back into CPU
          memory. Once this step is done, the Cache Engine immediately submits asynchronous
          write-back tasks to persist the data onto SSDs".
  Alg.1   P:488-495 prefetch phase: in CPU -> BumpPriority, in SSD -> SubmitSSDToCPULoad, else
          break; P:499-505 plan phase: in CPU -> cpu_to_gpu, in SSD -> trigger load and
          ssd_to_gpu, else gpu_to_cpu; P:512 DrainCompletedSSDLoads.

Readings (R19-R23), chosen so that every decision is independent of I/O timing:
  R19 the SSD is a flat LRU key->record store of committed chunks (capacity in chunks); a
      write-back of every committed chunk is submitted at release(commit); when the
      SSD is full the least recently used entry is overwritten.  Loads and writes touch MRU.
  R20 a prefetch (bump phase) of an SSD-only chunk reserves a DRAM slot exactly like a new
      chunk (lowest free, else leaf-LRU eviction), inserts the node LOADING and io-pinned; it
      becomes RESIDENT when drained.  The walk continues past it (it is retrievable).
  R21 match treats LOADING chunks as present and loads SSD-only chunks of the request's own
      chain on demand (ssd_to_gpu); the call returns only when those are in DRAM.
  R22 DrainCompletedSSDLoads = pcr_release of the request whose match submitted the loads
      waits for them (the reads overlap that request's GPU work).
  R23 a chunk whose key is on the SSD is never reserved as new (reserve stops there).
  R24 the scheduled request's DRAM-resident chain is protected (temporarily pinned) during the
      prefetch phase, so look-ahead loads never evict the chunks of the request about to run.
  R25 while one pending request's chain is walked, the chunks already walked are protected
      until that walk ends (a load never evicts the prefix it is being attached to).
"""
from __future__ import annotations

from collections import OrderedDict

from .chunks import ROOT_KEY
from .tree import RESIDENT, Node, PlanError, PlanOracle

LOADING = 2


class TieredPlanOracle(PlanOracle):
    def __init__(self, C, S_pg, store_chunks, n_pages, window, ssd_chunks):
        super().__init__(C, S_pg, store_chunks, n_pages, window)
        self.ssd_cap = ssd_chunks
        self.ssd = OrderedDict()            # key -> (ssd_slot, parent_key, tokens), LRU first
        self.free_ssd = set(range(ssd_chunks))
        self.stats = dict(prefetch=0, ondemand=0, writeback=0, ssd_evict=0, dram_evict=0)
        self.loads = {}                     # req -> keys loaded by its match (drained at release)

    # ---- helpers ------------------------------------------------------------------
    def _on_ssd(self, key, parent, tok):
        e = self.ssd.get(key)
        return e is not None and e[1] == parent and e[2] == tok

    def _take_slot(self):
        if not self.free_slots:
            victim = next((k for k in self.leaves
                           if self.nodes[k].pins == 0 and self.nodes[k].state == RESIDENT), None)
            if victim is None:
                return None
            vn = self.nodes.pop(victim)
            self.leaves.remove(victim)
            self.free_slots.add(vn.slot)
            self._evicted.append((victim, vn.slot))
            self.stats["dram_evict"] += 1
            pch = self._children(vn.parent)
            pch.discard(victim)
            if vn.parent != ROOT_KEY and not pch:
                self._become_leaf(vn.parent)
        slot = min(self.free_slots)
        self.free_slots.remove(slot)
        return slot

    def _insert(self, key, parent, tok, state, pins):
        slot = self._take_slot()
        if slot is None:
            return False
        if parent != ROOT_KEY and parent in self.leaves:
            self.leaves.remove(parent)
        self._children(parent).add(key)
        self.nodes[key] = Node(key, parent, tok, slot, state, pins=pins)
        self._become_leaf(key)
        return True

    def _load(self, req_id, key, parent, tok, kind):
        """Start an SSD->DRAM load: a LOADING node holding an io pin."""
        if not self._insert(key, parent, tok, LOADING, pins=1):
            return False
        self.ssd.move_to_end(key)
        self.loads.setdefault(req_id, []).append(key)
        self.stats[kind] += 1
        return True

    def _drain(self, keys):
        for k in keys:
            n = self.nodes[k]
            if n.state == LOADING:
                n.state = RESIDENT
                n.pins -= 1

    # ---- API ----------------------------------------------------------------------
    def match_prefix(self, req_id: int, pending_ids=()):
        r = self.reqs.get(req_id)
        if r is None:
            raise PlanError("NOREQ", "unknown request")
        if r.planned:
            raise PlanError("STATE", "request already planned")
        pend = list(pending_ids)[: self.window]
        if req_id in pend or len(set(pend)) != len(pend):
            raise PlanError("INVAL", "pending ids contain the request or duplicates")
        for p in pend:
            if p not in self.reqs:
                raise PlanError("NOREQ", "unknown pending request")
        N = len(r.tokens)
        need_pages = -(-N // self.S_pg)
        if need_pages > len(self.free_pages):
            raise PlanError("NOMEM", "pool pages exhausted")
        self._evicted = []

        # 0. protect the scheduled request's resident chain during the prefetch phase (R24)
        guard, parent = [], ROOT_KEY
        for key, tok in zip(r.keys, r.chunk_tokens):
            if not (self._valid_child(key, parent, tok) and self.nodes[key].state == RESIDENT):
                break
            self.nodes[key].pins += 1
            guard.append(key)
            parent = key

        # 1. prefetch phase over Reverse(window): DRAM -> bump, SSD -> load task, else break
        for p in reversed(pend):
            pr = self.reqs[p]
            parent, walked = ROOT_KEY, []
            for key, tok in zip(pr.keys, pr.chunk_tokens):
                if self._valid_child(key, parent, tok) and self.nodes[key].state in (RESIDENT, LOADING):
                    self._touch(key)
                elif key not in self.nodes and self._on_ssd(key, parent, tok):
                    if not self._load(req_id, key, parent, tok, "prefetch"):
                        break
                else:
                    break
                self.nodes[key].pins += 1          # R25
                walked.append(key)
                parent = key
            for key in walked:
                self.nodes[key].pins -= 1

        for key in guard:
            self.nodes[key].pins -= 1

        # 2. match + pin; SSD-only chunks of this chain are loaded on demand (ssd_to_gpu)
        parent, matched, ondemand = ROOT_KEY, [], 0
        for key, tok in zip(r.keys, r.chunk_tokens):
            if self._valid_child(key, parent, tok) and self.nodes[key].state in (RESIDENT, LOADING):
                self._touch(key)
            elif key not in self.nodes and self._on_ssd(key, parent, tok):
                if not self._load(req_id, key, parent, tok, "ondemand"):
                    break
                ondemand += 1
            else:
                break
            self.nodes[key].pins += 1
            matched.append(key)
            parent = key

        # 3. reserve new chunks (R23: not for keys on the SSD)
        reserved = []
        for key, tok in zip(r.keys[len(matched):], r.chunk_tokens[len(matched):]):
            if key in self.nodes or key in self.ssd:
                break
            if not self._insert(key, parent, tok, 0, pins=1):
                break
            reserved.append(key)
            parent = key

        # 4. pages; the request's own chain must be in DRAM when match returns (R21)
        pages = sorted(self.free_pages)[:need_pages]
        self.free_pages.difference_update(pages)
        self._drain([k for k in matched if self.nodes[k].state == LOADING])
        r.planned, r.matched, r.reserved, r.pages = True, matched, reserved, pages
        n1 = len(matched) * self.C
        return dict(
            n_matched=len(matched), n_reserved=len(reserved), n1=n1, n2=N - n1,
            slots=[self.nodes[k].slot for k in matched + reserved], pages=list(pages),
            evicted=list(self._evicted), matched_keys=list(matched), reserved_keys=list(reserved),
            n_from_ssd=ondemand,
        )

    def release(self, req_id: int, commit: bool = True):
        r = self.reqs.get(req_id)
        if r is None:
            raise PlanError("NOREQ", "unknown request")
        if not r.planned:
            raise PlanError("STATE", "request not planned")
        self._drain(self.loads.pop(req_id, []))            # DrainCompletedSSDLoads (R22)
        reserved = list(r.reserved)
        super().release(req_id, commit)
        if commit and self.ssd_cap > 0:                     # asynchronous write-back
            for k in reserved:
                n = self.nodes[k]
                if k in self.ssd:
                    self.ssd.move_to_end(k)
                    continue
                if not self.free_ssd:
                    old, (slot, _, _) = self.ssd.popitem(last=False)
                    self.free_ssd.add(slot)
                    self.stats["ssd_evict"] += 1
                slot = min(self.free_ssd)
                self.free_ssd.remove(slot)
                self.ssd[k] = (slot, n.parent, n.tokens)
                self.stats["writeback"] += 1

    def ssd_slot(self, key):
        return self.ssd[key][0]
