"""O2 — prefix tree of chunks with look-ahead leaf-LRU, and the per-request plan.
(Oracle: test infrastructure only.)

Paper passages followed, in the paper's order (Alg. 1):
  P:362  chunks form a prefix tree; a request is matched "chunk-wise ... starting from the
         root node, until a mismatch occurs".
  P:364  "eviction is restricted to the leaf nodes"; "all leaves are maintained using an
         LRU"; look-ahead "leverages pending requests from the waiting queue ... and
         protect[s] corresponding chunks"; "when C4 is evicted, its parent becomes a new
         leaf and is added to the leaf set; ... upon inserting C9, C8 transitions from a
         leaf to an internal node and is removed from the leaf set".
  P:480  the waiting requests in the preloading window (4) are sent to the cache engine,
         which will "update the recency for matched chunks".
  Alg.1  P:488-495 prefetch phase over Reverse(prefetch_reqs): in CPU -> BumpPriority,
         else break (the SSD branch is out of the hot path); P:499-506 plan phase:
         in CPU -> cpu_to_gpu, else -> gpu_to_cpu (new chunk to offload); AdjustTokens.

Readings (R7-R12), which reproduce the printed example of P:364 exactly,
including its order {C6, C2, C3, C9}:
  * one ordered leaf list, LRU -> MRU;
  * R1  a node that becomes a leaf (inserted, or its last child removed) is appended at MRU;
  * R2  a leaf that gains a child leaves the list;
  * R3  touch(n) moves n to MRU if n is a leaf, else does nothing (BumpPriority and the
        recency update of matched chunks are both touches);
  * bump walks Reverse(pending[:W]) root-first, touching RESIDENT chunks, break at the
    first chunk that is not RESIDENT;
  * matched and reserved chunks are pinned until release; PENDING (reserved, not yet
    written) chunks are neither matchable nor "in CPU" for the bump;
  * reserve = for each remaining cacheable chunk in order: lowest free slot, else evict
    the first unpinned RESIDENT leaf of the list; stop at the first chunk that cannot
    get a slot (starvation) or whose key already exists;
  * pages: ceil(N / S_pg) pool pages, lowest free first.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .chunks import ROOT_KEY, chain_keys

PENDING, RESIDENT = 0, 1


class PlanError(Exception):
    """code is one of 'INVAL', 'NOMEM', 'STATE', 'NOREQ' (the pcr_status names)."""

    def __init__(self, code: str, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclass
class Node:
    key: bytes
    parent: bytes          # ROOT_KEY for a root child
    tokens: bytes
    slot: int
    state: int
    pins: int = 0
    children: set = field(default_factory=set)


@dataclass
class Request:
    tokens: np.ndarray
    keys: list
    chunk_tokens: list     # bytes of each cacheable chunk (for token verification)
    planned: bool = False
    matched: list = field(default_factory=list)
    reserved: list = field(default_factory=list)
    pages: list = field(default_factory=list)


class PlanOracle:
    def __init__(self, C: int, S_pg: int, store_chunks: int, n_pages: int, window: int):
        self.C, self.S_pg, self.window = C, S_pg, window
        self.store_chunks, self.n_pages = store_chunks, n_pages
        self.nodes: dict[bytes, Node] = {}
        self.root_children: set = set()
        self.leaves: list[bytes] = []          # LRU -> MRU
        self.free_slots = set(range(store_chunks))
        self.free_pages = set(range(n_pages))
        self.reqs: dict[int, Request] = {}

    # ---- list rules ---------------------------------------------------------------
    def _children(self, key):
        return self.root_children if key == ROOT_KEY else self.nodes[key].children

    def _become_leaf(self, key):          # R1
        self.leaves.append(key)

    def _touch(self, key):                # R3
        if key in self.leaves:
            self.leaves.remove(key)
            self.leaves.append(key)

    def _valid_child(self, key, parent, tok):
        n = self.nodes.get(key)
        return n is not None and n.parent == parent and n.tokens == tok

    # ---- API ----------------------------------------------------------------------
    def submit(self, req_id: int, tokens, n_cacheable: int | None = None):
        tokens = np.asarray(tokens, dtype=np.uint32)
        if n_cacheable is None:
            n_cacheable = len(tokens)
        if req_id in self.reqs:
            raise PlanError("STATE", "request id already submitted")
        if not (0 <= n_cacheable <= len(tokens)) or len(tokens) < 1:
            raise PlanError("INVAL", "n_cacheable out of range")
        keys = chain_keys(tokens, self.C, n_cacheable)
        chunks = [tokens[i * self.C:(i + 1) * self.C].astype("<u4").tobytes() for i in range(len(keys))]
        self.reqs[req_id] = Request(tokens, keys, chunks)

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

        # 1. look-ahead bump: Reverse(pending window), root-first, break at first non-resident.
        for p in reversed(pend):
            pr = self.reqs[p]
            parent = ROOT_KEY
            for key, tok in zip(pr.keys, pr.chunk_tokens):
                if not (self._valid_child(key, parent, tok) and self.nodes[key].state == RESIDENT):
                    break
                self._touch(key)
                parent = key

        # 2. match + pin (recency update of matched chunks).
        parent, matched = ROOT_KEY, []
        for key, tok in zip(r.keys, r.chunk_tokens):
            if not (self._valid_child(key, parent, tok) and self.nodes[key].state == RESIDENT):
                break
            self._touch(key)
            self.nodes[key].pins += 1
            matched.append(key)
            parent = key

        # 3. reserve slots for the remaining cacheable chunks (gpu_to_cpu, Alg.1).
        reserved, evicted = [], []
        for key, tok in zip(r.keys[len(matched):], r.chunk_tokens[len(matched):]):
            if key in self.nodes:
                break
            if not self.free_slots:
                victim = next((k for k in self.leaves
                               if self.nodes[k].pins == 0 and self.nodes[k].state == RESIDENT), None)
                if victim is None:
                    break                      # starvation: stop reserving (reading R11)
                vn = self.nodes.pop(victim)
                self.leaves.remove(victim)
                self.free_slots.add(vn.slot)
                evicted.append((victim, vn.slot))
                pch = self._children(vn.parent)
                pch.discard(victim)
                if vn.parent != ROOT_KEY and not pch:
                    self._become_leaf(vn.parent)
            slot = min(self.free_slots)
            self.free_slots.remove(slot)
            if parent != ROOT_KEY and parent in self.leaves:
                self.leaves.remove(parent)     # R2
            self._children(parent).add(key)
            self.nodes[key] = Node(key, parent, tok, slot, PENDING, pins=1)
            self._become_leaf(key)             # R1
            reserved.append(key)
            parent = key

        # 4. pool pages, lowest free first.
        pages = sorted(self.free_pages)[:need_pages]
        self.free_pages.difference_update(pages)
        r.planned, r.matched, r.reserved, r.pages = True, matched, reserved, pages
        n1 = len(matched) * self.C
        return dict(
            n_matched=len(matched), n_reserved=len(reserved), n1=n1, n2=N - n1,
            slots=[self.nodes[k].slot for k in matched + reserved], pages=list(pages),
            evicted=evicted, matched_keys=list(matched), reserved_keys=list(reserved),
        )

    def release(self, req_id: int, commit: bool = True):
        r = self.reqs.get(req_id)
        if r is None:
            raise PlanError("NOREQ", "unknown request")
        if not r.planned:
            raise PlanError("STATE", "request not planned")
        for k in r.matched + r.reserved:
            self.nodes[k].pins -= 1
        if commit:
            for k in r.reserved:
                self.nodes[k].state = RESIDENT
        else:
            for k in reversed(r.reserved):     # deepest first
                n = self.nodes.pop(k)
                self.leaves.remove(k)
                self.free_slots.add(n.slot)
                pch = self._children(n.parent)
                pch.discard(k)
                if n.parent != ROOT_KEY and not pch:
                    self._become_leaf(n.parent)
        self.free_pages.update(r.pages)
        del self.reqs[req_id]

    # ---- inspection ---------------------------------------------------------------
    def resident_keys(self):
        return {k for k, n in self.nodes.items() if n.state == RESIDENT}

    def leaf_list(self):
        return list(self.leaves)
