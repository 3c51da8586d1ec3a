"""O2' — an independent, brute-force formulation of the look-ahead leaf-LRU planner and
the checks that pin `oracle.tree`.  (Test infrastructure only.)

`StampPlanner` shares no state machinery with `tree.PlanOracle`: instead of an ordered
leaf list it keeps an explicit integer recency stamp per node (stamp := ++clock whenever
a node becomes a leaf or a leaf is touched) and, at every eviction, rescans ALL nodes
for childless, unpinned, RESIDENT ones and takes the minimum stamp.  Chunk identity is
checked by comparing full token paths from the root (no hashing), so it also pins the
hit length to the chunk-granular longest common prefix ("until a mismatch occurs").
"""
from __future__ import annotations

import numpy as np

from .chunks import n_cacheable_chunks


class StampPlanner:
    def __init__(self, C, S_pg, store_chunks, n_pages, window):
        self.C, self.S_pg, self.W = C, S_pg, window
        self.cap, self.n_pages = store_chunks, n_pages
        self.clock = 0
        # node id -> dict(path=tuple of token tuples from root, slot, resident, pins, stamp)
        self.nodes = {}
        self.next_id = 0
        self.used_pages = set()
        self.reqs = {}
        self.audit = []   # (event, node path) for invariant checks

    def _tick(self):
        self.clock += 1
        return self.clock

    def _children_of(self, path):
        return [i for i, n in self.nodes.items() if len(n["path"]) == len(path) + 1 and n["path"][:-1] == path]

    def _find(self, path):
        for i, n in self.nodes.items():
            if n["path"] == path:
                return i
        return None

    def _is_leaf(self, i):
        return not self._children_of(self.nodes[i]["path"])

    def _touch(self, i):
        if self._is_leaf(i):
            self.nodes[i]["stamp"] = self._tick()

    def submit(self, rid, tokens, n_cacheable=None):
        tokens = [int(t) for t in tokens]
        if n_cacheable is None:
            n_cacheable = len(tokens)
        m = n_cacheable_chunks(len(tokens), n_cacheable, self.C)
        chunks = [tuple(tokens[i * self.C:(i + 1) * self.C]) for i in range(m)]
        self.reqs[rid] = dict(tokens=tokens, chunks=chunks)

    def _resident_prefix(self, chunks):
        out = []
        for j in range(len(chunks)):
            i = self._find(tuple(chunks[:j + 1]))
            if i is None or not self.nodes[i]["resident"]:
                break
            out.append(i)
        return out

    def match_prefix(self, rid, pending=()):
        r = self.reqs[rid]
        pend = list(pending)[: self.W]
        N = len(r["tokens"])
        need = -(-N // self.S_pg)
        for p in reversed(pend):
            for i in self._resident_prefix(self.reqs[p]["chunks"]):
                self._touch(i)
        matched = self._resident_prefix(r["chunks"])
        for i in matched:
            self._touch(i)
            self.nodes[i]["pins"] += 1
        reserved, evicted = [], []
        for j in range(len(matched), len(r["chunks"])):
            path = tuple(r["chunks"][:j + 1])
            if self._find(path) is not None:
                break
            used = {n["slot"] for n in self.nodes.values()}
            free = sorted(set(range(self.cap)) - used)
            if not free:
                cands = [i for i in self.nodes if self._is_leaf(i) and self.nodes[i]["pins"] == 0
                         and self.nodes[i]["resident"]]
                if not cands:
                    break
                v = min(cands, key=lambda i: self.nodes[i]["stamp"])
                assert len({self.nodes[i]["stamp"] for i in cands}) == len(cands)  # total order
                assert not self._children_of(self.nodes[v]["path"])   # only leaves removed
                vn = self.nodes.pop(v)
                self.audit.append(("evict", vn["path"]))
                evicted.append((vn["path"], vn["slot"]))
                ppath = vn["path"][:-1]
                if ppath:
                    pi = self._find(ppath)
                    if not self._children_of(ppath):
                        self.nodes[pi]["stamp"] = self._tick()      # parent becomes a leaf
                free = [vn["slot"]]
            slot = free[0]
            nid = self.next_id
            self.next_id += 1
            self.nodes[nid] = dict(path=path, slot=slot, resident=False, pins=1, stamp=self._tick())
            reserved.append(nid)
        used_pages = sorted(self.used_pages)
        pages = sorted(set(range(self.n_pages)) - set(used_pages))[:need]
        self.used_pages.update(pages)
        r.update(matched=matched, reserved=reserved, pages=pages)
        n1 = len(matched) * self.C
        return dict(n_matched=len(matched), n_reserved=len(reserved), n1=n1, n2=N - n1,
                    slots=[self.nodes[i]["slot"] for i in matched + reserved], pages=pages,
                    evicted=evicted)

    def release(self, rid, commit=True):
        r = self.reqs.pop(rid)
        for i in r["matched"] + r["reserved"]:
            self.nodes[i]["pins"] -= 1
        if commit:
            for i in r["reserved"]:
                self.nodes[i]["resident"] = True
        else:
            for i in reversed(r["reserved"]):
                assert not self._children_of(self.nodes[i]["path"])
                n = self.nodes.pop(i)
                self.audit.append(("drop", n["path"]))
                ppath = n["path"][:-1]
                if ppath and not self._children_of(ppath):
                    self.nodes[self._find(ppath)]["stamp"] = self._tick()
        self.used_pages.difference_update(r["pages"])

    # ---- invariants -------------------------------------------------
    def check_invariants(self):
        paths = {n["path"] for n in self.nodes.values()}
        for p in paths:                       # parent-dependency / prefix-closed
            assert len(p) == 1 or p[:-1] in paths
        assert len(self.nodes) <= self.cap    # capacity
        slots = [n["slot"] for n in self.nodes.values()]
        assert len(set(slots)) == len(slots)


def path_of(oracle_tree, key):
    """Token path (tuple of chunk token tuples) of a node of tree.PlanOracle."""
    from .chunks import ROOT_KEY
    out = []
    while key != ROOT_KEY:
        n = oracle_tree.nodes[key]
        out.append(tuple(int(x) for x in np.frombuffer(n.tokens, dtype="<u4")))
        key = n.parent
    return tuple(reversed(out))


def lcp_hit_chunks(resident_paths, tokens, C, cap):
    """Chunk-granular longest common prefix of `tokens` with any resident chain, by direct
    token comparison (the north_star's 'block-granular longest common prefix')."""
    best = 0
    toks = [int(t) for t in tokens]
    for path in resident_paths:
        d = 0
        while d < len(path) and d < cap and list(path[d]) == toks[d * C:(d + 1) * C]:
            d += 1
        best = max(best, d)
    return best
