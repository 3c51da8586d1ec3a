"""f2 oracle pins: the paper's prefetch example (fig:prefetch), equivalence with the pinned
DRAM-only planner when the SSD tier is empty, hit length = chunk-LCP over chains available in
DRAM or on SSD, and "never prefetch what is already in DRAM"."""
import numpy as np

from oracle.brute import lcp_hit_chunks, path_of
from oracle.tiers import LOADING, TieredPlanOracle
from oracle.tree import RESIDENT, PlanOracle
from pcrgen import make_rng, random_tiny_trace

C = 4


def _doc(rng, n):
    return rng.integers(0, 1000, n * C, dtype=np.uint32)


def _req(*parts, rng):
    return np.concatenate(list(parts) + [rng.integers(0, 1000, 1, dtype=np.uint32)])


def test_prefetch_example_fig_prefetch():
    """R1's KV in DRAM -> no action; R2 and R4 on SSD -> asynchronous loads; R3 in neither
    -> recomputed.  With the window, R2 and R4 later hit entirely from DRAM (no on-demand SSD
    load); without it they pay on-demand loads."""
    for W in (4, 0):
        rng = make_rng(3)
        d1, d2, d3, d4 = _doc(rng, 2), _doc(rng, 1), _doc(rng, 2), _doc(rng, 1)
        filler, filler2 = _doc(rng, 6), _doc(rng, 2)
        t = TieredPlanOracle(C=C, S_pg=C, store_chunks=8, n_pages=256, window=W, ssd_chunks=16)
        # history: R2's and R4's docs were computed (DRAM + SSD write-back), then pushed out of
        # DRAM by later requests; R1's doc computed last (in DRAM); R3's doc never seen.
        hist = [_req(d2, rng=rng), _req(d4, rng=rng), _req(filler, rng=rng), _req(filler2, rng=rng),
                _req(d1, rng=rng)]
        for i, h in enumerate(hist):
            t.submit(100 + i, h)
            t.match_prefix(100 + i, [])
            t.release(100 + i, True)
        r0, r1, r2, r3, r4 = (_req(x, rng=rng) for x in (filler[:C], d1, d2, d3, d4))
        for i, x in enumerate((r0, r1, r2, r3, r4)):
            t.submit(i, x)
        assert t.stats["prefetch"] == 0
        t.match_prefix(0, [1, 2, 3, 4])
        if W:
            assert t.stats["prefetch"] == 2            # R2 (1 chunk) and R4 (1 chunk)
            loaded = t.loads[0]
            assert len(loaded) == 2 and all(t.nodes[k].state == LOADING for k in loaded)
        t.release(0, True)
        total_ondemand = 0
        for i, x in enumerate((r1, r2, r3, r4), start=1):
            p = t.match_prefix(i, list(range(i + 1, 5)))
            total_ondemand += p["n_from_ssd"]
            if i == 3:
                assert p["n_matched"] == 0               # R3: recompute
            else:
                assert p["n_matched"] == len(t.reqs[i].keys)
            t.release(i, True)
        assert total_ondemand == (0 if W else 2)


def test_empty_ssd_equals_dram_only_planner():
    rng = make_rng(8)
    for _ in range(120):
        reqs = random_tiny_trace(rng, C=2, n_docs=5, max_doc_chunks=3, n_requests=10)
        cap, W = int(rng.integers(2, 8)), int(rng.integers(0, 4))
        a = PlanOracle(C=2, S_pg=2, store_chunks=cap, n_pages=4096, window=W)
        b = TieredPlanOracle(C=2, S_pg=2, store_chunks=cap, n_pages=4096, window=W, ssd_chunks=0)
        for i, t in enumerate(reqs):
            a.submit(i, t)
            b.submit(i, t)
        for i in range(len(reqs)):
            pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
            pa, pb = a.match_prefix(i, pend), b.match_prefix(i, pend)
            for f in ("n_matched", "n_reserved", "n1", "n2", "slots", "pages", "evicted"):
                assert pa[f] == pb[f]
            a.release(i, i % 3 != 2)
            b.release(i, i % 3 != 2)
            assert a.leaf_list() == b.leaf_list()


def _available_paths(t):
    """Token paths of every chunk retrievable from DRAM (RESIDENT) or the SSD index."""
    paths = {path_of(t, k) for k, n in t.nodes.items() if n.state == RESIDENT}
    by_key = dict(t.ssd)

    def ssd_path(k, depth=0):
        if k in t.nodes and t.nodes[k].state == RESIDENT:
            return path_of(t, k)
        if k not in by_key or depth > 64:
            return None
        _, parent, tok = by_key[k]
        pre = () if parent == bytes(16) else ssd_path(parent, depth + 1)
        if pre is None:
            return None
        return pre + (tuple(int(x) for x in np.frombuffer(tok, dtype="<u4")),)

    for k in by_key:
        p = ssd_path(k)
        if p is not None:
            paths.add(p)
    return paths


def test_hit_length_is_lcp_over_dram_and_ssd_and_no_redundant_prefetch():
    rng = make_rng(21)
    for case in range(150):
        reqs = random_tiny_trace(rng, C=2, n_docs=6, max_doc_chunks=3, n_requests=14)
        W = int(rng.integers(0, 4))
        # DRAM large enough for one request's chain plus the window's loads: no starvation
        t = TieredPlanOracle(C=2, S_pg=2, store_chunks=int(rng.integers(26, 32)), n_pages=4096, window=W,
                             ssd_chunks=int(rng.integers(2, 40)))
        for i, x in enumerate(reqs):
            t.submit(i, x)
        for i in range(len(reqs)):
            pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
            avail = _available_paths(t)
            in_dram_before = {k for k, n in t.nodes.items() if n.state == RESIDENT}
            before = t.stats["prefetch"]
            p = t.match_prefix(i, pend)
            cap = len(t.reqs[i].keys)
            assert p["n_matched"] == lcp_hit_chunks(avail, reqs[i], 2, cap), case
            evicted_now = {k for k, _ in p["evicted"]}
            for k in t.loads.get(i, []):                 # never prefetch what is in DRAM: a load of a
                assert k not in in_dram_before or k in evicted_now   # chunk in DRAM before the call
                # is only possible if this same call evicted it first (window thrash)
            assert t.stats["prefetch"] >= before
            t.release(i, True)
            assert len(t.ssd) <= t.ssd_cap and len(t.nodes) <= t.store_chunks
