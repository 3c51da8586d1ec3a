"""O2 pins: the paper's printed eviction example, brute-force agreement on random
tiny traces, invariants, hit length = chunk-granular LCP, error model."""
import numpy as np
import pytest

from oracle.brute import StampPlanner, lcp_hit_chunks, path_of
from oracle.chunks import chain_keys
from oracle.tree import RESIDENT, PlanError, PlanOracle
from pcrgen import appendix_c_trace, make_rng, random_tiny_trace
from tests._trace import load_golden, named_chunks, replay

C4 = 4  # chunk tokens for the tiny fixtures


def _fig_tokens():
    return {f"C{i}": np.full(C4, 100 + i, dtype=np.uint32) for i in range(1, 10)}


def _req(chunks, toks, q=7):
    return np.concatenate([toks[c] for c in chunks] + [np.array([q], dtype=np.uint32)])


def _fig_setup():
    g = load_golden("appendix_a_fig_prefixcache.json")
    toks = _fig_tokens()
    t = PlanOracle(C=C4, S_pg=4, store_chunks=g["capacity_chunks"], n_pages=64, window=4)
    for i, chunks in enumerate(g["commit_order"]):
        t.submit(100 + i, _req(chunks, toks))
        t.match_prefix(100 + i, [])
        t.release(100 + i, True)
    names = {}
    for chunks in g["commit_order"] + [g["current_request"]]:
        for k, n in zip(chain_keys(_req(chunks, toks), C4), chunks):
            names[k] = n
    return g, toks, t, names


def test_fig_prefixcache_initial_leaves():
    g, toks, t, names = _fig_setup()
    assert [names[k] for k in t.leaf_list()] == g["leaves_before"]   # C2 oldest, C4 second


@pytest.mark.parametrize("lookahead", [True, False])
def test_fig_prefixcache_eviction(lookahead):
    g, toks, t, names = _fig_setup()
    t.submit(1, _req(g["current_request"], toks))
    t.submit(2, _req(g["pending_request"], toks, q=9))
    plan = t.match_prefix(1, [2] if lookahead else [])
    assert [names[k] for k in plan["matched_keys"]] == g["matched"]          # C7, C8
    assert plan["n_matched"] == 2 and plan["n_reserved"] == 1
    assert len(plan["evicted"]) == 1
    victim = names[plan["evicted"][0][0]]
    leaves = [names[k] for k in t.leaf_list()]
    if lookahead:
        assert victim == g["with_lookahead"]["victim"]                     # C4
        assert leaves == g["with_lookahead"]["leaves_after"]               # [C6, C2, C3, C9]
    else:
        assert victim == g["without_lookahead"]["victim"]                  # C2
        assert set(leaves) == set(g["without_lookahead"]["leaves_after_set"])
    # C9 inserted as a child of C8
    c9 = plan["reserved_keys"][0]
    assert names[t.nodes[c9].parent] == "C8"


@pytest.mark.parametrize("W", [0, 2])
def test_appendix_c_trace(W):
    g = load_golden("appendix_c_trace_T.json")
    docs, order, reqs = appendix_c_trace(0)
    t = PlanOracle(C=g["C"], S_pg=g["S_pg"], store_chunks=g["store_chunks"], n_pages=1024, window=W)
    names = named_chunks(docs, g["C"])
    for i, r in enumerate(reqs):
        t.submit(i, r)
    hits, evs = [], []
    for i in range(len(reqs)):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
        # record every chain path we may later see evicted
        paths = {}
        for k in t.nodes:
            paths[k] = "/".join(names[c] for c in
                                [np.asarray(x, dtype="<u4").tobytes() for x in path_of(t, k)])
        plan = t.match_prefix(i, pend)
        hits.append(plan["n_matched"])
        evs.append([paths[k] for k, _ in plan["evicted"]])
        t.release(i, True)
    exp = g[f"W{W}"]
    assert hits == exp["hits"]
    assert evs == exp["evictions"]


def _compare_planners(reqs, C, cap, W, commit_pattern=None):
    a = PlanOracle(C=C, S_pg=2, store_chunks=cap, n_pages=4096, window=W)
    b = StampPlanner(C, 2, cap, 4096, W)
    for i, t in enumerate(reqs):
        a.submit(i, t)
        b.submit(i, t)
    for i in range(len(reqs)):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
        resident_paths = [path_of(a, k) for k in a.resident_keys()]
        pa = a.match_prefix(i, pend)
        pb = b.match_prefix(i, pend)
        # hit length == chunk-granular LCP against committed resident chains
        cap_chunks = len(a.reqs[i].keys)
        assert pa["n_matched"] == lcp_hit_chunks(resident_paths, reqs[i], C, cap_chunks)
        for f in ("n_matched", "n_reserved", "n1", "n2", "slots", "pages"):
            assert pa[f] == pb[f], (i, f, pa[f], pb[f])
        assert [s for _, s in pa["evicted"]] == [s for _, s in pb["evicted"]]
        commit = True if commit_pattern is None else bool(commit_pattern[i % len(commit_pattern)])
        a.release(i, commit)
        b.release(i, commit)
        b.check_invariants()
        # list-policy invariants: the leaf list is exactly the childless nodes
        assert set(a.leaves) == {k for k, n in a.nodes.items() if not n.children}
        assert len(a.nodes) <= cap
    # StampPlanner asserts at every removal that the node is childless (S:151 leaf-only)


def test_bruteforce_random_traces():
    """S:156 + SURVEY App. A: incremental list policy == stamp argmin on seeded random traces
    (5 docs of 1-3 chunks, 1-3 docs per request, capacity 2-7 chunks, W in [0,3])."""
    rng = make_rng(1234)
    for case in range(600):
        C = int(rng.integers(1, 4))
        reqs = random_tiny_trace(rng, C=C, n_docs=5, max_doc_chunks=3, n_requests=10)
        cap = int(rng.integers(2, 8))
        W = int(rng.integers(0, 4))
        pattern = None if case % 3 else [1, 1, 0]
        _compare_planners(reqs, C, cap, W, pattern)


def test_bruteforce_tiny_exhaustive():
    """<= 8-node trees: the victim equals the argmin over an explicit enumeration of
    every candidate."""
    rng = make_rng(99)
    for _ in range(300):
        reqs = random_tiny_trace(rng, C=2, n_docs=4, max_doc_chunks=2, n_requests=8, max_docs_per_req=2)
        _compare_planners(reqs, 2, int(rng.integers(2, 9)), int(rng.integers(0, 3)))


def test_lookahead_protects_window():
    """With W>0 a chunk of the next request is not evicted while an untouched leaf exists."""
    rng = make_rng(7)
    C = 2
    docs = [rng.integers(0, 1000, n * C, dtype=np.uint32) for n in (2, 2, 1)]
    q = lambda: rng.integers(0, 1000, 1, dtype=np.uint32)  # noqa: E731
    reqs = [np.concatenate([docs[0], q()]), np.concatenate([docs[1], q()]),
            np.concatenate([docs[2], q()]), np.concatenate([docs[0], q()])]
    for W, expect_hit in ((0, 1), (1, 2)):
        t = PlanOracle(C=C, S_pg=2, store_chunks=4, n_pages=64, window=W)
        plans = replay(t, reqs, W)
        # request 2 needs one eviction: plain LRU takes doc0's last chunk (the oldest leaf);
        # with request 3 in request 2's window, doc0's chain is bumped and doc1's leaf goes
        assert plans[3]["n_matched"] == expect_hit


def test_errors_and_strong_guarantee():
    t = PlanOracle(C=4, S_pg=4, store_chunks=4, n_pages=3, window=2)
    toks = np.arange(9, dtype=np.uint32)
    with pytest.raises(PlanError) as e:
        t.match_prefix(5, [])
    assert e.value.code == "NOREQ"
    t.submit(0, toks)
    with pytest.raises(PlanError) as e:
        t.submit(0, toks)
    assert e.value.code == "STATE"
    with pytest.raises(PlanError) as e:
        t.submit(1, toks, n_cacheable=10)
    assert e.value.code == "INVAL"
    with pytest.raises(PlanError) as e:
        t.match_prefix(0, [0])
    assert e.value.code == "INVAL"
    t.submit(1, toks)
    with pytest.raises(PlanError) as e:
        t.match_prefix(0, [1, 1])
    assert e.value.code == "INVAL"
    with pytest.raises(PlanError) as e:
        t.match_prefix(0, [7])
    assert e.value.code == "NOREQ"
    with pytest.raises(PlanError) as e:
        t.release(0, True)
    assert e.value.code == "STATE"
    big = np.arange(13, dtype=np.uint32)   # needs 4 pages of 4 tokens, pool has 3
    t.submit(2, big)
    snap = (dict(t.nodes), list(t.leaves), set(t.free_slots), set(t.free_pages))
    with pytest.raises(PlanError) as e:
        t.match_prefix(2, [0, 1])
    assert e.value.code == "NOMEM"
    assert snap == (dict(t.nodes), list(t.leaves), set(t.free_slots), set(t.free_pages))
    # extras beyond the window are ignored, not an error
    p = t.match_prefix(0, [1, 2, 99])
    assert p["n1"] + p["n2"] == 9 and p["n2"] >= 1


def test_abort_drops_pending_chain():
    t = PlanOracle(C=2, S_pg=2, store_chunks=8, n_pages=16, window=0)
    a = np.arange(7, dtype=np.uint32)
    t.submit(0, a)
    p = t.match_prefix(0, [])
    assert p["n_matched"] == 0 and p["n_reserved"] == 3
    t.release(0, commit=False)
    assert t.nodes == {} and t.leaves == [] and len(t.free_slots) == 8 and len(t.free_pages) == 16
    t.submit(1, a)
    p = t.match_prefix(1, [])
    t.release(1, True)
    t.submit(2, a)
    p = t.match_prefix(2, [])
    assert p["n_matched"] == 3 and p["n2"] == 1
    assert all(n.state == RESIDENT for n in t.nodes.values())


def test_pending_chunks_not_matchable():
    """Reading R10: a reserved (PENDING) chunk is not a hit for a concurrent request."""
    t = PlanOracle(C=2, S_pg=2, store_chunks=8, n_pages=32, window=0)
    a = np.arange(7, dtype=np.uint32)
    t.submit(0, a)
    t.submit(1, a)
    p0 = t.match_prefix(0, [])
    p1 = t.match_prefix(1, [])
    assert p0["n_reserved"] == 3 and p1["n_matched"] == 0 and p1["n_reserved"] == 0
    assert set(p0["pages"]).isdisjoint(p1["pages"])
