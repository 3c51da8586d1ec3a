"""Preset Z (BASELINE configs[4]): the 1000-request Zipf trace through the library's host control
(host-only context) and the oracle planner, look-ahead W in {0, 4}: every plan (hits, slots,
pages, evictions in order) must agree bit-exactly; the look-ahead window must not lower the hit
ratio on this popularity-skewed trace."""
import numpy as np
import pytest

from oracle.tree import PlanOracle
from pcrgen import zipf_trace

pcr = pytest.importorskip("paper_2603_23049_b200.pcr")


@pytest.mark.parametrize("W", [0, 4])
def test_zipf_trace_planner_parity(W):
    reqs, _, ndoc = zipf_trace(seed=4)
    C, S, cap = 256, 64, 1188            # store = 10% of the trace's distinct chunks
    n_pages = 4 * (max(len(r) for r in reqs) // S + 1)
    o = PlanOracle(C=C, S_pg=S, store_chunks=cap, n_pages=n_pages, window=W)
    page_bytes = 1 * 1 * 2 * S * 8 * 2
    lib = pcr.Context(1, 1, 1, 8, C, S, cap, W, device=-1, pool_bytes=n_pages * page_bytes,
                      max_tokens=max(len(r) for r in reqs))
    hits = 0
    for i, (t, n) in enumerate(zip(reqs, ndoc)):
        o.submit(i, t, n)
        lib.submit(i, t, n)
    for i in range(len(reqs)):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
        po, pl = o.match_prefix(i, pend), lib.match_prefix(i, pend)
        for f in ("n_matched", "n_reserved", "n1", "n2", "slots", "pages"):
            assert po[f] == pl[f], (i, f)
        assert po["evicted"] == pl["evicted"], i
        hits += po["n_matched"]
        o.release(i, True)
        lib.release(i, True)
    assert o.leaf_list() == lib.leaf_list()
    lib.close()
    total = sum(n // C for n in ndoc)
    ratio = hits / total
    print(f"W={W} chunk hit ratio {ratio:.4f}")
    assert 0.05 < ratio < 0.6
