"""f2 on CPU: libpcr's SSD tier (I/O thread + file) vs the tiered oracle — plans, evictions,
on-demand loads and counters bit-exact on random traces; and the data itself survives the
DRAM -> SSD -> DRAM round trip (every matched slot holds the record committed for that chunk)."""
import hashlib

import numpy as np
import pytest

from oracle.tiers import TieredPlanOracle
from pcrgen import make_rng, random_tiny_trace, zipf_trace

pcr = pytest.importorskip("paper_2603_23049_b200.pcr")

L, H, D = 1, 1, 8    # tiny geometry: slot record = L*H*2*C*D*2 bytes


def _ctx(tmp_path, C, S, cap, ssd, W, n_pages=4096, tag="a"):
    page_bytes = L * H * 2 * S * D * 2
    return pcr.Context(L, 1, H, D, C, S, cap, W, device=-1, pool_bytes=n_pages * page_bytes,
                       ssd_path=str(tmp_path / f"ssd_{tag}.bin"), ssd_chunks=ssd, max_inflight=8)


def _record(key: bytes, nbytes: int) -> np.ndarray:
    """Deterministic per-chunk payload (what 'offload' would have written for that chunk)."""
    seed = int.from_bytes(hashlib.blake2b(key, digest_size=8).digest(), "little")
    return make_rng(seed).integers(0, 1 << 16, nbytes // 2, dtype=np.uint16)


def _run(tmp_path, reqs, C, S, cap, ssd, W, commit_pattern=None, tag="a", n_cacheable=None):
    o = TieredPlanOracle(C=C, S_pg=S, store_chunks=cap, n_pages=4096, window=W, ssd_chunks=ssd)
    lib = _ctx(tmp_path, C, S, cap, ssd, W, tag=tag)
    nb = lib.slot_bytes
    for i, t in enumerate(reqs):
        nc = None if n_cacheable is None else n_cacheable[i]
        o.submit(i, t, nc)
        lib.submit(i, t, nc)
    for i in range(len(reqs)):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W + 1)))
        po, pl = o.match_prefix(i, pend), lib.match_prefix(i, pend)
        for f in ("n_matched", "n_reserved", "n1", "n2", "slots", "pages", "n_from_ssd"):
            assert po[f] == pl[f], (i, f, po[f], pl[f])
        assert po["evicted"] == pl["evicted"], i
        # data: every matched chunk's DRAM slot holds exactly the record committed for its key
        for key, slot in zip(po["matched_keys"], po["slots"]):
            assert np.array_equal(lib.store_read(slot), _record(key, nb)), (i, slot)
        # "offload": write the new chunks' records before committing
        for key, slot in zip(po["reserved_keys"], po["slots"][po["n_matched"]:]):
            lib.store_write(slot, _record(key, nb))
        commit = True if commit_pattern is None else bool(commit_pattern[i % len(commit_pattern)])
        o.release(i, commit)
        lib.release(i, commit)
        assert o.leaf_list() == lib.leaf_list()
    st = lib.stats
    assert (st["prefetch_loads"], st["ondemand_loads"], st["writebacks"], st["ssd_evictions"],
            st["dram_evictions"]) == (o.stats["prefetch"], o.stats["ondemand"], o.stats["writeback"],
                                      o.stats["ssd_evict"], o.stats["dram_evict"])
    lib.close()
    return o.stats


def test_random_traces_with_ssd_tier(tmp_path):
    rng = make_rng(77)
    loads = 0
    for case in range(60):
        C = int(rng.integers(2, 5))
        reqs = random_tiny_trace(rng, C=C, n_docs=6, max_doc_chunks=3, n_requests=14)
        st = _run(tmp_path, reqs, C, C, int(rng.integers(3, 12)), int(rng.integers(0, 30)),
                  int(rng.integers(0, 4)), [None, [1, 1, 0]][case % 2], tag=str(case))
        loads += st["prefetch"] + st["ondemand"]
    assert loads > 50      # the traces really exercise the SSD path


def test_zipf_trace_with_ssd_tier(tmp_path):
    """Preset Z's first 300 requests with a 3% DRAM store and a 25% SSD (f2 capacity setting)."""
    reqs, _, ndoc = zipf_trace(seed=4, n_requests=300, C=256)
    st = _run(tmp_path, reqs, 256, 64, 120, 1000, 4, tag="z", n_cacheable=ndoc)
    assert st["prefetch"] > 0 and st["writeback"] > 0


def test_ssd_file_lifecycle(tmp_path):
    """pcr_create creates the tier file (sized for ssd_chunks records); pcr_destroy removes it."""
    lib = _ctx(tmp_path, 4, 4, 4, 16, 0, tag="life")
    f = tmp_path / "ssd_life.bin"
    assert f.exists() and f.stat().st_size == 16 * lib.slot_bytes
    lib.close()
    assert not f.exists()
