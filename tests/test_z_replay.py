"""Preset Z oracle replay: every pass of the GPU Z-trace sweep
(`bench.py --workload Z --z-windows ... --z-store-fracs ... --rho ... --z-log DIR`) logged each
pcr_match_prefix input -- the request and the pending ids of its look-ahead window, which under
Poisson arrivals depend on the measured service times -- with the library's decisions.  Here the
fp64-free oracle planner (oracle/tree.py, oracle/tiers.py with an SSD tier) replays those inputs
on the same regenerated trace and must reach the same decisions bit for bit: hits, reserved
chunks, store slots in chain order, the slots freed by evictions in order, and SSD on-demand
loads.  The logs are committed under tests/golden/z_plans/ (written on the B200 by the bench; no
value in them comes from the oracle)."""
import glob
import gzip
import json
import os

import pytest

from oracle.tiers import TieredPlanOracle
from oracle.tree import PlanOracle
from pcrgen import zipf_trace

HERE = os.path.dirname(os.path.abspath(__file__))
LOGS = sorted(glob.glob(os.path.join(HERE, "golden", os.environ.get("PCR_Z_PLANS", "z_plans"), "*.jsonl.gz")))


def _read(path):
    with gzip.open(path, "rt") as f:
        lines = [json.loads(ln) for ln in f]
    return lines[0], lines[1:]


def test_logs_are_present():
    assert LOGS, "no committed Z plan logs under tests/golden/z_plans/"


@pytest.mark.parametrize("path", LOGS, ids=[os.path.basename(p)[:-9] for p in LOGS])
def test_replay_matches_the_gpu_run(path):
    h, recs = _read(path)
    reqs, _, ndoc = zipf_trace(seed=4, n_requests=h["requests"], C=h["C"])
    assert len(recs) == h["requests"]
    kw = dict(C=h["C"], S_pg=h["S_pg"], store_chunks=h["store_chunks"], n_pages=h["n_pool_pages"],
              window=h["window"])
    o = TieredPlanOracle(ssd_chunks=h["ssd_chunks"], **kw) if h["ssd_chunks"] else PlanOracle(**kw)
    for i, (t, n) in enumerate(zip(reqs, ndoc)):
        o.submit(i, t, 0 if h["no_reuse"] else n)
    hits = 0
    for rec in recs:
        i = rec["i"]
        assert len(rec["pend"]) <= h["window"]
        po = o.match_prefix(i, rec["pend"])
        got = (po["n_matched"], po["n_reserved"], po["slots"], [s for _, s in po["evicted"]],
               po.get("n_from_ssd", 0))
        assert got == (rec["nm"], rec["nr"], rec["slots"], rec["ev"], rec["ssd"]), (os.path.basename(path), i)
        hits += po["n_matched"]
        o.release(i, True)
    if h["pass"] == "poisson":
        # the windows really came from the arrival process: not all full, not all empty
        sizes = {len(r["pend"]) for r in recs}
        assert len(sizes) > 1 or h["window"] == 0
    print(f"{os.path.basename(path)}: {len(recs)} plans replayed, {hits} chunk hits")
