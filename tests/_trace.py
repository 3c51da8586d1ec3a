"""Test-side helpers to replay request traces against a planner (oracle or library)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def replay(planner, reqs, W, commit=True, n_cacheable=None):
    """Submit all requests, then for each i: match_prefix(i, next W ids) -> release(i).
    Returns the list of plans."""
    for i, t in enumerate(reqs):
        planner.submit(i, t, None if n_cacheable is None else n_cacheable[i])
    plans = []
    for i in range(len(reqs)):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
        plans.append(planner.match_prefix(i, pend))
        planner.release(i, commit)
    return plans


def named_chunks(tokens_by_name, C):
    """Map chunk-token bytes -> name like 'A1' for docs split in chunks."""
    out = {}
    for name, toks in tokens_by_name.items():
        for j in range(len(toks) // C):
            out[np.asarray(toks[j * C:(j + 1) * C], dtype="<u4").tobytes()] = f"{name}{j + 1}"
    return out
