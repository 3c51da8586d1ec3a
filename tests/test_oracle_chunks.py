"""O1 pins: chunking (S:42-49 examples) and the position-dependence of chunk keys."""
import numpy as np
from hypothesis import given, settings, strategies as st

from oracle.chunks import ROOT_KEY, chain_keys, chunk_key, chunkify, n_cacheable_chunks


def test_chunkify_examples_spec():
    # 600 tokens at C=256 -> 2 chunks + 88-token tail; empty; exact multiple.
    ch, tail = chunkify(np.arange(600), 256)
    assert len(ch) == 2 and len(tail) == 88
    ch, tail = chunkify([], 256)
    assert ch == [] and len(tail) == 0
    ch, tail = chunkify(np.arange(256), 256)
    assert len(ch) == 1 and len(tail) == 0


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 4 * 8), st.integers(1, 8))
def test_chunkify_roundtrip(n, C):
    toks = np.arange(n, dtype=np.uint32) * 7 + 3
    ch, tail = chunkify(toks, C)
    assert all(len(c) == C for c in ch) and len(tail) < C
    assert np.array_equal(np.concatenate(ch + [tail]) if ch else tail, toks)


def test_key_position_dependence():
    """equal chunk tokens under different prefixes are different nodes (C6 vs C8);
    equal prefixes map to the same node (C1 shared by D1 and D2)."""
    rng = np.random.default_rng(0)
    a, b, x = (rng.integers(0, 1000, 16, dtype=np.uint32) for _ in range(3))
    k_ax = chain_keys(np.concatenate([a, x, [1]]), 16)
    k_bx = chain_keys(np.concatenate([b, x, [1]]), 16)
    k_ab = chain_keys(np.concatenate([a, b, [1]]), 16)
    assert k_ax[0] == k_ab[0]            # shared first chunk -> same key
    assert k_ax[1] != k_bx[1]            # same tokens, different parent -> different key
    assert k_ax[0] != k_bx[0]


def test_key_chain_structure():
    """k*C tokens yield k keys, chunk i parented by chunk i-1; a single changed token
    changes its own key and every later key, never an earlier one."""
    rng = np.random.default_rng(1)
    toks = rng.integers(0, 1 << 32, 5 * 8 + 1, dtype=np.uint64).astype(np.uint32)
    keys = chain_keys(toks, 8)
    assert len(keys) == 5
    parent = ROOT_KEY
    for i, k in enumerate(keys):
        assert k == chunk_key(parent, toks[i * 8:(i + 1) * 8])
        parent = k
    for pos in (0, 13, 39):
        t2 = toks.copy()
        t2[pos] ^= 1
        k2 = chain_keys(t2, 8)
        c = pos // 8
        assert k2[:c] == keys[:c]
        assert all(k2[j] != keys[j] for j in range(c, 5))


def test_keys_distinct_bruteforce():
    """no digest collisions over 1000 random (parent, tokens) pairs."""
    rng = np.random.default_rng(2)
    seen = set()
    for _ in range(1000):
        parent = bytes(rng.integers(0, 256, 16, dtype=np.uint8))
        seen.add(chunk_key(parent, rng.integers(0, 50, 4, dtype=np.uint32)))
    assert len(seen) == 1000


def test_cacheable_cap():
    """Reading R5: at least one token is always recomputed (N2 >= 1)."""
    assert n_cacheable_chunks(320, 320, 64) == 4      # floor(319/64)
    assert n_cacheable_chunks(256, 256, 64) == 3      # exact multiple leaves the last chunk
    assert n_cacheable_chunks(4224, 4224, 256) == 16  # L8: 4096 cached + 128 query
    assert n_cacheable_chunks(4224, 4096, 256) == 16
    assert n_cacheable_chunks(4224, 1000, 256) == 3
    assert n_cacheable_chunks(1, 1, 1) == 0
    assert n_cacheable_chunks(0, 0, 4) == 0
