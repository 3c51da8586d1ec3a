"""O1 — fixed-size chunking and chained chunk keys.  (Oracle: test infrastructure only.)

P:362  "each document is divided into fixed-size chunks ... Chunks sharing identical
        prefixes are mapped to the same tree node ... the KV cache is position-dependent"
Alg.1 P:489-490 Chunkify / HashPrefix(chunk); P:500-501 HashPrefix(chunk, parent).
S:40-67 chunkify/chunk_key contract: full chunks only, root parent = 16 zero bytes.

Reading (R5/R6): key_i = BLAKE2b-128(key_{i-1} || tokens_i as little-endian
uint32), key_{-1} = 16 zero bytes; the number of cacheable chunks of a request is
min(n_cacheable // C, (n_tokens - 1) // C) so that at least one token is always
recomputed (N2 >= 1).
"""
from __future__ import annotations

import hashlib

import numpy as np

ROOT_KEY = bytes(16)


def chunkify(tokens, C: int):
    """Split into full chunks + tail: concat(chunks) + tail == tokens."""
    tokens = np.asarray(tokens, dtype=np.uint32)
    n = len(tokens) // C
    return [tokens[i * C:(i + 1) * C] for i in range(n)], tokens[n * C:]


def chunk_key(parent: bytes, chunk_tokens) -> bytes:
    """HashPrefix(chunk, parent) (Alg.1): BLAKE2b with a 16-byte digest."""
    assert len(parent) == 16
    data = parent + np.asarray(chunk_tokens, dtype="<u4").tobytes()
    return hashlib.blake2b(data, digest_size=16).digest()


def n_cacheable_chunks(n_tokens: int, n_cacheable: int, C: int) -> int:
    """Cacheable full chunks; capped so that N2 = n_tokens - m*C >= 1 (reading R5)."""
    if n_tokens <= 0:
        return 0
    return max(0, min(n_cacheable // C, (n_tokens - 1) // C))


def chain_keys(tokens, C: int, n_cacheable: int | None = None) -> list[bytes]:
    """Keys of the cacheable chunks of a request, root-first (each parented by the previous)."""
    tokens = np.asarray(tokens, dtype=np.uint32)
    if n_cacheable is None:
        n_cacheable = len(tokens)
    m = n_cacheable_chunks(len(tokens), n_cacheable, C)
    keys, parent = [], ROOT_KEY
    for i in range(m):
        parent = chunk_key(parent, tokens[i * C:(i + 1) * C])
        keys.append(parent)
    return keys
