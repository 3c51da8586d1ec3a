"""O3 — per-layer KV load from the DRAM chunk store into the paged pool, and the suffix
append.  (Oracle: test infrastructure only.)

P:478  vLLM "partitions each sequence's KV cache into small blocks ... mapping several
       non-consecutive small physical blocks to a large, virtually consecutive KV cache
       block"; "the KV cache is allocated layer by layer ... so we can do layer-wise
       memory copying".
P:480  "copy KV cache from a CPU chunk to multiple non-consecutive GPU memory blocks"
       (chunk 256 tokens vs block 16).
P:227  "the KV cache is generated layer by layer" -> the N2 new tokens' K/V are written
       after the prefix.

Layouts (include/pcr.h): store  [slot][L][Hkv_loc][2][C][d]      (2 = K, V)
                         pool   [L][page][Hkv_loc][2][S_pg][d]
Logical token t of the request lives at pool[l, pages[t // S_pg], :, :, t % S_pg, :].
All arrays hold bf16 bit patterns (uint16); the operation is a bit copy.
"""
from __future__ import annotations

import numpy as np


def load_layer(pool, store, slots, pages, layer, n1, C, S_pg):
    """pool[l][pages[t//S_pg]][h][kv][t%S_pg] = store[slots[t//C]][l][h][kv][t%C], t < N1."""
    for t in range(n1):
        pool[layer, pages[t // S_pg], :, :, t % S_pg, :] = store[slots[t // C], layer, :, :, t % C, :]


def append_layer(pool, k_new, v_new, pages, layer, n1, S_pg):
    """Suffix token i (absolute position N1+i): k_new/v_new are [N2][Hkv_loc][d]."""
    for i in range(k_new.shape[0]):
        t = n1 + i
        pool[layer, pages[t // S_pg], :, 0, t % S_pg, :] = k_new[i]
        pool[layer, pages[t // S_pg], :, 1, t % S_pg, :] = v_new[i]


def logical_kv(pool, pages, layer, n_tokens, S_pg):
    """Read back the logical K, V sequence [N][Hkv_loc][d] of one layer from the pool."""
    H, d = pool.shape[2], pool.shape[5]
    k = np.empty((n_tokens, H, d), dtype=pool.dtype)
    v = np.empty((n_tokens, H, d), dtype=pool.dtype)
    for t in range(n_tokens):
        k[t] = pool[layer, pages[t // S_pg], :, 0, t % S_pg, :]
        v[t] = pool[layer, pages[t // S_pg], :, 1, t % S_pg, :]
    return k, v


def load_bytes_per_layer(n1, hkv_loc, d, elem_bytes=2):
    """Algorithmic bytes moved host->HBM per layer: K and V of N1 tokens."""
    return 2 * n1 * hkv_loc * d * elem_bytes
