"""O4 — suffix-query causal attention over prefix + suffix KV, fp64, by definition.
(Oracle: test infrastructure only.)

P:225-231  reusing the KV of an identical prefix and computing only "[doc3:query2]" must
           give what full prefill gives ("exact prefix matching is essential ... to
           preserve the LLM's accuracy"), so the suffix rows of attention over the
           reused+new KV are the suffix rows of ordinary causal attention over the whole
           context: for query head h (kv head g = floor(h / G), R3), suffix row i
           at absolute position p = N1 + i,
               s_j = q_i . k_j / sqrt(d)   for j in [0, p]
               o_i = sum_j exp(s_j - m) v_j / sum_j exp(s_j - m),   m = max_j s_j
               lse_i = m + ln sum_j exp(s_j - m)
Readings: scale 1/sqrt(d), causal over absolute positions, K cached post-RoPE, no
sliding window / softcap / ALiBi (R2).  Inputs are the exact bf16 values.
"""
from __future__ import annotations

import numpy as np


def bf16_bits_to_f64(bits) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint16))
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def suffix_attention(q, k_ctx, v_ctx, n1, rows=None):
    """q [N2][Hq][d], k_ctx/v_ctx [N1+N2][Hkv][d] as float64.  Returns (out, lse) for the
    selected suffix rows (default: all), out [R][Hq][d], lse [R][Hq]."""
    N2, Hq, d = q.shape
    Hkv = k_ctx.shape[1]
    G = Hq // Hkv
    rows = np.arange(N2) if rows is None else np.asarray(rows)
    out = np.empty((len(rows), Hq, d))
    lse = np.empty((len(rows), Hq))
    scale = 1.0 / np.sqrt(d)
    for h in range(Hq):
        g = h // G
        for r, i in enumerate(rows):
            p = n1 + int(i)
            s = (k_ctx[: p + 1, g, :] @ q[i, h, :]) * scale
            m = s.max()
            e = np.exp(s - m)
            out[r, h] = (e @ v_ctx[: p + 1, g, :]) / e.sum()
            lse[r, h] = m + np.log(e.sum())
    return out, lse


def suffix_attention_blocked(q, k_ctx, v_ctx, n1):
    """Same definition, evaluated with one masked matrix product per head (fast enough
    for the L8-sized full check).  Pinned against `suffix_attention` in tests."""
    N2, Hq, d = q.shape
    Hkv = k_ctx.shape[1]
    G = Hq // Hkv
    N = k_ctx.shape[0]
    out = np.empty((N2, Hq, d))
    lse = np.empty((N2, Hq))
    mask = np.arange(N)[None, :] > (n1 + np.arange(N2))[:, None]
    for h in range(Hq):
        g = h // G
        s = (q[:, h, :] @ k_ctx[:, g, :].T) / np.sqrt(d)
        s[mask] = -np.inf
        m = s.max(axis=1, keepdims=True)
        e = np.exp(s - m)
        z = e.sum(axis=1, keepdims=True)
        out[:, h] = (e @ v_ctx[:, g, :]) / z
        lse[:, h] = (m + np.log(z))[:, 0]
    return out, lse


def attention_flops_per_layer(n1, n2, hq_loc, d):
    """Algorithmic flops of one layer (QK^T and PV over the causal triangle), SURVEY §8(d)."""
    return 4 * hq_loc * d * (n2 * n1 + n2 * (n2 + 1) // 2)
