"""Seeded synthetic workloads with the shapes of the paper's RAG requests.

Only random draws and array packing live here (see package docstring).  Every
generator takes an explicit seed; the recipe per preset is documented in
DESIGN.md §"Input recipe" and SURVEY.md §8(d).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "PRESETS", "make_rng", "f32_to_bf16_bits", "randn_bf16", "doc_tokens",
    "appendix_c_trace", "rag_request_tokens", "stress_values", "pack_store_slots",
    "random_tiny_trace", "l8_request", "hit_ratio_request", "zipf_trace",
]

# Model geometry per preset (BASELINE.json configs[0..3]).
# C = chunk tokens (paper: 256), S_pg = pool page tokens (paper's vLLM block = 16).
PRESETS = {
    "T": dict(L=2, Hq=4, Hkv=2, d=64, C=64, S_pg=16),      # configs[0]
    "L8": dict(L=32, Hq=32, Hkv=8, d=128, C=256, S_pg=64),  # configs[1]  Llama-3-8B shape
    "M7": dict(L=32, Hq=32, Hkv=8, d=128, C=256, S_pg=64),  # configs[2]  Mistral-7B shape
    "L70": dict(L=80, Hq=64, Hkv=8, d=128, C=256, S_pg=64),  # configs[3]  Llama-3-70B shape
}

VOCAB = 128256  # Llama-3 vocabulary size; token ids only need to fit in 32 bits.


def make_rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def f32_to_bf16_bits(x) -> np.ndarray:
    """Round fp32 -> bf16 (round-to-nearest-even), returned as uint16 bit patterns."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    bias = ((u >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)
    return ((u + bias) >> np.uint64(16)).astype(np.uint16)


def randn_bf16(rng: np.random.Generator, shape, scale: float = 1.0) -> np.ndarray:
    return f32_to_bf16_bits(rng.standard_normal(shape, dtype=np.float32) * np.float32(scale))


def doc_tokens(rng: np.random.Generator, n_docs: int, doc_len: int) -> list[np.ndarray]:
    return [rng.integers(0, VOCAB, size=doc_len, dtype=np.uint32) for _ in range(n_docs)]


def rag_request_tokens(docs, query_len: int, rng: np.random.Generator) -> np.ndarray:
    """[doc_a : doc_b : ... : query] as in the paper's RAG prompt (§2.1)."""
    q = rng.integers(0, VOCAB, size=query_len, dtype=np.uint32)
    return np.concatenate(list(docs) + [q]).astype(np.uint32)


def appendix_c_trace(seed: int = 0):
    """SURVEY Appendix C canonical preset-T trace: docs A..D (128 tokens = 2 chunks of
    C=64), requests [docX, docY] + 64-token query, in the order AB AB AC CA BA AB CA DB."""
    rng = make_rng(seed)
    docs = dict(zip("ABCD", doc_tokens(rng, 4, 128)))
    order = ["AB", "AB", "AC", "CA", "BA", "AB", "CA", "DB"]
    reqs = [rag_request_tokens([docs[a], docs[b]], 64, rng) for a, b in order]
    return docs, order, reqs


def l8_request(seed: int = 1, n_docs: int = 4, doc_len: int = 1024, query_len: int = 128):
    """configs[1]: 4 docs x 1k cached prefix + 128-token query."""
    rng = make_rng(seed)
    docs = doc_tokens(rng, n_docs, doc_len)
    return docs, rag_request_tokens(docs, query_len, rng)


def hit_ratio_request(seed: int, doc_tokens_total: int, query_len: int, C: int, ratio: float):
    """configs[2]: a request whose first round(ratio * doc_chunks) chunks are cached.
    Returns (warm_tokens, request_tokens): committing `warm_tokens` first makes exactly
    that many leading chunks resident (the warm request diverges right after them)."""
    rng = make_rng(seed)
    doc = rng.integers(0, VOCAB, size=doc_tokens_total, dtype=np.uint32)
    req = np.concatenate([doc, rng.integers(0, VOCAB, size=query_len, dtype=np.uint32)])
    n_hit = int(round(ratio * (doc_tokens_total // C)))
    warm = req.copy()
    warm[n_hit * C:] = rng.integers(0, VOCAB, size=len(req) - n_hit * C, dtype=np.uint32)
    return warm, req


def stress_values(kind: str, seed: int, N1: int, N2: int, Hq: int, Hkv: int, d: int):
    """Q [N2][Hq][d], K/V context [N1+N2][Hkv][d] as bf16 bits.

    kinds (SURVEY §8(c) O4 sensitivity): 'iid' N(0,1); 'q4' Q x 4; 'kout' four K
    outlier channels x 8; 'advfuture' k[N1+i+1] aligned with q[i] at norm 2*sqrt(d)
    so any key leaking past the causal boundary of row i dominates that row.
    """
    rng = make_rng(seed)
    N = N1 + N2
    q = rng.standard_normal((N2, Hq, d), dtype=np.float32)
    k = rng.standard_normal((N, Hkv, d), dtype=np.float32)
    v = rng.standard_normal((N, Hkv, d), dtype=np.float32)
    if kind == "iid":
        pass
    elif kind == "q4":
        q *= 4
    elif kind == "kout":
        ch = rng.choice(d, size=4, replace=False)
        k[:, :, ch] *= 8
    elif kind == "advfuture":
        G = Hq // Hkv
        for i in range(N2 - 1):
            for g in range(Hkv):
                qi = q[i, g * G]
                k[N1 + i + 1, g] = qi / np.linalg.norm(qi) * (2.0 * np.sqrt(d))
    else:
        raise ValueError(kind)
    return f32_to_bf16_bits(q), f32_to_bf16_bits(k), f32_to_bf16_bits(v)


def pack_store_slots(k_ctx: np.ndarray, v_ctx: np.ndarray, n_chunks: int, C: int) -> np.ndarray:
    """Pack per-layer context K/V into DRAM-store chunk records.

    k_ctx, v_ctx: [L][N][Hkv_loc][d] (uint16 bf16 bits).  Returns
    [n_chunks][L][Hkv_loc][2][C][d]: the store-slot layout of include/pcr.h
    (one record = one chunk x all layers, "chunk ... 256 tokens").
    """
    L, N, H, d = k_ctx.shape
    out = np.empty((n_chunks, L, H, 2, C, d), dtype=np.uint16)
    for c in range(n_chunks):
        sl = slice(c * C, (c + 1) * C)
        out[c, :, :, 0] = k_ctx[:, sl].transpose(0, 2, 1, 3)
        out[c, :, :, 1] = v_ctx[:, sl].transpose(0, 2, 1, 3)
    return out


def random_tiny_trace(rng: np.random.Generator, C: int = 4, n_docs: int = 5,
                      max_doc_chunks: int = 3, n_requests: int = 12, max_docs_per_req: int = 3,
                      query_len=(1, 6)):
    """Tiny request traces for the brute-force eviction checks:
    docs of 1..max_doc_chunks chunks, 1..max_docs_per_req docs per request, short queries."""
    docs = [rng.integers(0, 50, size=C * int(rng.integers(1, max_doc_chunks + 1)), dtype=np.uint32)
            for _ in range(n_docs)]
    reqs = []
    for _ in range(n_requests):
        k = int(rng.integers(1, max_docs_per_req + 1))
        pick = [docs[int(i)] for i in rng.integers(0, n_docs, size=k)]
        ql = int(rng.integers(query_len[0], query_len[1] + 1))
        reqs.append(np.concatenate(pick + [rng.integers(0, 50, size=ql, dtype=np.uint32)]))
    return reqs


def zipf_trace(seed: int = 4, n_docs: int = 1000, n_requests: int = 1000, C: int = 256,
               doc_chunks=(4, 16), zipf_s: float = 1.0, query_len=(128, 256)):
    """configs[4] / SURVEY §8(d) preset Z: a corpus of n_docs documents of 4-16 chunks, doc
    popularity Zipf(s) over a seeded random ranking; each request = 2 distinct docs (ordered,
    drawn by popularity) + a 128-256-token query (2 docs per query).  Returns
    (requests: list of uint32 token arrays, doc_ids: list of (a, b), n_doc_tokens: list)."""
    rng = make_rng(seed)
    docs = [rng.integers(0, VOCAB, size=C * int(rng.integers(doc_chunks[0], doc_chunks[1] + 1)),
                         dtype=np.uint32) for _ in range(n_docs)]
    ranks = rng.permutation(n_docs)
    w = 1.0 / np.arange(1, n_docs + 1, dtype=np.float64) ** zipf_s
    prob = np.empty(n_docs)
    prob[ranks] = w / w.sum()
    reqs, ids, ndoc = [], [], []
    for _ in range(n_requests):
        a, b = rng.choice(n_docs, size=2, replace=False, p=prob)
        ql = int(rng.integers(query_len[0], query_len[1] + 1))
        q = rng.integers(0, VOCAB, size=ql, dtype=np.uint32)
        reqs.append(np.concatenate([docs[a], docs[b], q]))
        ids.append((int(a), int(b)))
        ndoc.append(len(docs[a]) + len(docs[b]))
    return reqs, ids, ndoc
