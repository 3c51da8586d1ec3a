"""O5 — a tiny fp64 decoder used to pin the method identity "reuse-then-attend equals
full recompute" and to export realistic (non-iid) Q/K/V for preset T.
(Oracle: test infrastructure only.)

P:227  "the KV cache is computed by multiplying the hidden states with the K and V
       projection weights in each Attention module ... the KV cache is generated layer
       by layer. When two input sequences share the same prefix, they produce identical
       KV caches for that shared portion."
P:230  "this reuse is restricted to scenarios with identical prefixes because each
       document's representations become intertwined with preceding documents."

Per layer (a generic pre-norm GQA decoder; the paper's models are Llama/Qwen):
RMSNorm -> Wq, Wk, Wv -> RoPE at absolute positions -> causal GQA attention (K cached
after RoPE) -> Wo -> residual -> RMSNorm -> SiLU-gated MLP -> residual.
"""
from __future__ import annotations

import numpy as np

from pcrgen import make_rng


class TinyModel:
    def __init__(self, L=2, Hq=4, Hkv=2, d=64, d_model=96, d_ff=128, vocab=512, seed=0):
        self.L, self.Hq, self.Hkv, self.d = L, Hq, Hkv, d
        self.G = Hq // Hkv
        rng = make_rng(seed)
        w = lambda *s: rng.standard_normal(s) / np.sqrt(s[0])  # noqa: E731
        self.emb = rng.standard_normal((vocab, d_model))
        self.layers = [dict(wq=w(d_model, Hq * d), wk=w(d_model, Hkv * d), wv=w(d_model, Hkv * d),
                            wo=w(Hq * d, d_model), w1=w(d_model, d_ff), w3=w(d_model, d_ff),
                            w2=w(d_ff, d_model)) for _ in range(L)]

    @staticmethod
    def _rms(x):
        return x / np.sqrt((x * x).mean(axis=-1, keepdims=True) + 1e-6)

    def _rope(self, x, pos):
        d = x.shape[-1]
        half = d // 2
        inv = 10000.0 ** (-np.arange(half) / half)
        ang = pos[:, None] * inv[None, :]
        c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return np.concatenate([x1 * c - x2 * s, x1 * s + x2 * c], axis=-1)

    def forward(self, tokens, past=None):
        """Run positions [P0, P0+n) where P0 = len of `past` K/V (per layer (K, V) arrays
        [P0][Hkv][d]).  Returns (hidden [n][d_model], kv [(K, V) over all P0+n positions],
        q [per layer [n][Hq][d]])."""
        tokens = np.asarray(tokens, dtype=np.int64)
        n = len(tokens)
        p0 = 0 if past is None else past[0][0].shape[0]
        pos = np.arange(p0, p0 + n, dtype=np.float64)
        x = self.emb[tokens]
        kv_out, q_out = [], []
        for li, W in enumerate(self.layers):
            h = self._rms(x)
            q = self._rope((h @ W["wq"]).reshape(n, self.Hq, self.d), pos)
            k = self._rope((h @ W["wk"]).reshape(n, self.Hkv, self.d), pos)
            v = (h @ W["wv"]).reshape(n, self.Hkv, self.d)
            if past is not None:
                k = np.concatenate([past[li][0], k], axis=0)
                v = np.concatenate([past[li][1], v], axis=0)
            kv_out.append((k, v))
            q_out.append(q)
            att = np.empty((n, self.Hq, self.d))
            for hh in range(self.Hq):
                g = hh // self.G
                s = (q[:, hh, :] @ k[:, g, :].T) / np.sqrt(self.d)
                s[np.arange(p0 + n)[None, :] > (p0 + np.arange(n))[:, None]] = -np.inf
                e = np.exp(s - s.max(axis=1, keepdims=True))
                att[:, hh] = (e @ v[:, g, :]) / e.sum(axis=1, keepdims=True)
            x = x + att.reshape(n, -1) @ W["wo"]
            h = self._rms(x)
            a = h @ W["w1"]
            x = x + ((a / (1 + np.exp(-a))) * (h @ W["w3"])) @ W["w2"]
        return x, kv_out, q_out
