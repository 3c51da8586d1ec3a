"""O6 — the paper's cost model and the layer-wise overlap recurrence.
(Oracle: test infrastructure only.)

P:282-285 Eq.(1)  C = (N1/N) C1 + (N2/N) C2 + (N2/N) C1 = C1 + (N2/N) C2, where C1 = time to
                  load (or offload) the KV of N tokens and C2 = compute time for N tokens.
P:287     example: Llama2-13B, 8k tokens, half reused, C2 ~ 2 s, C1 ~ 0.5 s -> 25% overhead.
P:400     layer-wise overlap "reduces the overhead to (1/n) C1"; P:402 requires per-layer
          load/offload <= per-layer compute.
P:480     three streams: CPU->GPU, compute, GPU->CPU.
S:270-273 recurrence and its example (n=4, load 1, compute 3, offload 1: SYNC 20, overlap 14).
P:267/269 KV size arithmetic (H100 80 GB ~ 163,000 Llama2-7B tokens; Llama2-13B 8192K tokens
          ~ 6.23 TB); P:480 one Llama2-13B chunk-layer.
"""
from __future__ import annotations


def eq1_cost(n1, n2, c1, c2):
    n = n1 + n2
    return (n1 / n) * c1 + (n2 / n) * c2 + (n2 / n) * c1


def sync_time(load, attn, offload=None):
    offload = offload or [0.0] * len(load)
    return sum(load) + sum(attn) + sum(offload)


def overlap_recurrence(load, attn, offload=None):
    """Three in-order streams: L_l = L_{l-1} + load_l;  A_l = max(L_l, A_{l-1}) + attn_l;
    O_l = max(A_l, O_{l-1}) + offload_l.  Returns (finish time, per-layer A_l)."""
    Lt = At = Ot = 0.0
    a_list = []
    for l in range(len(load)):
        Lt = Lt + load[l]
        At = max(Lt, At) + attn[l]
        a_list.append(At)
        if offload is not None:
            Ot = max(At, Ot) + offload[l]
    return (Ot if offload is not None else At), a_list


def pipelined_bound(load, attn):
    """T* = t_ld(0) + sum_{l<L-1} max(t_at(l), t_ld(l+1)) + t_at(L-1)."""
    n = len(load)
    return load[0] + sum(max(attn[l], load[l + 1]) for l in range(n - 1)) + attn[n - 1]


def kv_bytes(tokens, n_layers, n_kv_heads, head_dim, elem_bytes=2):
    """K and V of `tokens` tokens over all layers."""
    return 2 * n_layers * n_kv_heads * head_dim * elem_bytes * tokens
