"""O3/O5/O6 pins: pool layout round trip and its necessity, reuse == recompute on a tiny fp64
transformer, the paper's cost arithmetic (Eq.1) and
KV-size arithmetic."""
import numpy as np

from oracle.attention import bf16_bits_to_f64, suffix_attention
from oracle.chunks import chain_keys
from oracle.kvload import append_layer, load_bytes_per_layer, load_layer, logical_kv
from oracle.timing_model import (eq1_cost, kv_bytes, overlap_recurrence, pipelined_bound,
                                 sync_time)
from oracle.tiny_model import TinyModel
from pcrgen import make_rng, pack_store_slots, randn_bf16


# ---------------------------------------------------------------- O3 load / append
def _pool_case(seed=0, L=2, H=2, d=16, C=8, S_pg=4, n_chunks=3, N2=5):
    rng = make_rng(seed)
    N1 = n_chunks * C
    k = randn_bf16(rng, (L, N1 + N2, H, d))
    v = randn_bf16(rng, (L, N1 + N2, H, d))
    store = np.zeros((6, L, H, 2, C, d), np.uint16)
    slots = [4, 0, 2]
    store[slots] = pack_store_slots(k[:, :N1], v[:, :N1], n_chunks, C)
    n_pages = -(-(N1 + N2) // S_pg)
    pages = list(rng.permutation(16)[:n_pages])
    pool = np.zeros((L, 16, H, 2, S_pg, d), np.uint16)
    return k, v, store, slots, pages, pool, N1, N2, C, S_pg


def test_load_append_roundtrip():
    k, v, store, slots, pages, pool, N1, N2, C, S_pg = _pool_case()
    for l in range(2):
        load_layer(pool, store, slots, pages, l, N1, C, S_pg)
        append_layer(pool, k[l, N1:], v[l, N1:], pages, l, N1, S_pg)
        kk, vv = logical_kv(pool, pages, l, N1 + N2, S_pg)
        assert np.array_equal(kk, k[l]) and np.array_equal(vv, v[l])
    assert load_bytes_per_layer(4096, 8, 128) == 16 * 2 ** 20   # L8: 16 MiB per layer (App. B)


def test_page_swap_invisible_to_attention_but_not_to_pool():
    """Why O3's bitwise check is mandatory: attention is permutation-invariant over prefix
    (k, v) pairs, so a page-table bug inside the prefix leaves the output unchanged."""
    k, v, store, slots, pages, pool, N1, N2, C, S_pg = _pool_case(seed=1)
    load_layer(pool, store, slots, pages, 0, N1, C, S_pg)
    append_layer(pool, k[0, N1:], v[0, N1:], pages, 0, N1, S_pg)
    bad = list(pages)
    bad[0], bad[1] = bad[1], bad[0]
    kk, vv = logical_kv(pool, bad, 0, N1 + N2, S_pg)
    assert not np.array_equal(kk, k[0])
    q = bf16_bits_to_f64(randn_bf16(make_rng(2), (N2, 2, 16)))
    o_ok, _ = suffix_attention(q, bf16_bits_to_f64(k[0]), bf16_bits_to_f64(v[0]), N1)
    o_bad, _ = suffix_attention(q, bf16_bits_to_f64(kk), bf16_bits_to_f64(vv), N1)
    assert np.abs(o_ok - o_bad).max() < 1e-12


# ---------------------------------------------------------------- O5 reuse == recompute
def test_reuse_equals_recompute_and_negative_control():
    """P:227 [doc1:doc2:query1] then [doc1:doc3:query2] reuses doc1; P:230 [doc2:doc3:query3]
    reuses nothing — forcing reuse of doc2's KV cached at the wrong offset is wrong."""
    m = TinyModel(L=2, Hq=4, Hkv=2, d=16, d_model=32, d_ff=48, vocab=97, seed=3)
    rng = make_rng(4)
    C = 8
    D1, D2, D3 = (rng.integers(0, 97, 2 * C) for _ in range(3))
    q1, q2, q3 = (rng.integers(0, 97, 5) for _ in range(3))
    A = np.concatenate([D1, D2, q1])
    B = np.concatenate([D1, D3, q2])
    Cq = np.concatenate([D2, D3, q3])
    _, kvA, _ = m.forward(A)
    # prefix tree: B shares exactly D1's two chunks with A; C shares nothing
    kA, kB, kC = chain_keys(A, C), chain_keys(B, C), chain_keys(Cq, C)
    assert kA[:2] == kB[:2] and kA[2] != kB[2]
    assert not set(kC) & set(kA)
    n1 = 2 * C
    past = [(k[:n1], v[:n1]) for k, v in kvA]
    h_reuse, kv_reuse, _ = m.forward(B[n1:], past=past)
    h_full, kv_full, _ = m.forward(B)
    assert np.allclose(h_reuse, h_full[n1:], rtol=1e-12, atol=1e-12)
    for (kr, vr), (kf, vf) in zip(kv_reuse, kv_full):
        assert np.allclose(kr, kf, rtol=1e-12, atol=1e-12) and np.allclose(vr, vf, rtol=1e-12, atol=1e-12)
    # negative control: D2's KV (computed at offset |D1| after D1) reused as C's prefix
    past_bad = [(k[n1:2 * n1], v[n1:2 * n1]) for k, v in kvA]
    h_bad, _, _ = m.forward(Cq[n1:], past=past_bad)
    h_ok, _, _ = m.forward(Cq)
    assert np.abs(h_bad - h_ok[n1:]).max() > 1e-3


# ---------------------------------------------------------------- O6 cost model
def test_eq1_identity_and_example():
    for n1, n2, c1, c2 in [(4096, 4096, 0.5, 2.0), (100, 7, 3.0, 11.0), (0, 10, 1.0, 1.0)]:
        assert np.isclose(eq1_cost(n1, n2, c1, c2), c1 + n2 / (n1 + n2) * c2)
    # half of 8k reused, C1 = 0.5 s, C2 = 2 s -> 1.5 s; transfer 0.5 s vs compute 2 s = 25%
    assert np.isclose(eq1_cost(4096, 4096, 0.5, 2.0), 1.5)
    assert np.isclose(0.5 / 2.0, 0.25)


def test_spec_pipeline_example():
    """n=4 layers, load 1, compute 3, offload 1 -> SYNC 20, overlap 14."""
    load, attn, off = [1] * 4, [3] * 4, [1] * 4
    assert sync_time(load, attn, off) == 20
    assert overlap_recurrence(load, attn, off)[0] == 14


def test_overlap_overhead_is_one_layer_of_load():
    """with per-layer load <= per-layer compute, overhead C1 -> C1/n."""
    for n, c1, c2 in [(32, 0.5, 2.0), (80, 1.0, 1.5), (4, 2.0, 2.0)]:
        t, _ = overlap_recurrence([c1 / n] * n, [c2 / n] * n)
        assert np.isclose(t - c2, c1 / n)
        assert np.isclose(sync_time([c1 / n] * n, [c2 / n] * n) - c2, c1)


def test_recurrence_vs_tick_simulation_and_bounds():
    """the recurrence equals a brute-force unit-tick simulation of two in-order
    streams with a per-layer event dependency; SYNC >= overlap >= max(sum load, sum attn)."""
    rng = make_rng(11)
    for _ in range(1000):
        n = int(rng.integers(1, 7))
        load = [int(x) for x in rng.integers(0, 5, n)]
        attn = [int(x) for x in rng.integers(1, 5, n)]
        # tick simulation
        t, li, ai, lrem, arem, loaded, done = 0, 0, 0, None, None, 0, 0
        while done < n:
            if lrem is None and li < n:
                lrem = load[li]
            if arem is None and ai < n and loaded > ai:
                arem = attn[ai]
            while lrem == 0:            # zero-length loads complete instantly
                loaded += 1
                li += 1
                lrem = load[li] if li < n else None
                if arem is None and ai < n and loaded > ai:
                    arem = attn[ai]
            t += 1
            if lrem is not None:
                lrem -= 1
                if lrem == 0:
                    loaded, li, lrem = loaded + 1, li + 1, None
            if arem is not None:
                arem -= 1
                if arem == 0:
                    done, ai, arem = done + 1, ai + 1, None
        rec, _ = overlap_recurrence(load, attn)
        assert rec == t, (load, attn, rec, t)
        assert sync_time(load, attn) >= rec >= max(sum(load), sum(attn))
        # T* equals the recurrence when every layer costs the same
        u = overlap_recurrence([load[0]] * n, [attn[0]] * n)[0]
        assert pipelined_bound([load[0]] * n, [attn[0]] * n) == u


def test_kv_size_arithmetic():
    # H100 80 GB holds "about 163,000" Llama2-7B tokens (32 layers, 32 heads, d=128, 2 B)
    assert (80 * 2 ** 30) // kv_bytes(1, 32, 32, 128) == 163_840
    # Llama2-13B (40 layers, 40 heads) at 8192K tokens "6.23 TB" == 6.25 TiB
    assert kv_bytes(8192 * 1024, 40, 40, 128) == int(6.25 * 2 ** 40)
    # one Llama2-13B chunk-layer = 256 tokens x 1 layer = 5 MiB; 0.261 ms -> 20.1 GB/s
    b = kv_bytes(256, 1, 40, 128)
    assert b == 5_242_880 and abs(b / 0.261e-3 / 1e9 - 20.09) < 0.01
