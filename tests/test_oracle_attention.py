"""O4 pins: fp64 suffix attention against library routines and closed-form special cases
(SURVEY §8(c) O4), plus the sensitivity of the parity check to plausible kernel bugs."""
import numpy as np
import pytest
import torch

from oracle.attention import (attention_flops_per_layer, bf16_bits_to_f64, suffix_attention,
                              suffix_attention_blocked)
from pcrgen import f32_to_bf16_bits, make_rng, stress_values

TOL_REL_L2, TOL_MAX_ABS = 5e-3, 2e-2   # BASELINE.json north_star


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _inputs(kind, N1, N2, Hq=4, Hkv=2, d=64, seed=0):
    q, k, v = stress_values(kind, seed, N1, N2, Hq, Hkv, d)
    return bf16_bits_to_f64(q), bf16_bits_to_f64(k), bf16_bits_to_f64(v)


def _sdpa(q, k, v, n1):
    """torch fp64 scaled_dot_product_attention with an explicit causal mask over absolute
    positions and GQA expanded by repeat_interleave (kv head = floor(h/G))."""
    N2, Hq, d = q.shape
    G = Hq // k.shape[1]
    qt = torch.from_numpy(q).permute(1, 0, 2)
    kt = torch.from_numpy(k).permute(1, 0, 2).repeat_interleave(G, 0)
    vt = torch.from_numpy(v).permute(1, 0, 2).repeat_interleave(G, 0)
    N = k.shape[0]
    mask = torch.arange(N)[None, :] <= (n1 + torch.arange(N2))[:, None]
    o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask)
    return o.permute(1, 0, 2).numpy()


def test_bf16_decode_exact():
    x = np.array([1.0, -2.5, 3.140625, 0.0, 1e-3], dtype=np.float32)
    bits = f32_to_bf16_bits(x)
    back = bf16_bits_to_f64(bits)
    assert back[0] == 1.0 and back[1] == -2.5 and back[2] == 3.140625 and back[3] == 0.0
    assert abs(back[4] - 1e-3) < 1e-3 * 2 ** -8


@pytest.mark.parametrize("kind", ["iid", "q4", "kout", "advfuture"])
@pytest.mark.parametrize("N1,N2", [(0, 37), (64, 64), (200, 17), (128, 1)])
def test_matches_torch_sdpa(kind, N1, N2):
    q, k, v = _inputs(kind, N1, N2)
    o, _ = suffix_attention(q, k, v, N1)
    assert np.allclose(o, _sdpa(q, k, v, N1), rtol=1e-10, atol=1e-12)
    ob, _ = suffix_attention_blocked(q, k, v, N1)
    assert np.allclose(o, ob, rtol=1e-11, atol=1e-13)


def test_n1_zero_is_causal_self_attention():
    q, k, v = _inputs("iid", 0, 50)
    o, _ = suffix_attention(q, k, v, 0)
    G = 2
    qt = torch.from_numpy(q).permute(1, 0, 2)
    kt = torch.from_numpy(k).permute(1, 0, 2).repeat_interleave(G, 0)
    vt = torch.from_numpy(v).permute(1, 0, 2).repeat_interleave(G, 0)
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True)
    assert np.allclose(o, ref.permute(1, 0, 2).numpy(), rtol=1e-10, atol=1e-12)


def test_single_visible_key():
    q, k, v = _inputs("iid", 0, 5)
    o, lse = suffix_attention(q, k, v, 0, rows=[0])
    for h in range(4):
        assert np.allclose(o[0, h], v[0, h // 2], atol=0, rtol=1e-15)
        assert np.isclose(lse[0, h], q[0, h] @ k[0, h // 2] / 8.0)


def test_all_equal_keys_gives_mean_of_visible_values():
    q, k, v = _inputs("iid", 40, 10)
    k[:] = k[0]
    o, lse = suffix_attention(q, k, v, 40)
    for i in range(10):
        for h in range(4):
            assert np.allclose(o[i, h], v[: 40 + i + 1, h // 2].mean(axis=0), rtol=1e-12, atol=1e-13)
            s = q[i, h] @ k[0, h // 2] / 8.0
            assert np.isclose(lse[i, h], s + np.log(40 + i + 1))


def test_dominant_logit_selects_its_value():
    q, k, v = _inputs("iid", 30, 4)
    j = 11
    k[j, 0] = q[2, 0] / np.linalg.norm(q[2, 0]) * 400.0
    o, _ = suffix_attention(q, k, v, 30, rows=[2])
    assert np.allclose(o[0, 0], v[j, 0], atol=1e-12)


def test_lse_closed_form_uniform_scores():
    q, k, v = _inputs("iid", 10, 3)
    q[:] = 0.0
    _, lse = suffix_attention(q, k, v, 10)
    assert np.allclose(lse, np.log(10 + 1 + np.arange(3))[:, None])


def test_flops_formula():
    # L8 per layer (8.73 GFLOP) and M7 r=0 (567.14 GFLOP)
    assert abs(attention_flops_per_layer(4096, 128, 32, 128) / 1e9 - 8.73) < 0.01
    assert abs(attention_flops_per_layer(0, 8320, 32, 128) / 1e9 - 567.14) < 0.01


# ---- sensitivity: the parity check must FAIL for plausible kernel bugs -----------------

def _leaky(q, k, v, n1, shift=1):
    """Causal mask shifted by `shift` (row i sees keys up to N1+i+shift)."""
    N2 = q.shape[0]
    kk = np.concatenate([k, np.zeros((shift,) + k.shape[1:])])
    vv = np.concatenate([v, np.zeros((shift,) + v.shape[1:])])
    o, _ = suffix_attention(q, kk, vv, n1 + shift)
    return o


def _wrong_group(q, k, v, n1):
    Hq, Hkv = q.shape[1], k.shape[1]
    perm = [h % Hkv for h in range(Hq)]     # h % Hkv instead of floor(h / G)
    G = Hq // Hkv
    kk = np.stack([k[:, perm[h]] for h in range(0, Hq, G)] if False else [k[:, p] for p in perm], 1)
    vv = np.stack([v[:, p] for p in perm], 1)
    # run as MHA (G = 1) over the permuted per-q-head K/V
    o = np.empty_like(q)
    for h in range(Hq):
        oh, _ = suffix_attention(q[:, h:h + 1], kk[:, h:h + 1], vv[:, h:h + 1], n1)
        o[:, h] = oh[:, 0]
    return o


def test_mutation_shifted_mask_fails_advfuture():
    q, k, v = _inputs("advfuture", 96, 32)
    ref, _ = suffix_attention(q, k, v, 96)
    bad = _leaky(q, k, v, 96)
    assert rel_l2(bad, ref) > 100 * TOL_REL_L2


def test_mutation_wrong_kv_head_map_fails():
    q, k, v = _inputs("iid", 64, 16, Hq=8, Hkv=2)
    ref, _ = suffix_attention(q, k, v, 64)
    bad = _wrong_group(q, k, v, 64)
    assert rel_l2(bad, ref) > 10 * TOL_REL_L2


def test_bf16_pipeline_emulation_within_tolerance():
    """A numpy emulation of the kernel's arithmetic (fp32 scores, 128-key online softmax,
    bf16 P, fp32 accumulation, bf16 output) stays inside the north_star tolerance: the bar
    is achievable, and it is not so loose that the mutations above pass."""
    rng = make_rng(5)
    N1, N2, d = 512, 64, 128
    q, k, v = _inputs("kout", N1, N2, Hq=4, Hkv=1, d=d, seed=3)
    ref, _ = suffix_attention(q, k, v, N1)
    f32 = np.float32
    out = np.empty_like(ref)
    bf = lambda x: bf16_bits_to_f64(f32_to_bf16_bits(x)).astype(f32)  # noqa: E731
    for h in range(4):
        for i in range(N2):
            p = N1 + i
            m, l, acc = -np.inf, f32(0), np.zeros(d, f32)
            for j0 in range(0, p + 1, 128):
                ks = k[j0:min(p + 1, j0 + 128), 0].astype(f32)
                s = (ks @ q[i, h].astype(f32)) * f32(1 / np.sqrt(d))
                mn = max(m, float(s.max()))
                a = f32(np.exp(m - mn)) if m != -np.inf else f32(0)
                pr = np.exp(s - f32(mn)).astype(f32)
                l = l * a + pr.sum(dtype=f32)
                acc = acc * a + bf(pr) @ v[j0:j0 + len(ks), 0].astype(f32)
                m = mn
            out[i, h] = bf(acc / l)
    assert rel_l2(out, ref) < TOL_REL_L2 / 2
    assert np.abs(out - ref).max() < TOL_MAX_ABS / 2
    del rng
