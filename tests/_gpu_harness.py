"""Test-side GPU harness: drives libpcr.so through its binding and builds the oracle's
expectation for the same seeded inputs.  (Tests only; the product never imports this.)"""
from __future__ import annotations

import numpy as np

from oracle.attention import bf16_bits_to_f64, suffix_attention, suffix_attention_blocked
from oracle.kvload import append_layer, load_layer, logical_kv
from pcrgen import make_rng, pack_store_slots

TOL_REL_L2, TOL_MAX_ABS = 5e-3, 2e-2   # BASELINE.json north_star (bf16 in, fp32 accumulate)


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


def to_host(t):
    return t.cpu().numpy().view(np.uint16)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


class Rig:
    """One device context plus a numpy mirror of the store (what pcr_store_write put there)."""

    def __init__(self, L, Hq, Hkv, d, C, S, store_chunks, n_pool_pages, window=0, rank=0, world=1, **kw):
        import torch
        from paper_2603_23049_b200 import Context
        split = 1 if kw.get("shard_mode", 0) == 1 else world   # context split: all heads on every rank
        self.L, self.Hq, self.Hkv, self.d, self.C, self.S = L, Hq // split, Hkv // split, d, C, S
        page_elems = L * self.Hkv * 2 * S * d
        self.pool = torch.zeros(n_pool_pages * page_elems, dtype=torch.int16, device="cuda")
        self.ctx = Context(L, Hq, Hkv, d, C, S, store_chunks, window, device=torch.cuda.current_device(),
                           pool=self.pool, rank=rank, world=world, **kw)
        self.n_pool_pages = n_pool_pages
        self.store = np.zeros((store_chunks, L, self.Hkv, 2, C, d), np.uint16)
        self.cs = torch.cuda.Stream()
        self.ls = torch.cuda.Stream()

    def write_slot(self, slot, rec):
        self.store[slot] = rec
        self.ctx.store_write(slot, rec)

    def pool_np(self):
        return to_host(self.pool).reshape(self.L, self.n_pool_pages, self.Hkv, 2, self.S, self.d)

    def run(self, req_id, q, k_new, v_new, mode=0, times=False):
        """q [L][N2][Hq][d], k_new/v_new [L][N2][Hkv][d] (bf16 bits) -> out [L][N2][Hq][d] bits."""
        import torch
        qd, kd, vd = to_dev(q), to_dev(k_new), to_dev(v_new)
        out = torch.empty_like(qd)
        t = self.ctx.run_prefill(req_id, qd, kd, vd, out, self.cs, self.ls, mode=mode, layer_times=times)
        self.cs.synchronize()
        return to_host(out), t

    def expected_context(self, plan, k_new, v_new, layer):
        """Logical K/V of the request for one layer: matched store chunks, then the suffix."""
        n_m = plan["n_matched"]
        ks = [self.store[s, layer, :, 0] .transpose(1, 0, 2) for s in plan["slots"][:n_m]]
        vs = [self.store[s, layer, :, 1].transpose(1, 0, 2) for s in plan["slots"][:n_m]]
        k = np.concatenate(ks + [k_new[layer]], axis=0)
        v = np.concatenate(vs + [v_new[layer]], axis=0)
        return k, v

    def expected_pool(self, plan, k_new, v_new, layer, pool_before=None):
        pool = np.zeros((self.L, self.n_pool_pages, self.Hkv, 2, self.S, self.d), np.uint16) \
            if pool_before is None else pool_before.copy()
        load_layer(pool, self.store, plan["slots"], plan["pages"], layer, plan["n1"], self.C, self.S)
        append_layer(pool, k_new[layer], v_new[layer], plan["pages"], layer, plan["n1"], self.S)
        return pool


def check_attention(out_bits, q, k_ctx, v_ctx, n1, rows=None, blocked=False):
    """Compare one layer's GPU output with the fp64 oracle. Returns (rel_l2, max_abs)."""
    qf, kf, vf = bf16_bits_to_f64(q), bf16_bits_to_f64(k_ctx), bf16_bits_to_f64(v_ctx)
    if rows is None:
        ref, _ = (suffix_attention_blocked if blocked else suffix_attention)(qf, kf, vf, n1)
        got = bf16_bits_to_f64(out_bits)
    else:
        ref, _ = suffix_attention(qf, kf, vf, n1, rows=rows)
        got = bf16_bits_to_f64(out_bits[rows])
    return rel_l2(got, ref), float(np.abs(got - ref).max())


def pool_tokens(pool, pages, layer, n_tokens, S):
    return logical_kv(pool, pages, layer, n_tokens, S)


def sample_rows(n2, n1, C, S, k=64, seed=0):
    """Seeded sample incl. row 0, row N2-1 and rows at chunk / page / tile boundaries."""
    rng = make_rng(seed)
    must = {0, n2 - 1}
    for b in (C, S, 128):
        for t in range(0, n1 + n2 + b, b):
            for dt in (-1, 0):
                i = t + dt - n1
                if 0 <= i < n2:
                    must.add(i)
    rest = [i for i in range(n2) if i not in must]
    extra = rng.choice(rest, size=min(len(rest), max(0, k - len(must))), replace=False) if rest else []
    return np.array(sorted(must | set(int(x) for x in extra)))


__all__ = ["Rig", "check_attention", "to_dev", "to_host", "rel_l2", "TOL_REL_L2", "TOL_MAX_ABS",
           "pack_store_slots", "sample_rows"]
