"""GPU parity: libpcr.so (sm_100a kernels, through the C-ABI) vs the fp64 oracle on the same
seeded inputs.  Pool contents bit-exact (O3), attention within the north_star tolerance
(rel-L2 <= 5e-3, max-abs <= 2e-2, O4), plans bit-exact (O2)."""
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.tree import PlanOracle  # noqa: E402
from oracle.tiny_model import TinyModel  # noqa: E402
from pcrgen import (appendix_c_trace, f32_to_bf16_bits, make_rng, pack_store_slots,  # noqa: E402
                    stress_values)
from oracle.attention import bf16_bits_to_f64, suffix_attention_blocked  # noqa: E402
from oracle.kvload import append_layer, load_layer  # noqa: E402
from tests._gpu_harness import (TOL_MAX_ABS, TOL_REL_L2, Rig, check_attention, rel_l2, sample_rows,  # noqa: E402
                                to_dev, to_host)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _warm_prefix(rig, req_id, doc_tokens, k_ctx, v_ctx, n_chunks):
    """Commit a request whose first n_chunks chunks are `doc_tokens`, writing their KV."""
    toks = np.concatenate([doc_tokens, np.array([7], np.uint32)])
    rig.ctx.submit(req_id, toks)
    plan = rig.ctx.match_prefix(req_id, [])
    assert plan["n_matched"] == 0 and plan["n_reserved"] == n_chunks
    recs = pack_store_slots(k_ctx, v_ctx, n_chunks, rig.C)
    for c, s in enumerate(plan["slots"]):
        rig.write_slot(s, recs[c])
    rig.ctx.release(req_id, True)


def _single_request(kind, L, Hq, Hkv, d, C, S, N1, N2, seed, mode=0, world=1, rank=0, local_only=False,
                    fragment=False, **ctx_kw):
    """Warm N1 tokens, then run one request [doc | query] and return everything to compare.
    local_only: draw only this rank's heads (full-size sharded shapes) instead of slicing them out
    of all heads."""
    rng = make_rng(seed)
    Hkv_l, Hq_l = Hkv // world, Hq // world
    q, k, v = [], [], []
    for l in range(L):
        ql, kl, vl = stress_values(kind, seed * 100 + l, N1, N2, Hq_l if local_only else Hq,
                                   Hkv_l if local_only else Hkv, d)
        q.append(ql)
        k.append(kl)
        v.append(vl)
    q, k, v = np.stack(q), np.stack(k), np.stack(v)       # [L][N2][Hq][d], [L][N][Hkv][d]
    if not local_only:
        hs = slice(rank * Hkv_l, (rank + 1) * Hkv_l)
        qs = slice(rank * Hq_l, (rank + 1) * Hq_l)
        q, k, v = q[:, :, qs], k[:, :, hs], v[:, :, hs]
    n_pages = (N1 + N2) // S + 8
    rig = Rig(L, Hq, Hkv, d, C, S, store_chunks=max(1, N1 // C) + 2, n_pool_pages=n_pages + N1 // S + 2,
              rank=rank, world=world, **ctx_kw)
    doc = rng.integers(0, 1000, N1, dtype=np.uint32)
    if N1:
        _warm_prefix(rig, 1000, doc, k[:, :N1], v[:, :N1], N1 // C)
    if fragment:
        # two one-page requests hold pool pages 0 and 1; releasing the first leaves a hole, so
        # the request's pages are [0, 2, 3, ...]: its first chunk's pages are not consecutive
        for hid in (2000, 2001):
            rig.ctx.submit(hid, rng.integers(5000, 6000, S, dtype=np.uint32), n_cacheable=0)
            assert rig.ctx.match_prefix(hid, [])["pages"] == [hid - 2000]
        rig.ctx.release(2000, False)
    toks = np.concatenate([doc, rng.integers(0, 1000, N2, dtype=np.uint32)])
    rig.ctx.submit(1, toks, n_cacheable=N1)
    plan = rig.ctx.match_prefix(1, [])
    assert plan["n1"] == N1 and plan["n2"] == N2
    out, _ = rig.run(1, q, k[:, N1:], v[:, N1:], mode=mode)
    return rig, plan, q, k, v, out


CASES = [
    # (L, Hq, Hkv, d, C, S, N1, N2)
    (2, 32, 8, 128, 256, 64, 1024, 128),   # L8 geometry, short
    (2, 32, 8, 128, 256, 16, 512, 200),    # ragged N2, paper's 16-token pages
    (2, 64, 8, 128, 256, 64, 768, 77),     # G = 8 (Llama-3-70B shape)
    (2, 8, 8, 128, 128, 32, 256, 300),     # G = 1 (MHA), several M tiles
    (2, 4, 2, 64, 64, 16, 256, 64),        # preset T geometry
    (1, 32, 8, 128, 256, 128, 0, 333),     # N1 = 0: plain causal self-attention
    (1, 32, 8, 128, 256, 64, 2048, 1),     # N2 = 1: decode-like row
    (1, 8, 2, 64, 64, 16, 512, 700),       # d = 64, several M blocks, ragged
    (1, 4, 2, 64, 64, 16, 4096, 32),       # d = 64 with KV splits (small grid, long prefix)
    (1, 32, 8, 128, 512, 128, 1024, 100),  # 512-token chunks, 128-token pages
]


@pytest.mark.parametrize("kind", ["iid", "q4", "kout", "advfuture"])
@pytest.mark.parametrize("case", CASES, ids=[f"L{c[0]}H{c[1]}/{c[2]}d{c[3]}S{c[5]}N{c[6]}+{c[7]}" for c in CASES])
def test_attention_and_pool_vs_oracle(kind, case):
    L, Hq, Hkv, d, C, S, N1, N2 = case
    rig, plan, q, k, v, out = _single_request(kind, L, Hq, Hkv, d, C, S, N1, N2, seed=zlib.crc32(repr((kind,) + case).encode()) % 1000)
    pool = rig.pool_np()
    for l in range(L):
        # O3: the WHOLE pool layer bit-exact (the request's pages, the tail rows of its last page
        # -- zero-filled by the append, a kernel property -- and every other page, still zero)
        exp_pool = rig.expected_pool(plan, k[:, N1:], v[:, N1:], l)
        assert np.array_equal(pool[l], exp_pool[l]), l
        kc, vc = rig.expected_context(plan, k[:, N1:], v[:, N1:], l)
        assert np.array_equal(kc, k[l]) and np.array_equal(vc, v[l])
        r, m = check_attention(out[l], q[l], kc, vc, N1, blocked=True)
        assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (l, r, m)


def test_overlap_sync_and_per_layer_api_are_bitwise_identical():
    rig, plan, q, k, v, out = _single_request("iid", 3, 32, 8, 128, 256, 64, 1024, 130, seed=5)
    rig.ctx.release(1, True)
    toks_plan = rig.ctx
    # same request again: SYNC mode
    rng = make_rng(5)
    doc = rng.integers(0, 1000, 1024, dtype=np.uint32)
    toks = np.concatenate([doc, rng.integers(0, 1000, 130, dtype=np.uint32)])
    toks_plan.submit(2, toks, n_cacheable=1024)
    p2 = toks_plan.match_prefix(2, [])
    assert p2["n1"] == 1024
    out_sync, _ = rig.run(2, q, k[:, 1024:], v[:, 1024:], mode=1)
    assert np.array_equal(out_sync, out)
    # per-layer API on two streams, ordered by the caller
    toks_plan.release(2, True)
    toks_plan.submit(3, toks, n_cacheable=1024)
    toks_plan.match_prefix(3, [])
    qd, kd, vd = to_dev(q), to_dev(k[:, 1024:]), to_dev(v[:, 1024:])
    o = torch.empty_like(qd)
    for l in range(3):
        rig.ctx.load_layer_kv(3, l, rig.ls)
        ev = torch.cuda.Event()
        ev.record(rig.ls)
        rig.cs.wait_event(ev)
        rig.ctx.prefill_attn_layer(3, l, qd[l], kd[l], vd[l], o[l], rig.cs)
    rig.cs.synchronize()
    assert np.array_equal(to_host(o), out)


@pytest.mark.parametrize("mode,load_mode,ring", [(0, 0, 2), (1, 0, 0), (0, 0, 0), (0, 1, 2), (1, 1, 2), (0, 2, 0)])
def test_host_io_matches_device_buffers(mode, load_mode, ring):
    """pcr_run_prefill_ex with host_io: page-locked HOST q/k/v/out, staged per layer by the library
    (in OVERLAP mode the inputs ride in the layer's load: inside the gather launch with the SM
    gather, one cudaMemcpyAsync each ahead of the copy-engine baselines), gives the device-buffer
    result bit for bit (OVERLAP and SYNC); 5 layers with a 2-deep staging ring so it wraps, and the
    default (whole-request) ring; pageable host memory is refused."""
    L, n1, n2 = 5, 1024, 130
    rig, plan, q, k, v, out = _single_request("iid", L, 32, 8, 128, 256, 64, n1, n2, seed=9, load_mode=load_mode)
    rig.ctx.release(1, True)
    rng = make_rng(9)
    doc = rng.integers(0, 1000, n1, dtype=np.uint32)
    toks = np.concatenate([doc, rng.integers(0, 1000, n2, dtype=np.uint32)])
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).pin_memory()  # noqa: E731
    qh, kh, vh = pin(q), pin(k[:, n1:]), pin(v[:, n1:])
    oh = torch.zeros_like(qh).pin_memory()
    for rid in (2, 3):
        rig.ctx.submit(rid, toks, n_cacheable=n1)
        assert rig.ctx.match_prefix(rid, [])["n1"] == n1
        rig.ctx.run_prefill_ex(rid, qh, kh, vh, oh, rig.cs, rig.ls, mode=mode, host_io=True, io_ring_layers=ring)
        rig.cs.synchronize()
        assert np.array_equal(oh.numpy().view(np.uint16), out), rid
        rig.ctx.release(rid, True)
        oh.zero_()
    rig.ctx.submit(4, toks, n_cacheable=n1)
    rig.ctx.match_prefix(4, [])
    with pytest.raises(Exception):
        rig.ctx.run_prefill_ex(4, torch.from_numpy(q.view(np.int16)), kh, vh, oh, rig.cs, rig.ls, mode=mode,
                               host_io=True)


def test_page_size_does_not_change_results():
    outs = []
    for S in (16, 32, 64, 128):
        _, _, _, _, _, out = _single_request("kout", 1, 32, 8, 128, 256, S, 1024, 96, seed=9)
        outs.append(out)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_full_context_self_consistency():
    """suffix_attn with N1 = 0 over the whole context, last N2 rows == the reuse
    path's output (the kernel's per-row math does not depend on the M-tile split)."""
    L, Hq, Hkv, d, C, S, N1, N2 = 1, 32, 8, 128, 256, 64, 512, 128
    rig, plan, q, k, v, out = _single_request("iid", L, Hq, Hkv, d, C, S, N1, N2, seed=3)
    # full-context run: queries for all N tokens (prefix rows random, suffix rows = q)
    rng = make_rng(4)
    qfull = np.concatenate([f32_to_bf16_bits(rng.standard_normal((L, N1, Hq, d), dtype=np.float32)), q], axis=1)
    rig2 = Rig(L, Hq, Hkv, d, C, S, store_chunks=2, n_pool_pages=(N1 + N2) // S + 4)
    rig2.ctx.submit(5, rng.integers(0, 1000, N1 + N2, dtype=np.uint32), n_cacheable=0)
    p = rig2.ctx.match_prefix(5, [])
    assert p["n1"] == 0
    full, _ = rig2.run(5, qfull, k, v)
    a, b = full[:, N1:], out
    from tests._gpu_harness import rel_l2
    from oracle.attention import bf16_bits_to_f64
    assert rel_l2(bf16_bits_to_f64(a), bf16_bits_to_f64(b)) <= TOL_REL_L2
    print("full-context vs reuse bitwise equal:", np.array_equal(a, b))


def test_kv_head_sharding_concat_equals_single_gpu():
    """SURVEY §8(e)/O7 on one GPU: rank r's context owns kv heads [r*Hkv/P, (r+1)*Hkv/P);
    concatenating the P ranks' outputs by head equals the P=1 output bit for bit, and each
    rank's pool holds exactly its head slice."""
    full = _single_request("iid", 2, 32, 8, 128, 256, 64, 512, 100, seed=21)[5]
    for P in (2, 4, 8):
        parts = [_single_request("iid", 2, 32, 8, 128, 256, 64, 512, 100, seed=21, world=P, rank=r)[5]
                 for r in range(P)]
        assert np.array_equal(np.concatenate(parts, axis=2), full)


def test_appendix_c_trace_tiny_model():
    """Preset T end to end: the Appendix C trace with realistic (tiny-transformer) Q/K/V,
    look-ahead W=2: plans bit-exact vs the oracle planner, pool bit-exact, attention in tol."""
    g = dict(L=2, Hq=4, Hkv=2, d=64, C=64, S=16)
    docs, order, reqs = appendix_c_trace(0)
    model = TinyModel(L=2, Hq=4, Hkv=2, d=64, d_model=96, d_ff=128, vocab=1 << 17, seed=0)
    W = 2
    rig = Rig(g["L"], g["Hq"], g["Hkv"], g["d"], g["C"], g["S"], store_chunks=10, n_pool_pages=64, window=W)
    orc = PlanOracle(C=64, S_pg=16, store_chunks=10, n_pages=64, window=W)
    for i, t in enumerate(reqs):
        rig.ctx.submit(i, t)
        orc.submit(i, t)
    for i, toks in enumerate(reqs):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
        plan = rig.ctx.match_prefix(i, pend)
        po = orc.match_prefix(i, pend)
        for f in ("n_matched", "n_reserved", "n1", "n2", "slots", "pages"):
            assert plan[f] == po[f]
        assert plan["evicted"] == po["evicted"]
        _, kv, qs = model.forward(toks)
        N1, N = plan["n1"], len(toks)
        q = np.stack([f32_to_bf16_bits(qs[l][N1:].astype(np.float32)) for l in range(2)])
        k = np.stack([f32_to_bf16_bits(kv[l][0].astype(np.float32)) for l in range(2)])
        v = np.stack([f32_to_bf16_bits(kv[l][1].astype(np.float32)) for l in range(2)])
        out, _ = rig.run(i, q, k[:, N1:], v[:, N1:])
        pool = rig.pool_np()
        for l in range(2):
            exp_pool = rig.expected_pool(plan, k[:, N1:], v[:, N1:], l, pool_before=pool)
            assert np.array_equal(pool[l], exp_pool[l])
            kc, vc = rig.expected_context(plan, k[:, N1:], v[:, N1:], l)
            r, m = check_attention(out[l], q[l], kc, vc, N1)
            assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (i, l, r, m)
        # "offload": the reserved chunks' KV as computed by this request
        recs = pack_store_slots(k, v, plan["n_matched"] + plan["n_reserved"], 64)
        for c in range(plan["n_matched"], plan["n_matched"] + plan["n_reserved"]):
            rig.write_slot(plan["slots"][c], recs[c])
        rig.ctx.release(i, True)
        orc.release(i, True)


def test_l8_full_size_full_check():
    """configs[1] at full size in the bench's launch configuration (OVERLAP, 32 layers, SM gather,
    4096 cached + 128 query): EVERY output row of every head of all 32 layers against the fp64
    oracle ("Full checks run on T and L8"), and the WHOLE pool array bit-exact
    (O3): a stray 16-byte store into another page or layer fails it.  Prints the worst
    (layer, head)."""
    L, Hq, Hkv, d, C, S, N1, N2 = 32, 32, 8, 128, 256, 64, 4096, 128
    rig, plan, q, k, v, out = _single_request("iid", L, Hq, Hkv, d, C, S, N1, N2, seed=1)
    st = rig.ctx.stats
    assert st["sm_layer_loads"] == L and st["ce_layer_loads"] == 0   # the mover bench.py times
    pool = rig.pool_np()
    exp_pool = np.zeros_like(pool)
    for l in range(L):
        load_layer(exp_pool, rig.store, plan["slots"], plan["pages"], l, N1, C, S)
        append_layer(exp_pool, k[l, N1:], v[l, N1:], plan["pages"], l, N1, S)
    assert np.array_equal(pool, exp_pool)
    worst = (0.0, None)
    rels = []
    for l in range(L):
        kc, vc = rig.expected_context(plan, k[:, N1:], v[:, N1:], l)
        qf, kf, vf = bf16_bits_to_f64(q[l]), bf16_bits_to_f64(kc), bf16_bits_to_f64(vc)
        ref, _ = suffix_attention_blocked(qf, kf, vf, N1)
        got = bf16_bits_to_f64(out[l])
        r, m = rel_l2(got, ref), float(np.abs(got - ref).max())
        rels.append(r)
        assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (l, r, m)
        for h in range(Hq):
            rh = rel_l2(got[:, h], ref[:, h])
            if rh > worst[0]:
                worst = (rh, (l, h))
    print(f"L8 full check: rel-L2 mean {np.mean(rels):.3e} max {max(rels):.3e}; worst (layer, head) "
          f"{worst[1]} rel-L2 {worst[0]:.3e}")


def _check_sampled(rig, plan, q, k, v, out, N1, N2, C, S, layers, seed):
    rows = sample_rows(N2, N1, C, S, k=48, seed=seed)
    pool = rig.pool_np()
    for l in layers:
        exp_pool = rig.expected_pool(plan, k[:, N1:], v[:, N1:], l)
        assert np.array_equal(pool[l], exp_pool[l]), l      # whole layer of the pool
        kc, vc = rig.expected_context(plan, k[:, N1:], v[:, N1:], l)
        r, m = check_attention(out[l], q[l], kc, vc, N1, rows=rows)
        assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (l, r, m)


def test_m7_half_hit_full_size_sampled():
    """configs[2] (Mistral-7B shape, 8k-token document context) at 50% prefix hit, full size,
    OVERLAP: 32 layers, N1 = 4096 cached + N2 = 4224 computed (multi-wave attention grid, no KV
    split); sampled rows vs the oracle and the pool bit-exact on layers 0, 17, 31."""
    L, Hq, Hkv, d, C, S, N1, N2 = 32, 32, 8, 128, 256, 64, 4096, 4224
    rig, plan, q, k, v, out = _single_request("iid", L, Hq, Hkv, d, C, S, N1, N2, seed=4)
    _check_sampled(rig, plan, q, k, v, out, N1, N2, C, S, (0, 17, 31), seed=4)


def test_l70_rank_slice_full_size_sampled():
    """configs[3] (Llama-3-70B shape, 80 layers, 64/8 heads) KV-head-sharded over 8 GPUs: the
    per-GPU workload of rank 5 (8 query heads, 1 KV head) at 16k context, 50% hit -- N1 = 8192
    cached + N2 = 8320 computed; sampled rows and pool on layers 0, 41, 79."""
    L, Hq, Hkv, d, C, S, N1, N2 = 80, 64, 8, 128, 256, 64, 8192, 8320
    rig, plan, q, k, v, out = _single_request("iid", L, Hq, Hkv, d, C, S, N1, N2, seed=6, world=8, rank=5,
                                              local_only=True)
    _check_sampled(rig, plan, q, k, v, out, N1, N2, C, S, (0, 41, 79), seed=6)


def test_sharded_run_with_nccl_allgather_world1():
    """The in-library per-layer NCCL all-gather path (pcr_run_prefill_sharded) on a world-1
    communicator: the gathered tensor equals the local output bit for bit, and the output
    equals pcr_run_prefill's."""
    from paper_2603_23049_b200 import comm_unique_id
    rig, plan, q, k, v, out = _single_request("iid", 2, 32, 8, 128, 256, 64, 512, 100, seed=33)
    rig.ctx.release(1, True)
    rng = make_rng(33)
    doc = rng.integers(0, 1000, 512, dtype=np.uint32)
    toks = np.concatenate([doc, rng.integers(0, 1000, 100, dtype=np.uint32)])
    rig.ctx.submit(2, toks, n_cacheable=512)
    rig.ctx.match_prefix(2, [])
    rig.ctx.comm_init(comm_unique_id())
    qd, kd, vd = to_dev(q), to_dev(k[:, 512:]), to_dev(v[:, 512:])
    o = torch.empty_like(qd)
    gathered = torch.empty((2, 1) + tuple(qd.shape[1:]), dtype=qd.dtype, device="cuda")
    xs = torch.cuda.Stream()
    rig.ctx.run_prefill_sharded(2, qd, kd, vd, o, gathered, rig.cs, rig.ls, xs)
    rig.cs.synchronize()
    assert np.array_equal(to_host(o), out)
    assert np.array_equal(to_host(gathered)[:, 0], out)


@pytest.mark.parametrize("fragment", [False, True])
@pytest.mark.parametrize("load_mode,frac", [(1, 0.0), (2, 0.0), (3, 0.0), (4, 0.34), (4, 1.0)])
def test_copy_engine_baselines_match_gather(load_mode, frac, fragment):
    """f4 baselines (the paper's copy-engine path: one cudaMemcpyAsync per merged run or per
    page image), the TMA experiment and the hybrid copy-engine + gather-kernel load produce the same
    pool bits and outputs as the SM gather kernel, and the whole pool equals the oracle's (O3) --
    with the request's pages consecutive (copy-engine runs merge to whole chunk-layers) and with a
    hole in them."""
    args = ("kout", 2, 32, 8, 128, 256, 16, 768, 90)
    rig0, plan0, q, k, v, out0 = _single_request(*args, seed=44, fragment=fragment)
    rig1, plan1, _, _, _, out1 = _single_request(*args, seed=44, fragment=fragment, load_mode=load_mode,
                                                 load_ce_fraction=frac)
    assert plan0["pages"] == plan1["pages"] and plan0["slots"] == plan1["slots"]
    if fragment:
        assert plan1["pages"][:3] == [0, 2, 3]
    assert np.array_equal(out0, out1)
    p0, p1 = rig0.pool_np(), rig1.pool_np()
    assert np.array_equal(p0, p1)
    for layer in range(2):
        exp = rig1.expected_pool(plan1, k[:, 768:], v[:, 768:], layer)
        assert np.array_equal(p1[layer], exp[layer])
    st = rig1.ctx.stats
    if load_mode in (1, 2):
        assert st["ce_layer_loads"] == 2 and st["sm_layer_loads"] == 0
    if load_mode == 1:   # 3 chunks x 16 page images; merged to one run per chunk unless fragmented
        assert st["ce_copies"] == 2 * (3 if not fragment else 4)
    if load_mode == 2:
        assert st["ce_copies"] == 2 * 3 * 16


@pytest.mark.parametrize("fragment", [False, True])
@pytest.mark.parametrize("load_mode", [0, 1])
def test_offload_long_runs_store_records(load_mode, fragment):
    """f1 offload at the L8 geometry (1 MiB chunk-layers) through the SM scatter kernel, with either
    load path configured: every reserved slot then holds exactly the request's K/V record (bitwise,
    O3 in reverse), with the request's pool pages consecutive and with a hole in them."""
    L, Hq, Hkv, d, C, S, n_doc, n2q = 2, 32, 8, 128, 256, 64, 768, 90
    rng = make_rng(77)
    rig = Rig(L, Hq, Hkv, d, C, S, store_chunks=6, n_pool_pages=40, load_mode=load_mode)
    if fragment:
        for hid in (2000, 2001):
            rig.ctx.submit(hid, rng.integers(5000, 6000, S, dtype=np.uint32), n_cacheable=0)
            rig.ctx.match_prefix(hid, [])
        rig.ctx.release(2000, False)
    N = n_doc + n2q
    toks = rng.integers(0, 1000, N, dtype=np.uint32)
    rig.ctx.submit(1, toks, n_cacheable=n_doc)
    plan = rig.ctx.match_prefix(1, [])
    assert plan["n_matched"] == 0 and plan["n_reserved"] == 3
    q, k, v = [], [], []
    for l in range(L):
        ql, kl, vl = stress_values("iid", 500 + l, 0, N, Hq, Hkv, d)
        q.append(ql)
        k.append(kl)
        v.append(vl)
    q, k, v = np.stack(q), np.stack(k), np.stack(v)
    os_ = torch.cuda.Stream()
    qd, kd, vd = to_dev(q), to_dev(k), to_dev(v)
    od = torch.empty_like(qd)
    done = torch.cuda.Event(enable_timing=True)
    done.record(rig.cs)
    a = torch.cuda.Event(enable_timing=True)
    a.record(rig.cs)
    rig.ctx.run_prefill_ex(1, qd, kd, vd, od, rig.cs, rig.ls, offload_stream=os_, prefill_done_event=done)
    b = torch.cuda.Event(enable_timing=True)
    b.record(rig.cs)
    rig.cs.synchronize()
    assert 0 < a.elapsed_time(done) <= a.elapsed_time(b)   # prefill done before the offload join
    recs = pack_store_slots(k, v, 3, C)
    for c in range(3):
        got = rig.ctx.store_read(plan["slots"][c]).reshape(recs[c].shape)
        assert np.array_equal(got, recs[c]), c
    rig.ctx.release(1, True)


@pytest.mark.parametrize("mode,load_mode", [(0, 0), (1, 0), (2, 0), (3, 0), (0, 1), (3, 2)])
def test_offload_third_stream_commits_real_kv(mode, load_mode):
    """f1: the Appendix C trace where new chunks reach the store ONLY through the library's
    layer-wise offload on a third stream (pcr_run_prefill_ex); every committed slot must hold
    exactly the K/V the request computed (bitwise), and later hits must attend correctly -- in
    each of the paper's overlap settings: Up-Down, none, Only-Up, Only-Down."""
    docs, order, reqs = appendix_c_trace(0)
    model = TinyModel(L=2, Hq=4, Hkv=2, d=64, d_model=96, d_ff=128, vocab=1 << 17, seed=0)
    W = 2
    rig = Rig(2, 4, 2, 64, 64, 16, store_chunks=10, n_pool_pages=64, window=W, load_mode=load_mode)
    os_ = torch.cuda.Stream()
    for i, t in enumerate(reqs):
        rig.ctx.submit(i, t)
    for i, toks in enumerate(reqs):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W)))
        plan = rig.ctx.match_prefix(i, pend)
        _, kv, qs = model.forward(toks)
        N1 = plan["n1"]
        q = np.stack([f32_to_bf16_bits(qs[l][N1:].astype(np.float32)) for l in range(2)])
        k = np.stack([f32_to_bf16_bits(kv[l][0].astype(np.float32)) for l in range(2)])
        v = np.stack([f32_to_bf16_bits(kv[l][1].astype(np.float32)) for l in range(2)])
        qd, kd, vd = to_dev(q), to_dev(k[:, N1:]), to_dev(v[:, N1:])
        od = torch.empty_like(qd)
        t3 = rig.ctx.run_prefill_ex(i, qd, kd, vd, od, rig.cs, rig.ls, offload_stream=os_, layer_times=True,
                                    mode=mode)
        rig.cs.synchronize()
        assert t3.shape == (2, 3)
        out = to_host(od)
        for l in range(2):
            kc, vc = rig.expected_context(plan, k[:, N1:], v[:, N1:], l)
            r, m = check_attention(out[l], q[l], kc, vc, N1)
            assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (i, l, r, m)
        recs = pack_store_slots(k, v, plan["n_matched"] + plan["n_reserved"], 64)
        for c in range(plan["n_matched"], plan["n_matched"] + plan["n_reserved"]):
            got = rig.ctx.store_read(plan["slots"][c]).reshape(recs[c].shape)
            assert np.array_equal(got, recs[c]), (i, c)
            rig.store[plan["slots"][c]] = got          # mirror for expected_context of later hits
        rig.ctx.release(i, True)


@pytest.mark.parametrize("n1,n2", [(0, 200), (0, 333), (64, 300), (256, 520), (512, 200), (1024, 77), (128, 1)])
def test_split_kv_edge_sweep(n1, n2):
    """Small grids take the split-KV path; a split can hold only keys past some rows' causal
    limit (those rows see nothing in it).  Outputs must stay finite and within tolerance."""
    L, Hq, Hkv, d, C, S = 1, 32, 8, 128, 64, 16
    rig, plan, q, k, v, out = _single_request("iid", L, Hq, Hkv, d, C, S, n1, n2, seed=n1 * 7 + n2)
    from oracle.attention import bf16_bits_to_f64
    assert np.isfinite(bf16_bits_to_f64(out)).all()
    kc, vc = rig.expected_context(plan, k[:, n1:], v[:, n1:], 0)
    r, m = check_attention(out[0], q[0], kc, vc, n1, blocked=True)
    assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (r, m)


@pytest.mark.parametrize("P,load_mode,kind", [(2, 0, "iid"), (3, 1, "advfuture"), (4, 2, "kout"), (8, 0, "q4")])
def test_context_split_partials_merge_to_oracle(P, load_mode, kind):
    """shard_mode 1 (SURVEY §8(e) variant): P ranks (emulated on one GPU, one context each) split a
    request by chunk depth (chunk c -> rank c % P, the suffix keys -> rank n_matched % P).  Every
    rank's store holds NaN garbage in the slots it does not own, so a rank that touched another
    rank's chunk would poison the result.  The merged partials equal the fp64 oracle over the
    whole context; each rank's pool holds its own chunks bit for bit; its share of the new chunks
    reaches its store through the layer-wise offload."""
    L, Hq, Hkv, d, C, S = 2, 32, 8, 128, 256, 64
    n_doc, n_new, n_q = 5 * C, 2 * C, 150           # 5 cached chunks, 2 new cacheable chunks, query
    N1, N = n_doc, n_doc + n_new + n_q
    N2 = N - N1
    q, k, v = [], [], []
    for l in range(L):
        ql, kl, vl = stress_values(kind, 900 + l, N1, N2, Hq, Hkv, d)
        q.append(ql)
        k.append(kl)
        v.append(vl)
    q, k, v = np.stack(q), np.stack(k), np.stack(v)
    rng = make_rng(31)
    doc = rng.integers(0, 1000, n_doc, dtype=np.uint32)
    toks = np.concatenate([doc, rng.integers(0, 1000, N - n_doc, dtype=np.uint32)])
    recs = pack_store_slots(k, v, (n_doc + n_new) // C, C)
    garbage = np.full(recs[0].shape, 0x7FC0, np.uint16)   # bf16 NaN
    block = N2 * Hq * (d + 1)
    parts, rigs = [], []
    for r in range(P):
        rig = Rig(L, Hq, Hkv, d, C, S, store_chunks=12, n_pool_pages=N // S + 24, rank=r, world=P,
                  shard_mode=1, load_mode=load_mode)
        rig.ctx.submit(1000, np.concatenate([doc, [7]]).astype(np.uint32))
        warm = rig.ctx.match_prefix(1000, [])
        for c, slot in enumerate(warm["slots"]):
            rig.write_slot(slot, recs[c] if c % P == r else garbage)
        rig.ctx.release(1000, True)
        rig.ctx.submit(1, toks, n_cacheable=n_doc + n_new)
        plan = rig.ctx.match_prefix(1, [])
        assert plan["n_matched"] == 5 and plan["n_reserved"] == 2 and plan["n1"] == N1
        for c in range(5, 7):                            # reserved slots: garbage until offloaded
            rig.ctx.store_write(plan["slots"][c], garbage)
        part = torch.full((L, block), float("nan"), dtype=torch.float32, device="cuda")
        qd, kd, vd = to_dev(q), to_dev(k[:, N1:]), to_dev(v[:, N1:])
        os_ = torch.cuda.Stream()
        rig.ctx.run_prefill_ex(1, qd, kd, vd, None, rig.cs, rig.ls, offload_stream=os_, partial_all=part)
        rig.cs.synchronize()
        parts.append(part)
        rigs.append((rig, plan))
        # own prefix chunks in this rank's pool (bitwise), via the oracle's load on the own subset
        pool = rig.pool_np()
        ppc = C // S
        for l in range(L):
            for c in range(5):
                if c % P != r:
                    continue
                for pp in range(ppc):
                    page = plan["pages"][c * ppc + pp]
                    exp = recs[c][l][:, :, pp * S:(pp + 1) * S]            # [Hkv][2][S][d]
                    assert np.array_equal(pool[l, page], exp), (r, l, c, pp)
        # this rank's new chunks reached its store through the offload
        for c in range(5, 7):
            got = rig.ctx.store_read(plan["slots"][c]).reshape(recs[c].shape)
            assert np.array_equal(got, recs[c] if c % P == r else garbage), (r, c)
    rig0 = rigs[0][0]
    gathered = torch.stack(parts, dim=1).contiguous()    # [L][P][block]
    out = torch.empty((L, N2, Hq, d), dtype=torch.int16, device="cuda")
    for l in range(L):
        rig0.ctx.merge_partials(gathered[l], P, N2, out[l], rig0.cs)
    rig0.cs.synchronize()
    out = to_host(out)
    for l in range(L):
        r_l2, m = check_attention(out[l], q[l], k[l], v[l], N1)
        assert r_l2 <= TOL_REL_L2 and m <= TOL_MAX_ABS, (l, r_l2, m)
    for rig, _ in rigs:
        rig.ctx.release(1, False)


_PDL_SCRIPT = """
import sys, zlib
import numpy as np
sys.path.insert(0, {root!r})
from tests.test_gpu_parity import _single_request
rig, plan, q, k, v, out = _single_request("iid", 3, 32, 8, 128, 256, 64, 1024, 130, seed=5)
np.save({out_path!r}, out)
np.save({pool_path!r}, rig.pool_np())
print("CRC", zlib.crc32(out.tobytes()))
"""


def _run_variant(env_over, tmp_path):
    """The 3-layer L8-geometry request (split-KV at this shape) in a subprocess with experiment env
    switches; returns its output and pool arrays."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out_p, pool_p = str(tmp_path / "out.npy"), str(tmp_path / "pool.npy")
    res = subprocess.run([sys.executable, "-c", _PDL_SCRIPT.format(root=root, out_path=out_p, pool_path=pool_p)],
                         env=dict(os.environ, **env_over), capture_output=True, text=True, timeout=300, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    return np.load(out_p), np.load(pool_p)


def test_fused_append_and_cluster_reduce_match_the_unfused_path(tmp_path):
    """The default attention (suffix K/V read from k_new/v_new and stored into the pool by the
    kernel itself) against the separate append kernel (PCR_FUSED_APPEND=0), and the split-KV
    combine kernel against the experimental in-kernel reduce through L2 (PCR_SPLIT_SPIN=1): output
    and the whole pool bit-identical.  The experimental cluster split-KV reduce (PCR_SPLIT_CLUSTER=1: partials
    merged over DSMEM in-kernel) gives the same pool and the output within the split merge's
    rounding (another summation order), inside the oracle tolerance."""
    L, N1, N2 = 3, 1024, 130
    rig, plan, q, k, v, out = _single_request("iid", L, 32, 8, 128, 256, 64, N1, N2, seed=5)
    pool = rig.pool_np()
    out_fa, pool_fa = _run_variant({"PCR_FUSED_APPEND": "0"}, tmp_path)
    # the unfused append also zero-fills rows past N1+N2 of the last page; the fused one writes
    # the final 64-row box (zeros past N2), which here ends the page: identical arrays
    assert np.array_equal(out_fa, out)
    assert np.array_equal(pool, pool_fa)
    out_sp, pool_sp = _run_variant({"PCR_SPLIT_SPIN": "1"}, tmp_path)   # in-kernel reduce through L2
    assert np.array_equal(pool, pool_sp)                                 # instead of the combine kernel:
    assert np.array_equal(out_sp, out)                                   # same formula and order, same bits
    out_cl, pool_cl = _run_variant({"PCR_SPLIT_CLUSTER": "1"}, tmp_path)
    assert np.array_equal(pool, pool_cl)
    a, b = bf16_bits_to_f64(out), bf16_bits_to_f64(out_cl)
    assert rel_l2(a, b) <= 2e-3 and np.abs(a - b).max() <= 1e-2
    for l in range(L):
        kc, vc = rig.expected_context(plan, k[:, N1:], v[:, N1:], l)
        for o in (out, out_cl):
            r, m = check_attention(o[l], q[l], kc, vc, N1, blocked=True)
            assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (l, r, m)


def test_programmatic_dependent_launch_off_is_bitwise_identical():
    """PCR_PDL=0 (plain stream-ordered launches) gives the same bytes as the default PDL chain
    append -> attention -> split-KV combine (4 splits at this shape)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    _, _, _, _, _, out = _single_request("iid", 3, 32, 8, 128, 256, 64, 1024, 130, seed=5)
    env = dict(os.environ, PCR_PDL="0")
    res = subprocess.run([sys.executable, "-c", _PDL_SCRIPT.format(root=root, out_path="/tmp/pcr_pdl_out.npy",
                                                               pool_path="/tmp/pcr_pdl_pool.npy")],
                         env=env, capture_output=True, text=True, timeout=300, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    crc = int([ln for ln in res.stdout.splitlines() if ln.startswith("CRC")][0].split()[1])
    assert crc == zlib.crc32(out.tobytes())


def test_layer_body_reuse_equals_full_recompute():
    """f3 + O5 on the GPU: a tiny pre-norm GQA decoder (oracle/tiny_model.py weights) runs its
    SUFFIX through the per-layer C-ABI calls -- load(l) on the load stream, then on the compute
    stream RMSNorm -> Wq/Wk/Wv -> RoPE (torch fp32, rounded to bf16) -> pcr_prefill_attn_layer ->
    Wo -> MLP -- with the PREFIX's K/V reused from the DRAM store (computed once by the fp64
    model and committed).  The final hidden states of the suffix must equal the fp64 model's full
    recompute of the whole sequence (reuse-then-attend == full prefill) within the
    bf16 rounding of K/V/Q/attention output; a wrong chunk (the prefix of another document)
    breaks it by far."""
    L, Hq, Hkv, d, C, S = 2, 4, 2, 64, 64, 16
    m = TinyModel(L=L, Hq=Hq, Hkv=Hkv, d=d, d_model=96, d_ff=128, vocab=1000, seed=3)
    rng = make_rng(8)
    prefix = rng.integers(0, 1000, 4 * C, dtype=np.uint32)
    suffix = rng.integers(0, 1000, 60, dtype=np.uint32)
    toks = np.concatenate([prefix, suffix])
    N1, N2 = len(prefix), len(suffix)
    ref_full, _, _ = m.forward(toks)                       # full recompute (fp64)
    _, kv_pre, _ = m.forward(prefix)                       # the cached prefix KV (fp64)
    dev = torch.device("cuda")

    def run(kv_source):
        rig = Rig(L, Hq, Hkv, d, C, S, store_chunks=8, n_pool_pages=64)
        rig.ctx.submit(0, np.concatenate([prefix, [1]]).astype(np.uint32))
        warm = rig.ctx.match_prefix(0, [])
        kk = np.stack([f32_to_bf16_bits(kv_source[l][0].astype(np.float32)) for l in range(L)])
        vv = np.stack([f32_to_bf16_bits(kv_source[l][1].astype(np.float32)) for l in range(L)])
        recs = pack_store_slots(kk, vv, N1 // C, C)
        for c, s_ in enumerate(warm["slots"]):
            rig.write_slot(s_, recs[c])
        rig.ctx.release(0, True)
        rig.ctx.submit(1, toks, n_cacheable=N1)
        plan = rig.ctx.match_prefix(1, [])
        assert plan["n1"] == N1 and plan["n2"] == N2
        W = [{k: torch.tensor(v, dtype=torch.float32, device=dev) for k, v in lw.items()} for lw in m.layers]
        x = torch.tensor(m.emb[toks[N1:].astype(np.int64)], dtype=torch.float32, device=dev)
        pos = torch.arange(N1, N1 + N2, dtype=torch.float64, device=dev)
        half = d // 2
        inv = 10000.0 ** (-torch.arange(half, dtype=torch.float64, device=dev) / half)
        ang = pos[:, None] * inv[None, :]
        cos, sin = torch.cos(ang)[:, None, :].float(), torch.sin(ang)[:, None, :].float()

        def rope(t):
            t1, t2 = t[..., :half], t[..., half:]
            return torch.cat([t1 * cos - t2 * sin, t1 * sin + t2 * cos], dim=-1)

        def rms(t):
            return t / torch.sqrt((t * t).mean(dim=-1, keepdim=True) + 1e-6)

        out = torch.empty((L, N2, Hq, d), dtype=torch.int16, device=dev)
        ev = [torch.cuda.Event() for _ in range(L)]
        rig.ls.wait_stream(torch.cuda.current_stream())
        rig.cs.wait_stream(torch.cuda.current_stream())
        for l in range(L):
            rig.ctx.load_layer_kv(1, l, rig.ls)
            ev[l].record(rig.ls)
            with torch.cuda.stream(rig.cs):
                h = rms(x)
                q = rope((h @ W[l]["wq"]).view(N2, Hq, d)).to(torch.bfloat16).contiguous()
                k = rope((h @ W[l]["wk"]).view(N2, Hkv, d)).to(torch.bfloat16).contiguous()
                v = (h @ W[l]["wv"]).view(N2, Hkv, d).to(torch.bfloat16).contiguous()
                rig.cs.wait_event(ev[l])
                rig.ctx.prefill_attn_layer(1, l, q.view(torch.int16), k.view(torch.int16), v.view(torch.int16),
                                           out[l], rig.cs)
                x = x + out[l].view(torch.bfloat16).float().reshape(N2, Hq * d) @ W[l]["wo"]
                h = rms(x)
                a = h @ W[l]["w1"]
                x = x + (torch.nn.functional.silu(a) * (h @ W[l]["w3"])) @ W[l]["w2"]
        rig.cs.synchronize()
        rig.ctx.release(1, False)
        return x.double().cpu().numpy()

    ref = ref_full[N1:]
    got = run(kv_pre)
    err = rel_l2(got, ref)
    print(f"layer-body reuse vs full recompute: rel-L2 {err:.2e}")
    assert err <= 2e-2, err
    # negative control: the prefix KV of a different document (same positions) must not pass
    other = rng.integers(0, 1000, 4 * C, dtype=np.uint32)
    _, kv_other, _ = m.forward(other)
    assert rel_l2(run(kv_other), ref) > 10 * err


def test_two_requests_in_flight_on_two_streams():
    """Two planned requests with device work at once (max_inflight regions, separate compute and
    load streams): each has its own tables, split-KV workspace and layer counters (and the
    experimental in-kernel split reduce, which needs its whole grid resident, steps aside while
    another request is active).  Both outputs match the oracle and the pool holds both."""
    L, Hq, Hkv, d, C, S = 2, 32, 8, 128, 256, 64
    N1, N2 = 1024, 128
    rng = make_rng(71)
    rig = Rig(L, Hq, Hkv, d, C, S, store_chunks=12, n_pool_pages=64)
    reqs = []
    for rid, seed in ((1, 72), (2, 73)):
        q, k, v = [], [], []
        for l in range(L):
            ql, kl, vl = stress_values("iid", seed * 10 + l, N1, N2, Hq, Hkv, d)
            q.append(ql)
            k.append(kl)
            v.append(vl)
        q, k, v = np.stack(q), np.stack(k), np.stack(v)
        doc = rng.integers(0, 1000, N1, dtype=np.uint32)
        _warm_prefix(rig, 100 + rid, doc, k[:, :N1], v[:, :N1], N1 // C)
        rig.ctx.submit(rid, np.concatenate([doc, rng.integers(0, 1000, N2, dtype=np.uint32)]), n_cacheable=N1)
        reqs.append((rid, q, k, v))
    plans, outs, streams = {}, {}, {}
    for rid, q, k, v in reqs:
        plans[rid] = rig.ctx.match_prefix(rid, [])
        assert plans[rid]["n1"] == N1
    for rid, q, k, v in reqs:
        cs, ls = torch.cuda.Stream(), torch.cuda.Stream()
        qd, kd, vd = to_dev(q), to_dev(k[:, N1:]), to_dev(v[:, N1:])
        od = torch.empty_like(qd)
        rig.ctx.run_prefill(rid, qd, kd, vd, od, cs, ls)
        outs[rid], streams[rid] = (od, qd, kd, vd), cs
    for rid in streams:
        streams[rid].synchronize()
    pool = rig.pool_np()
    for rid, q, k, v in reqs:
        out = to_host(outs[rid][0])
        for l in range(L):
            kc, vc = rig.expected_context(plans[rid], k[:, N1:], v[:, N1:], l)
            r, m = check_attention(out[l], q[l], kc, vc, N1, blocked=True)
            assert r <= TOL_REL_L2 and m <= TOL_MAX_ABS, (rid, l, r, m)
            exp = rig.expected_pool(plans[rid], k[:, N1:], v[:, N1:], l)
            pg = plans[rid]["pages"]
            assert np.array_equal(pool[l][pg], exp[l][pg]), (rid, l)
    for rid, *_ in reqs:
        rig.ctx.release(rid, False)


@pytest.mark.gpu
def test_streamed_pipeline_with_default_priority_streams_never_starves_the_gather():
    """Regression: the streamed OVERLAP pipeline with the caller's streams at default priority and
    a multi-wave attention grid (M7-shaped suffix, 528 CTAs per layer).  The attention CTAs wait
    in-kernel for the gather's per-layer counters; the library runs the gather on its own
    greatest-priority stream so a full attention grid queued first cannot keep it from being
    dispatched (before the fix some runs ended in the attention's 10 s trap).  Every run must
    complete and give the same output as the per-layer API on the same request."""
    import torch
    from paper_2603_23049_b200 import Context
    from pcrgen import randn_bf16
    L, Hq, Hkv, d, C, S, N1, N2 = 8, 32, 8, 128, 256, 64, 4096, 4224
    rng = make_rng(31)
    n_pages = 2 * (-(-(N1 + N2) // S)) + 4
    pool = torch.zeros(n_pages * L * Hkv * 2 * S * d, dtype=torch.int16, device="cuda")
    ctx = Context(L, Hq, Hkv, d, C, S, N1 // C + 2, 0, device=torch.cuda.current_device(), pool=pool)
    doc = rng.integers(0, 1000, N1, dtype=np.uint32)
    ctx.submit(0, np.concatenate([doc, [1]]).astype(np.uint32))
    for s in ctx.match_prefix(0, [])["slots"]:
        ctx.store_write(s, randn_bf16(rng, (ctx.slot_bytes // 2,)))
    ctx.release(0, True)
    toks = np.concatenate([doc, rng.integers(0, 1000, N2, dtype=np.uint32)])
    q, k, v = (to_dev(randn_bf16(rng, (L, N2, h, d))) for h in (Hq, Hkv, Hkv))
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()   # default priority
    outs = []
    for rid in range(1, 5):
        ctx.submit(rid, toks, n_cacheable=N1)
        assert ctx.match_prefix(rid, [])["n1"] == N1
        o = torch.empty_like(q)
        ctx.run_prefill(rid, q, k, v, o, cs, ls)
        cs.synchronize()
        outs.append(to_host(o))
        ctx.release(rid, False)
    ctx.submit(9, toks, n_cacheable=N1)
    ctx.match_prefix(9, [])
    o = torch.empty_like(q)
    for l in range(L):
        ctx.load_layer_kv(9, l, ls)
        ev = torch.cuda.Event()
        ev.record(ls)
        cs.wait_event(ev)
        ctx.prefill_attn_layer(9, l, q[l], k[l], v[l], o[l], cs)
    cs.synchronize()
    ctx.release(9, False)
    ctx.close()
    for x in outs:
        assert np.array_equal(x, to_host(o))


_EPILOGUE_SCRIPT = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2603_23049_b200 import Context
from pcrgen import make_rng, randn_bf16
h = hashlib.sha256()
for (n1, n2, hq, hkv) in ((1024, 128, 32, 8), (512, 700, 32, 8), (256, 300, 8, 1)):
    L, d, C, S = 2, 128, 256, 64
    rng = make_rng(n1 + n2)
    pool = torch.zeros((2 * (-(-(n1 + n2) // S)) + 4) * L * hkv * 2 * S * d, dtype=torch.int16, device="cuda")
    ctx = Context(L, hq, hkv, d, C, S, n1 // C + 2, 0, device=0, pool=pool)
    doc = rng.integers(0, 1000, n1, dtype=np.uint32)
    ctx.submit(0, np.concatenate([doc, [1]]).astype(np.uint32))
    for s in ctx.match_prefix(0, [])["slots"]:
        ctx.store_write(s, randn_bf16(rng, (ctx.slot_bytes // 2,)))
    ctx.release(0, True)
    ctx.submit(1, np.concatenate([doc, rng.integers(0, 1000, n2, dtype=np.uint32)]), n_cacheable=n1)
    ctx.match_prefix(1, [])
    q, k, v = (torch.from_numpy(randn_bf16(rng, (L, n2, x, d)).view(np.int16)).cuda() for x in (hq, hkv, hkv))
    o = torch.empty_like(q)
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()
    ctx.run_prefill(1, q, k, v, o, cs, ls)
    cs.synchronize()
    h.update(o.cpu().numpy().tobytes())
    h.update(pool.cpu().numpy().tobytes())
    ctx.release(1, False)
    ctx.close()
print(h.hexdigest())
"""


def test_tma_store_epilogue_is_bitwise_identical_to_row_stores():
    """The TMA-store epilogue (bf16 out, and the fp32 split-KV partials a short suffix produces)
    writes exactly the bytes the per-thread row stores write (PCR_TMA_EPILOGUE=0), pool included."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _EPILOGUE_SCRIPT.format(root=root)
    digests = []
    for flag in ("1", "0"):
        env = dict(os.environ, PCR_TMA_EPILOGUE=flag)
        res = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, env=env, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        digests.append(res.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
