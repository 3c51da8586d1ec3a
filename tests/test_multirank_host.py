"""Multi-rank host control on CPU (gloo, world_size 2): every rank's libpcr context plans the
same trace independently; plans, evictions and leaf order must agree across ranks (no control
traffic is needed), and each rank's store record is its 1/P head slice: a record
written on every rank from its heads of the full record reads back bit-exactly, and the ranks'
records concatenated by KV head (all-gathered over gloo) are the full record.  O7 on the oracle:
the ranks' attention outputs for their query heads, all-gathered and concatenated by head, equal
the single-rank output (the layout pcr_run_prefill_sharded re-assembles on GPUs)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from pcrgen import appendix_c_trace, make_rng, random_tiny_trace


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, shard_mode=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_23049_b200 import Context
        L, Hq, Hkv, d, C, S = 2, 8, 4, 16, 64, 16
        split = 1 if shard_mode == 1 else world          # context split: all heads on every rank
        page_bytes = L * (Hkv // split) * 2 * S * d * 2
        ctx = Context(L, Hq, Hkv, d, C, S, 10, 2, device=-1, pool_bytes=256 * page_bytes, rank=rank, world=world,
                      shard_mode=shard_mode)
        _, _, reqs = appendix_c_trace(0)
        reqs = list(reqs) + random_tiny_trace(make_rng(5), C=C, n_docs=4, max_doc_chunks=3, n_requests=20,
                                              query_len=(1, 70))
        for i, t in enumerate(reqs):
            ctx.submit(i, t)
        log = []
        for i in range(len(reqs)):
            pend = list(range(i + 1, min(len(reqs), i + 3)))
            p = ctx.match_prefix(i, pend)
            log.append((p["n_matched"], p["n_reserved"], p["slots"], p["pages"], p["evicted"]))
            ctx.release(i, i % 3 != 2)
        log.append(ctx.leaf_list())
        logs = [None] * world
        dist.all_gather_object(logs, log)
        slot_bytes = [None] * world
        dist.all_gather_object(slot_bytes, ctx.slot_bytes)
        ok_store = ok_attn = True
        if shard_mode == 0:
            import torch
            from oracle.attention import bf16_bits_to_f64, suffix_attention
            from pcrgen import randn_bf16
            full = randn_bf16(make_rng(21), (L, Hkv, 2, C, d))              # one chunk, all heads
            hs = slice(rank * Hkv // world, (rank + 1) * Hkv // world)
            mine = np.ascontiguousarray(full[:, hs])
            ctx.store_write(3, mine)
            back = ctx.store_read(3).reshape(mine.shape)
            ok_store = bool(np.array_equal(back, mine))
            parts = [torch.zeros(back.shape, dtype=torch.int32) for _ in range(world)]   # (gloo: no int16)
            dist.all_gather(parts, torch.from_numpy(back.astype(np.int32)))
            cat = np.concatenate([p_.numpy().astype(np.uint16) for p_ in parts], axis=1)
            ok_store = ok_store and bool(np.array_equal(cat, full))
            # O7: head-sliced attention re-assembled by head == single rank
            n1, n2 = 64, 24
            qf = bf16_bits_to_f64(randn_bf16(make_rng(22), (n2, Hq, d)))
            kf = bf16_bits_to_f64(randn_bf16(make_rng(23), (n1 + n2, Hkv, d)))
            vf = bf16_bits_to_f64(randn_bf16(make_rng(24), (n1 + n2, Hkv, d)))
            qs = slice(rank * Hq // world, (rank + 1) * Hq // world)
            o_mine, _ = suffix_attention(qf[:, qs], kf[:, hs], vf[:, hs], n1)
            outs = [torch.zeros(o_mine.shape, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(outs, torch.from_numpy(o_mine))
            o_cat = np.concatenate([o_.numpy() for o_ in outs], axis=1)
            o_one, _ = suffix_attention(qf, kf, vf, n1)
            ok_attn = bool(np.array_equal(o_cat, o_one))
        q.put((rank, logs == [logs[0]] * world, slot_bytes, L * Hkv * 2 * C * d * 2 // split, ok_store, ok_attn))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shard_mode", [0, 1])
def test_two_ranks_replicate_host_decisions(shard_mode):
    """Both sharding modes (KV heads; context split, where each rank keeps all heads and owns the
    chunks at depth c % P) replicate the host plan without any control traffic."""
    pytest.importorskip("paper_2603_23049_b200.pcr")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, shard_mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, slot_bytes, full_bytes, ok_store, ok_attn in res:
        assert same, f"rank {rank} diverged"
        assert slot_bytes == [full_bytes] * world
        assert ok_store, f"rank {rank}: head-sliced store record"
        assert ok_attn, f"rank {rank}: head-sharded attention re-assembly"
