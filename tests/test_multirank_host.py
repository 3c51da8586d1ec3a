"""Multi-rank host control on CPU (gloo, world_size 2): every rank's libpcr context plans the
same trace independently; plans, evictions and leaf order must agree across ranks (no control
traffic is needed), and each rank's store record is its 1/P head slice."""
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
        q.put((rank, logs == [logs[0]] * world, slot_bytes, L * Hkv * 2 * C * d * 2 // split))
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
    for rank, same, slot_bytes, full_bytes in res:
        assert same, f"rank {rank} diverged"
        assert slot_bytes == [full_bytes] * world
