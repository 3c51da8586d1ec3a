"""Attention-only microbenchmark through the C-ABI (pcr_prefill_attn_layer, append + attention),
for comparing suffix_attn variants quickly.  Prints one JSON line per shape.

    python tools/attn_bench.py [--iters 20]
"""
import argparse
import json
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_23049_b200 import Context  # noqa: E402
from pcrgen import make_rng, randn_bf16  # noqa: E402


def run(n1, n2, hq, hkv, d=128, L=32, iters=20, C=256, S=64, bg=""):
    rng = make_rng(3)
    N = n1 + n2
    n_pages = 2 * (-(-N // S)) + 4
    pool = torch.empty(n_pages * L * hkv * 2 * S * d, dtype=torch.int16, device="cuda")
    ctx = Context(L, hq, hkv, d, C, S, n1 // C + 2, 0, device=0, pool=pool)
    doc = rng.integers(0, 1000, n1, dtype=np.uint32)
    if n1:
        ctx.submit(0, np.concatenate([doc, [1]]).astype(np.uint32))
        w = ctx.match_prefix(0, [])
        rec = randn_bf16(rng, (ctx.slot_bytes // 2,))
        for s in w["slots"]:
            ctx.store_write(s, rec)
        ctx.release(0, True)
    ctx.submit(1, np.concatenate([doc, rng.integers(0, 1000, n2, dtype=np.uint32)]), n_cacheable=n1)
    plan = ctx.match_prefix(1, [])
    assert plan["n1"] == n1
    dev = lambda a: torch.from_numpy(a.view(np.int16)).cuda()  # noqa: E731
    q = dev(randn_bf16(rng, (L, n2, hq, d)))
    k = dev(randn_bf16(rng, (L, n2, hkv, d)))
    v = dev(randn_bf16(rng, (L, n2, hkv, d)))
    o = torch.empty_like(q)
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()
    ctx.run_prefill(1, q, k, v, o, cs, ls)   # loads the pool, warms up
    cs.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = []
    stop = threading.Event()

    def poll():
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(0)
            while not stop.is_set():
                clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                stop.wait(0.005)
        except Exception:
            pass
    th = threading.Thread(target=poll, daemon=True)
    th.start()
    # interference experiment: a background host->HBM stream on another stream during the timed
    # region -- "gather": the SM gather kernel re-loading the request's prefix (same bytes, same
    # pages); "ce": copy-engine cudaMemcpyAsync of a pinned host buffer (no SMs)
    if bg:
        bs = torch.cuda.Stream()
        if bg == "gather":
            for _ in range(iters * 2):
                for l in range(L):
                    ctx.load_layer_kv(1, l, bs)
        elif bg == "ce":
            hb = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
            db = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            with torch.cuda.stream(bs):
                for _ in range(iters // 2 + 1):
                    db.copy_(hb, non_blocking=True)
    a.record(cs)
    for _ in range(iters):
        for l in range(L):
            ctx.prefill_attn_layer(1, l, q[l], k[l], v[l], o[l], cs)
    b.record(cs)
    b.synchronize()
    stop.set()
    th.join()
    ms = a.elapsed_time(b) / (iters * L)
    flops = 4 * hq * d * (n2 * n1 + n2 * (n2 + 1) // 2)
    ctx.release(1, False)
    ctx.close()
    if bg:
        torch.cuda.synchronize()
    return dict(n1=n1, n2=n2, hq=hq, hkv=hkv, L=L, bg=bg or None, ms_per_layer=ms, tflops=flops / ms / 1e9,
                sm_mhz=sorted(clk)[len(clk) // 2] if clk else None)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--small", action="store_true",
                    help="short-suffix shapes only: L8 at P=1/2/4/8 head slices, L70 r=1 rank slice of 8")
    ap.add_argument("--shape", default="", help="one shape n1,n2,hq,hkv")
    ap.add_argument("--layers", type=int, default=32,
                    help="layers (32 = each layer's K/V cold in L2 as in the pipeline; 4 leaves some of it warm: +5-8%%)")
    ap.add_argument("--bg", default="", choices=["", "gather", "ce"],
                    help="background host->HBM traffic during the timed region (interference experiment)")
    args = ap.parse_args()
    shapes = [(0, 8320, 32, 8), (4096, 4224, 32, 8), (6144, 2176, 32, 8), (4096, 128, 32, 8), (8192, 8320, 64, 8)]
    if args.small:
        shapes = [(4096, 128, 32, 8), (4096, 128, 16, 4), (4096, 128, 8, 2), (4096, 128, 4, 1), (16384, 128, 8, 1)]
    if args.shape:
        shapes = [tuple(int(x) for x in args.shape.split(","))]
    for n1, n2, hq, hkv in shapes:
        print(json.dumps(run(n1, n2, hq, hkv, L=args.layers, iters=args.iters, bg=args.bg)), flush=True)
