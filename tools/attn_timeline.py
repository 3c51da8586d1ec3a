"""Per-CTA timeline of suffix_attn inside the layer pipeline vs the attention alone (experiment;
needs the -DPCR_ATTN_TIMELINE=1 build: PCR_NVCC_EXTRA=-DPCR_ATTN_TIMELINE=1 python -m
paper_2603_23049_b200.build --force).  M7-shaped request (32 layers), streamed OVERLAP pipeline.

    python tools/attn_timeline.py [--shape n1,n2,hq,hkv]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_23049_b200 import Context, load_library  # noqa: E402
from pcrgen import make_rng, randn_bf16  # noqa: E402

TL_L, TL_C = 128, 2048


def read_tl(lib):
    buf = np.zeros((TL_L, TL_C, 6), dtype=np.uint64)
    assert lib.pcr_debug_attn_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_longlong(buf.nbytes)) == 0
    return buf


def summarise(tl, L, tag):
    recs = [tl[l][tl[l][:, 0] > 0].astype(np.int64) for l in range(L)]
    t0 = min(r[:, 0].min() for r in recs)
    starts = [r[:, 0].min() - t0 for r in recs]
    ends = [r[:, 3].max() - t0 for r in recs]
    loop0 = [r[:, 1].min() - t0 for r in recs]
    per = np.diff(ends) / 1e3
    pro = np.concatenate([(r[:, 1] - r[:, 0]) / 1e3 for r in recs[1:]])
    loop = np.concatenate([(r[:, 2] - r[:, 1]) / 1e3 for r in recs[1:]])
    epi = np.concatenate([(r[:, 3] - r[:, 2]) / 1e3 for r in recs[1:]])
    # SM-time: busy fraction of 148 SMs between the first start and last end of layers 1..L-1
    span = (ends[-1] - ends[0]) / 1e3
    busy = sum(((r[:, 3] - r[:, 0]).sum()) for r in recs[1:]) / 1e3
    out = dict(tag=tag, layers=L, ctas=int(len(recs[0])), end_to_end_ms=(ends[-1] - starts[0]) / 1e6,
               per_layer_us_median=float(np.median(per)), per_layer_us_mean=float(per.mean()),
               prologue_us=dict(mean=float(pro.mean()), p90=float(np.percentile(pro, 90)), max=float(pro.max())),
               loop_us_mean=float(loop.mean()), epilogue_us_mean=float(epi.mean()),
               sm_busy_frac=busy / (148 * span) if span > 0 else None,
               layer_start_vs_prev_end_us=float(np.median([(starts[l] - ends[l - 1]) / 1e3 for l in range(1, L)])),
               first_loop_vs_start_us=float(np.median([(loop0[l] - starts[l]) / 1e3 for l in range(1, L)])))
    print(json.dumps(out), flush=True)
    return recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="4096,4224,32,8")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--dump", default="", help="save the raw timelines (npz) to this path")
    args = ap.parse_args()
    n1, n2, hq, hkv = (int(x) for x in args.shape.split(","))
    d, C, S, L = 128, 256, 64, args.layers
    lib = load_library()
    if not hasattr(lib, "pcr_debug_attn_timeline"):
        sys.exit("build with -DPCR_ATTN_TIMELINE=1")
    lib.pcr_debug_attn_timeline.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
    rng = make_rng(3)
    N = n1 + n2
    n_pages = 2 * (-(-N // S)) + 4
    pool = torch.empty(n_pages * L * hkv * 2 * S * d, dtype=torch.int16, device="cuda")
    ctx = Context(L, hq, hkv, d, C, S, n1 // C + 2, 0, device=0, pool=pool)
    doc = rng.integers(0, 1000, n1, dtype=np.uint32)
    ctx.submit(0, np.concatenate([doc, [1]]).astype(np.uint32))
    w = ctx.match_prefix(0, [])
    rec = randn_bf16(rng, (ctx.slot_bytes // 2,))
    for s in w["slots"]:
        ctx.store_write(s, rec)
    ctx.release(0, True)
    ctx.submit(1, np.concatenate([doc, rng.integers(0, 1000, n2, dtype=np.uint32)]), n_cacheable=n1)
    assert ctx.match_prefix(1, [])["n1"] == n1
    dev = lambda a: torch.from_numpy(a.view(np.int16)).cuda()  # noqa: E731
    q = dev(randn_bf16(rng, (L, n2, hq, d)))
    k = dev(randn_bf16(rng, (L, n2, hkv, d)))
    v = dev(randn_bf16(rng, (L, n2, hkv, d)))
    o = torch.empty_like(q)
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        ctx.run_prefill(1, q, k, v, o, cs, ls)
    cs.synchronize()
    lib.pcr_debug_attn_timeline_clear()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cs)
    ctx.run_prefill(1, q, k, v, o, cs, ls)
    b.record(cs)
    torch.cuda.synchronize()
    print(json.dumps({"pipeline_ttft_ms": a.elapsed_time(b)}))
    tl_pipe = read_tl(lib)
    summarise(tl_pipe, L, "pipeline (streamed OVERLAP)")
    # the attention alone, back to back (pool already loaded)
    lib.pcr_debug_attn_timeline_clear()
    a.record(cs)
    for l in range(L):
        ctx.prefill_attn_layer(1, l, q[l], k[l], v[l], o[l], cs)
    b.record(cs)
    torch.cuda.synchronize()
    print(json.dumps({"attention_only_ms": a.elapsed_time(b)}))
    tl_alone = read_tl(lib)
    summarise(tl_alone, L, "attention only")
    if args.dump:
        np.savez_compressed(args.dump, pipeline=tl_pipe[:L], alone=tl_alone[:L])
    ctx.release(1, False)
    ctx.close()


if __name__ == "__main__":
    main()
