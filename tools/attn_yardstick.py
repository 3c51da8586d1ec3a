"""External yardstick (optional; not on the product path): the image's flashinfer
prefill kernels on the same suffix-attention problems as tools/attn_bench.py (contiguous K/V,
causal with the bottom-right alignment = suffix rows at absolute positions N1 + i).  Prints one
JSON line per (shape, backend) with TF/s by the same flop formula.

    python tools/attn_yardstick.py
"""
import json
import sys

import torch


def main():
    import flashinfer
    shapes = [(4096, 4224, 32, 8), (0, 8320, 32, 8), (6144, 2176, 32, 8), (4096, 128, 32, 8)]
    for n1, n2, hq, hkv in shapes:
        d = 128
        g = torch.Generator(device="cuda").manual_seed(0)
        q = torch.randn(n2, hq, d, device="cuda", dtype=torch.bfloat16, generator=g)
        k = torch.randn(n1 + n2, hkv, d, device="cuda", dtype=torch.bfloat16, generator=g)
        v = torch.randn(n1 + n2, hkv, d, device="cuda", dtype=torch.bfloat16, generator=g)
        flops = 4 * hq * d * (n2 * n1 + n2 * (n2 + 1) // 2)
        # trtllm-gen Blackwell FMHA through the paged context API (page 64, K and V caches
        # [pages][Hkv][64][d]); checked against the fa2 output of the same inputs
        try:
            S = 64
            n = n1 + n2
            n_pages = -(-n // S)
            pad = n_pages * S - n
            kc = torch.cat([k, k.new_zeros(pad, hkv, d)]).view(n_pages, S, hkv, d).transpose(1, 2).contiguous()
            vc = torch.cat([v, v.new_zeros(pad, hkv, d)]).view(n_pages, S, hkv, d).transpose(1, 2).contiguous()
            ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
            bt = torch.arange(n_pages, dtype=torch.int32, device="cuda").view(1, -1)
            sl = torch.tensor([n], dtype=torch.int32, device="cuda")
            cq = torch.tensor([0, n2], dtype=torch.int32, device="cuda")
            ck = torch.tensor([0, n], dtype=torch.int32, device="cuda")
            ft = lambda: flashinfer.prefill.trtllm_batch_context_with_kv_cache(  # noqa: E731
                q, (kc, vc), ws, bt, sl, n2, n, d ** -0.5, 1.0, 1, cq, ck, kv_layout="HND", causal=True)
            o_t = ft()
            o_r = flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, backend="fa2")
            rel = float((o_t.float() - o_r.float()).norm() / o_r.float().norm())
            for _ in range(3):
                ft()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                ft()
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b) / 20
            print(json.dumps({"n1": n1, "n2": n2, "hq": hq, "hkv": hkv, "backend": "trtllm-gen (paged context)",
                              "ms": ms, "tflops": flops / ms / 1e9, "rel_l2_vs_fa2": rel}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"n1": n1, "n2": n2, "backend": "trtllm-gen (paged context)", "error": str(e)[:400]}),
                  flush=True)
        for backend in ("auto", "fa2"):
            try:
                f = lambda: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, backend=backend)  # noqa: E731
                for _ in range(3):
                    f()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                iters = 20
                a.record()
                for _ in range(iters):
                    f()
                b.record()
                b.synchronize()
                ms = a.elapsed_time(b) / iters
                print(json.dumps({"n1": n1, "n2": n2, "hq": hq, "hkv": hkv, "backend": backend, "ms": ms,
                                  "tflops": flops / ms / 1e9}), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"n1": n1, "n2": n2, "backend": backend, "error": str(e)[:300]}), flush=True)


if __name__ == "__main__":
    sys.exit(main())
