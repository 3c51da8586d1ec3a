#!/bin/bash
# per-CTA fixed cost of the attention: same grid (N2 = 4224: 528 CTAs), N1 = 0 .. 12288
export PYTHONUNBUFFERED=1
for n1 in 0 1024 2048 4096 8192 12288; do
  timeout 300 python tools/attn_bench.py --shape $n1,4224,32,8 --iters 30 2>&1 | tail -1
done
