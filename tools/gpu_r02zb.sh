#!/bin/bash
# interference: attention alone vs with a background SM gather vs with a background copy-engine H2D
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for B in "" gather ce "" gather ce; do
  timeout 300 python tools/attn_bench.py --shape 4096,4224,32,8 ${B:+--bg $B} 2>&1 | tail -1
done
