#!/bin/bash
# 8 vs 9 split-KV CTAs per M block at the L8 short suffix (PCR_ATTN_SMS 136 vs 148), alternating
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for i in 1 2 3 4 5 6; do
  for N in 148 136; do echo "$N $(PCR_ATTN_SMS=$N timeout 300 python tools/attn_bench.py --shape 4096,128,32,8 --iters 30 2>&1 | tail -1 | cut -c90-150)"; done
done
