#!/bin/bash
# short-suffix split count sweep (PCR_ATTN_SMS): L8, the P=2 slice and the L70 r=1 slice
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for SH in 4096,128,32,8 4096,128,16,4 16384,128,8,1; do
  for N in 148 140 136 128 120 148 128; do echo "$SH PCR_ATTN_SMS=$N $(PCR_ATTN_SMS=$N timeout 300 python tools/attn_bench.py --shape $SH --iters 30 2>&1 | tail -1 | cut -c1-150)"; done
done
