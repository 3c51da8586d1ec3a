#!/bin/bash
# long suffix on a one-kv-head slice (M7 r=0.5 at P=8): split-KV (2 splits) vs none
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for N in 136 66 136 66; do echo "PCR_ATTN_SMS=$N $(PCR_ATTN_SMS=$N timeout 300 python tools/attn_bench.py --shape 4096,4224,4,1 --iters 10 2>&1 | tail -1 | cut -c1-170)"; done
for N in 136 100; do echo "P=4 PCR_ATTN_SMS=$N $(PCR_ATTN_SMS=$N timeout 300 python tools/attn_bench.py --shape 4096,4224,8,2 --iters 10 2>&1 | tail -1 | cut -c1-170)"; done
