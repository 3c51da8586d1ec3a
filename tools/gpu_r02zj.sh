#!/bin/bash
# short-suffix split count: PCR_ATTN_SMS caps the SMs the split-KV sizing counts on (splits = SMs / CTAs)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for N in 148 128 112 96 80 64 148; do echo "PCR_ATTN_SMS=$N"; PCR_ATTN_SMS=$N timeout 300 python tools/attn_bench.py --shape 4096,128,32,8 2>&1 | tail -1; done
for N in 148 96 64; do echo "P=8 slice PCR_ATTN_SMS=$N"; PCR_ATTN_SMS=$N timeout 300 python tools/attn_bench.py --shape 4096,128,4,1 2>&1 | tail -1; done
