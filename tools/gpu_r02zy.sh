#!/bin/bash
# per-CTA timeline of the one-kv-head long-suffix slice with 2 splits vs none
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for N in 136 66; do echo "PCR_ATTN_SMS=$N"; PCR_ATTN_SMS=$N timeout 300 python tools/attn_timeline.py --shape 4096,4224,4,1 2>&1 | tail -4 | cut -c1-600; done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
