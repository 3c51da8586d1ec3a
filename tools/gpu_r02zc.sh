#!/bin/bash
# per-CTA timeline of the attention in the streamed pipeline vs alone (M7 r=0.5, L70 slice shape)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 300 python tools/attn_timeline.py 2>&1 | tail -4
timeout 300 python tools/attn_timeline.py 2>&1 | tail -4
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
