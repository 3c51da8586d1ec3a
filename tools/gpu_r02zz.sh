#!/bin/bash
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
PCR_ATTN_SMS=136 timeout 300 python tools/attn_timeline.py --shape 4096,4224,4,1 --dump gpurun_out/r02zz_split2.npz 2>&1 | tail -1 | cut -c1-200
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
