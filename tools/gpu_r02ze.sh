#!/bin/bash
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for i in 1 2; do timeout 300 python tools/attn_timeline.py > gpurun_out/r02ze_$i.txt 2>&1; echo "rc=$?"; grep -v "^{" gpurun_out/r02ze_$i.txt | grep -v "^ " | head -12; done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
