#!/bin/bash
# CTA timeline of a bench step (M7 r=0.5) vs the standalone pipeline script
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
PCR_BENCH_TIMELINE=1 timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "tag|timeline_step|Error|error" | cut -c1-900
timeout 300 python tools/attn_timeline.py 2>&1 | tail -4 | cut -c1-900
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
