#!/bin/bash
# Q tile 0 in TMEM (three rotating S buffers) with the new producer; per-CTA timeline of the default
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PYTEST_K="attention_and_pool and not q4 or split_kv or self_consistency or page_size or l8_full or m7_half or fused_append" \
  bash tools/gpu_variant.sh "-DPCR_Q0_TMEM=1" "" 2>&1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 120 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 1 2>&1 | grep -E "^TL" > gpurun_out/r02z8_timeline_m7.txt
timeout 120 python tools/attn_bench.py --shape 4096,128,32,8 --iters 1 2>&1 | grep -E "^TL" > gpurun_out/r02z8_timeline_l8.txt
wc -l gpurun_out/r02z8_timeline_*.txt
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
