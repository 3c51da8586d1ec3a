#!/bin/bash
# TMA-store epilogue: full GPU suite, A/B against the per-thread row stores (PCR_TMA_EPILOGUE=0),
# the Q0-in-TMEM build on top, and the L8 per-CTA timeline
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for E in 1 0 1 0; do echo "PCR_TMA_EPILOGUE=$E"; PCR_TMA_EPILOGUE=$E timeout 300 python tools/attn_bench.py 2>&1 | tail -5; PCR_TMA_EPILOGUE=$E timeout 300 python tools/attn_bench.py --small 2>&1 | tail -5; done
PYTEST_K="attention_and_pool and not q4 or split_kv or self_consistency or page_size or l8_full or m7_half or fused_append or context_split" \
  bash tools/gpu_variant.sh "-DPCR_Q0_TMEM=1" 2>&1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 120 python tools/attn_bench.py --shape 4096,128,32,8 --iters 1 2>&1 | grep -E "^TL" > gpurun_out/r02z9_timeline_l8.txt
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
