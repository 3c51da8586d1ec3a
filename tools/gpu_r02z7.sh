#!/bin/bash
# 128-key tiles with the new producer; per-phase clocks of the 128-key build
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
ATTN_BENCH_ARGS="" PYTEST_K="attention_and_pool and not q4 or split_kv or self_consistency or page_size or l8_full or m7_half or fused_append" \
  bash tools/gpu_variant.sh "-DPCR_BLOCK_N=128" "-DPCR_BLOCK_N=128 -DPCR_POLY_PAIRS=3" 2>&1
for F in "-DPCR_ATTN_TIMING=1 -DPCR_BLOCK_N=128"; do
  echo "== timing flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 120 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 1 2>&1 | grep -E "TIMING" | tail -33
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
